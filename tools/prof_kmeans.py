"""One k-means call at a config (restarts 1, a few Lloyd iterations), for ncu launch lists and
captures of the k-means kernels.

  python tools/prof_kmeans.py [--config C5] [--iters 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import get_graph, CONFIG_KP  # noqa: E402
from paper_2605_26975_b200 import plp  # noqa: E402
from plp_inputs import draw_U, draw_uniforms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
k, _ = CONFIG_KP[a.config]
g = get_graph(a.config, "tile")
ctx = plp.Context(0)
U = torch.from_numpy(draw_U(g.n, k, 0)).cuda()
u = draw_uniforms(1, k)
lab, cent, sse, it = plp.kmeans(ctx, U, k, u, restarts=1, max_iters=a.iters, rel_tol=0.0)
plp.rcut(ctx, plp.Graph(ctx, g.row_ptr, g.col, g.w), k, lab)
torch.cuda.synchronize()
print("ok", sse, it)
