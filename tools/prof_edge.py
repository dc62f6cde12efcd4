"""Profiling driver: the bench workload's fused edge pass, a few launches (for ncu -k edge_kernel).

  python tools/prof_edge.py [--config C5] [--reps 3] [--order rcm]
Launch order: 1 objective pass (plp_fgrad), then `reps` fused plp_fgrad_hessvec calls.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import get_graph, CONFIG_KP  # noqa: E402
from paper_2605_26975_b200 import plp  # noqa: E402
from plp_inputs import draw_U, draw_eta  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--order", default="rcm")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--p", type=float, default=None)
    args = ap.parse_args()
    k, p = CONFIG_KP[args.config]
    if args.p is not None:
        p = args.p
    g = get_graph(args.config, args.order)
    ctx = plp.Context(0)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=0)
    U = torch.from_numpy(draw_U(g.n, k, 0)).cuda()
    eta = torch.from_numpy(draw_eta(g.n, k, 0)).cuda()
    F, AB, _ = plp.fgrad(ctx, G, U, p, want_grad=False)
    outs = None
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(args.reps):
        outs = plp.fgrad_hessvec(ctx, G, U, eta, p, AB_in=AB)
    torch.cuda.synchronize()
    print(f"{args.config} n={g.n} nnz={g.nnz} k={k} p={p}: {1e3 * (time.time() - t0) / args.reps:.3f} ms/call "
          f"F={outs[0].item():.12g}")


if __name__ == "__main__":
    main()
