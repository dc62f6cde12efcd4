"""NEXT-3 quality study (direction of PAPER.md Table I): on Delaunay graphs of
uniform points, cluster with the p = 2 spectral solution and with p-continuation to p_final, and
compare the balanced cut RCut of the k-means labels.  One JSON line per (graph, schedule).

  python tools/quality_study.py [D16 D20 ...] [--k 4] [--pfinal 1.2]"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import get_graph  # noqa: E402
from paper_2605_26975_b200 import plp, solver  # noqa: E402
from plp_inputs import draw_U, draw_uniforms  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["D16", "D20"])
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--pfinal", type=float, default=1.2)
    ap.add_argument("--fused", action="store_true", help="fused tCG passes also for k = 1, 2, 4 (folded)")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)  # a created stream: the solver replays tCG batches as CUDA graphs
    ctx = plp.Context(0, stream)
    for cfg in args.configs:
        g = get_graph(cfg, "tile")
        G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
        Z = torch.from_numpy(draw_U(g.n, args.k, 0)).cuda()
        u = draw_uniforms(10, args.k)
        for sched in ([2.0], [2.0, 1.6, args.pfinal]):
            t = time.time()
            U, tr = solver.continuation_solve(ctx, G, Z, sched,
                                              solver.SolverConfig(tcg_fused=True if args.fused else None))
            torch.cuda.synchronize()
            ts = time.time() - t
            t = time.time()
            lab, rc, sse = solver.cluster(ctx, G, U, args.k, u)
            tc = time.time() - t
            sizes = torch.bincount(lab.long(), minlength=args.k).tolist()
            print(json.dumps({"graph": cfg, "n": g.n, "nnz": g.nnz, "k": args.k, "schedule": sched,
                              "rcut": rc, "cluster_sizes": sizes, "F_final": tr.records[-1].F,
                              "outer_iters": len(tr.records),
                              "tcg_iters": sum(r.tcg_iters for r in tr.records), "solve_s": ts, "fused": args.fused,
                              "cluster_s": tc}),
                  flush=True)


if __name__ == "__main__":
    main()
