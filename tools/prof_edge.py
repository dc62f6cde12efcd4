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
    ap.add_argument("--order", default="tile")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--p", type=float, default=None)
    ap.add_argument("--events", action="store_true", help="also time the edge kernel with CUDA events")
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
    if args.events:
        import json
        Gr, Hv = outs[2], outs[3]
        for _ in range(3):
            plp.edge_pass(ctx, G, U, eta, p, 1e-9, AB_in=AB, G=Gr, Hv=Hv)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.reps + 1)]
        torch.cuda.synchronize()
        ev[0].record()
        for i in range(args.reps):
            plp.edge_pass(ctx, G, U, eta, p, 1e-9, AB_in=AB, G=Gr, Hv=Hv)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(args.reps))
        byts = 12 * g.nnz + 4 * (g.n + 1) + 32 * g.n * k
        print(json.dumps({"config": args.config, "k": k, "p": p, "kernel_ms_median": ts[len(ts) // 2],
                          "kernel_ms_min": ts[0], "GBps": byts / (ts[len(ts) // 2] * 1e-3) / 1e9,
                          "GNNZk": g.nnz * k / (ts[len(ts) // 2] * 1e-3) / 1e9,
                          "F": outs[0].item()}))


if __name__ == "__main__":
    main()
