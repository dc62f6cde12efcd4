"""NEXT-4 on one GPU: each rank's share of the multi-GPU step, measured alone.

  python tools/rank_share.py [--config C5] [--gpus 1,2,4,8] [--reps 20]

For N ranks the tile-ordered graph is split as bench.py --gpus N splits it (dist.row_bounds:
contiguous row blocks balanced on bytes, aligned to the halo kernel's tiles).  For every rank r the
tool builds that rank's local CSR exactly as plp_create_graph_dist does (owned columns j - r0, the
sorted halo after them), and times, on this one GPU, the fused F / G / Hv pass of the rank's rows
(the compute of its plp_fgrad_hessvec call) with CUDA events.  It also reports the bytes each rank
receives per step (the U and eta halo rows).  Nothing here measures the NCCL exchange or runs two
ranks at once: the per-rank times are what each GPU computes; the step on N GPUs also waits for the
halo exchange (overlapped with the interior tiles) and the A, B all-reduce.  Output: one JSON line
per N with the slowest rank's time, the aggregate GNNZ*k/s it implies (global nnz k / slowest
rank) and the halo volume."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import get_graph, CONFIG_KP  # noqa: E402
from paper_2605_26975_b200 import plp  # noqa: E402
from paper_2605_26975_b200.dist import row_bounds  # noqa: E402
from plp_inputs import draw_U, draw_eta  # noqa: E402


def local_csr(g, r0, r1):
    rp = g.row_ptr[r0:r1 + 1].astype(np.int64)
    col = g.col[rp[0]:rp[-1]].astype(np.int64)
    w = g.w[rp[0]:rp[-1]]
    rp = rp - rp[0]
    outside = (col < r0) | (col >= r1)
    halo = np.unique(col[outside])
    loc = np.where(outside, (r1 - r0) + np.searchsorted(halo, col), col - r0).astype(np.int32)
    return rp, loc, w, halo


def time_pass(ctx, G, U, E, p, AB, reps):
    for _ in range(3):
        plp.fgrad_hessvec(ctx, G, U, E, p, AB_in=AB)
    s = ctx.stream if hasattr(ctx, "stream") else None
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        plp.fgrad_hessvec(ctx, G, U, E, p, AB_in=AB)
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    k, p = CONFIG_KP[a.config]
    g = get_graph(a.config, "tile")
    ctx = plp.Context(0)
    U = draw_U(g.n, k, 0)
    E = draw_eta(g.n, k, 0)
    Gf = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=0)
    _, AB, _ = plp.fgrad(ctx, Gf, torch.from_numpy(U).cuda(), p, want_grad=False)
    del Gf
    for N in [int(x) for x in a.gpus.split(",")]:
        b = row_bounds(g.row_ptr, N, k)
        ranks = []
        for r in range(N):
            r0, r1 = int(b[r]), int(b[r + 1])
            rp, loc, w, halo = local_csr(g, r0, r1)
            n_own = r1 - r0
            G = plp.Graph(ctx, rp, loc, w, n_cols=n_own + halo.size, flags=0)
            rows = np.concatenate([np.arange(r0, r1), halo])
            Ul = torch.from_numpy(np.ascontiguousarray(U[rows])).cuda()
            El = torch.from_numpy(np.ascontiguousarray(E[rows])).cuda()
            ms = time_pass(ctx, G, Ul, El, p, AB, a.reps)
            ranks.append({"rank": r, "rows": n_own, "nnz": int(rp[-1]), "halo_rows": int(halo.size),
                          "halo_recv_MB": round(halo.size * k * 8 * 2 / 1e6, 3), "ms": round(ms, 4),
                          "kernel": plp.last_edge_kernel()})
            del G, Ul, El
            torch.cuda.empty_cache()
        slow = max(x["ms"] for x in ranks)
        print(json.dumps({"config": a.config, "k": k, "p": p, "n_gpus": N, "slowest_rank_ms": slow,
                          "aggregate_GNNZk_if_compute_bound": round(g.nnz * k / (slow * 1e-3) / 1e9, 1),
                          "max_halo_recv_MB": max(x["halo_recv_MB"] for x in ranks),
                          "ranks": ranks, "note": "each rank's share timed alone on one GPU; exchange not measured"}),
              flush=True)


if __name__ == "__main__":
    main()
