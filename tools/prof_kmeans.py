"""Profiling driver: k-means (a11) on an n x k embedding of the bench workload's size, a few Lloyd
iterations (for the ncu launch list and `ncu -k regex:km_assign`).

  python tools/prof_kmeans.py [--n 8388608] [--k 8] [--iters 3] [--time 5]
Launch order: the k-means++ seeding (K - 1 km_d2_kernel / km_pick_kernel rounds), then per Lloyd
iteration km_update_kernel, km_assign_mma_kernel (K, dim <= 8) and km_sum_kernel.
--time R also prints the Lloyd iteration's wall time per iteration (R repetitions, CUDA events).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_26975_b200 import plp  # noqa: E402
from plp_inputs import draw_U, draw_uniforms  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8388608, help="points (default: C5's n)")
    ap.add_argument("--k", type=int, default=8, help="clusters = embedding columns (default: C5's k)")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--time", type=int, default=0)
    args = ap.parse_args()
    n, k = args.n, args.k
    ctx = plp.Context(0)
    U = torch.from_numpy(draw_U(n, k, 0)).cuda()
    u = draw_uniforms(1, k)
    labels, cent, sse, iters = plp.kmeans(ctx, U, k, u, restarts=1, max_iters=args.iters, rel_tol=0.0)
    torch.cuda.synchronize()
    out = {"n": n, "k": k, "lloyd_iters": iters, "sse": sse}
    if args.time > 0:
        def timed(mi):
            ts = []
            for _ in range(args.time):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                plp.kmeans(ctx, U, k, u, restarts=1, max_iters=mi, rel_tol=0.0)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            return ts[len(ts) // 2]
        m0, m1 = timed(0), timed(20)
        out["lloyd_iteration_ms"] = (m1 - m0) / 20
        out["seeding_ms"] = m0
        out["algorithmic_bytes_per_iteration"] = 8 * n * k + 4 * n
    print(json.dumps(out))


if __name__ == "__main__":
    main()
