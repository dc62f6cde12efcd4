"""Runtime breakdown of a GPU continuation solve + clustering by component (SURVEY.md §8(f) NEXT-4's
"runtime breakdown per component", on one GPU): kernel time per family from the CUDA activity trace
(torch.profiler / CUPTI sees every kernel in the process, including libplp's), against wall time.

  python tools/solver_breakdown.py [D20] [--k 8] [--sched 2.0,1.5] [--graphs]"""
import argparse
import json
import os
import sys
import time
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import get_graph  # noqa: E402
from paper_2605_26975_b200 import plp, solver  # noqa: E402
from plp_inputs import draw_U, draw_uniforms  # noqa: E402

FAMILIES = [("edge pass (a3-a7)", ("edge_halo", "edge_staged", "edge_kernel", "edge_finalize",
                                   "full_epilogue", "objective_from")),
            ("tCG fused passes (NEXT-2)", ("tcg_gram_a", "tcg_update", "tcg_finish", "tcg_reduce", "tcg_expand")),
            ("tCG scalars / axpby (NEXT-1)", ("tcg_", "axpby_dev")),
            ("Gram / apply / Cholesky (a8, a9)", ("gram", "apply", "chol", "rmul", "sum_partials", "rinv")),
            ("dot / axpby / gather (a10)", ("dot_kernel", "axpby_kernel", "gather")),
            ("k-means (a11)", ("km_",)),
            ("RCut (a12)", ("rcut",))]


def family(name):
    for fam, keys in FAMILIES:
        if any(k in name for k in keys):
            return fam
    return "other (torch copies, fills)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", nargs="?", default="D20")
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--sched", default="2.0,1.5")
    ap.add_argument("--graphs", action="store_true", help="replay tCG batches as CUDA graphs")
    ap.add_argument("--fused", action="store_true", help="fused tCG passes also for k = 1, 2, 4 (folded)")
    a = ap.parse_args()
    sched = [float(x) for x in a.sched.split(",")]
    g = get_graph(a.config, "tile")
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = plp.Context(0, stream)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    Z = torch.from_numpy(draw_U(g.n, a.k, 0)).cuda()
    u = draw_uniforms(10, a.k)
    cfg = solver.SolverConfig(tcg_graph=a.graphs, tcg_fused=True if a.fused else None)
    solver.continuation_solve(ctx, G, Z, sched[:1], solver.SolverConfig(tcg_graph=a.graphs, max_outer=2))
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t = time.time()
        U, tr = solver.continuation_solve(ctx, G, Z, sched, cfg)
        lab, rc, sse = solver.cluster(ctx, G, U, a.k, u)
        torch.cuda.synchronize()
        wall = time.time() - t
    agg = defaultdict(float)
    cnt = defaultdict(int)
    per = defaultdict(lambda: [0.0, 0])
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            fam = family(ev.name)
            us = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
            agg[fam] += us / 1e3
            cnt[fam] += 1
            per[ev.name][0] += us / 1e3
            per[ev.name][1] += 1
    gpu = sum(agg.values())
    out = {"config": a.config, "n": g.n, "nnz": g.nnz, "k": a.k, "schedule": sched, "graphs": a.graphs,
           "fused_tcg": cfg.resolved(g.n, a.k).tcg_fused, "wall_s": wall,
           "gpu_busy_s": gpu / 1e3, "outer": len(tr.records), "tcg_iters": sum(r.tcg_iters for r in tr.records),
           "rcut": rc, "components_ms": {k: round(v, 3) for k, v in sorted(agg.items(), key=lambda x: -x[1])},
           "launches": dict(cnt),
           "top_kernels": [{"name": k[:120], "ms": round(v[0], 3), "launches": v[1], "ms_per_launch": round(v[0] / v[1], 4)}
                           for k, v in sorted(per.items(), key=lambda x: -x[1][0])[:12]]}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
