"""Wall time of the GPU solver (continuation solve, graphs in the library's tile order) under the
tCG variants: host-driven loop,
device-resident launches, CUDA-graph replay, fused passes (k = 8, 16).  Prints one JSON line per
(config, variant): seconds, outer and tCG iterations, ms per tCG iteration, final F.

  python tools/solver_time.py [C1 C2:20000 D16:8192 C5]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from plp_inputs import make_config, draw_U  # noqa: E402
from paper_2605_26975_b200 import plp, solver  # noqa: E402

RUNS = {"C1": (3, [2.0, 1.8, 1.5, 1.2], None), "C2": (2, [2.0, 1.1], None), "D16": (4, [2.0, 1.5], None),
        "C5": (8, [2.0], 4), "D20": (8, [2.0, 1.5], None)}
VARIANTS = {"host": dict(device_tcg=False), "device": dict(tcg_graph=False, tcg_fused=False),
            "graph": dict(tcg_fused=False), "fused": dict(tcg_graph=False, tcg_fused=True),
            "fused+graph": dict(tcg_fused=True)}


def main():
    specs = sys.argv[1:] or ["C1", "C2:20000", "D16:8192"]
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = plp.Context(0, stream)
    for spec in specs:
        name, _, nn = spec.partition(":")
        if not nn:
            from bench import get_graph
            g = get_graph(name, "tile")
        else:  # the library's tile order (RCM + BFS tiles), as the product path uses
            from plp_inputs import Graph
            g0 = make_config(name, n=int(nn))
            rp, col, w = plp.permute_csr(g0.row_ptr, g0.col, g0.w, plp.tile_order(g0.row_ptr, g0.col))
            g = Graph(name, g0.n, rp, col, w)
        k, sched, max_outer = RUNS[name]
        G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
        Z = torch.from_numpy(draw_U(g.n, k, 0)).cuda()
        for vname, kw in VARIANTS.items():
            if "fused" in vname and not (k in (8, 16) or (k in (1, 2, 4) and g.n * k % 8 == 0)):
                continue
            cfg = solver.SolverConfig(**kw)
            if max_outer:
                cfg.max_outer = max_outer
            solver.continuation_solve(ctx, G, Z, sched[:1], cfg)  # warm-up (graphs, allocator)
            torch.cuda.synchronize()
            t = time.perf_counter()
            U, tr = solver.continuation_solve(ctx, G, Z, sched, cfg)
            torch.cuda.synchronize()
            sec = time.perf_counter() - t
            nt = sum(r.tcg_iters for r in tr.records)
            print(json.dumps({"config": name, "n": g.n, "nnz": g.nnz, "k": k, "variant": vname, "seconds": sec,
                              "outer": len(tr.records), "tcg_iters": nt,
                              "ms_per_tcg_iter": 1e3 * sec / max(nt, 1), "F": tr.records[-1].F}), flush=True)


if __name__ == "__main__":
    main()
