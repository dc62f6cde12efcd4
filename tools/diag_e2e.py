"""Diagnostic: GPU continuation solve vs the oracle solver, outer iteration by outer iteration.

  python tools/diag_e2e.py D16 8192 4 2.0,1.5 [--order tile|gen] [--oracle-cache DIR]
Prints one JSON line per outer iteration of each solver (p, it, F, |grad|, delta, tCG iterations,
status, rho, accepted), then the labels / RCut comparison.  Env knobs of libplp (PLP_EDGE_STAGED,
...) select the edge kernel, so the same command shows whether a divergence follows the kernel.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from oracle import solver as osol  # noqa: E402
from paper_2605_26975_b200 import plp, solver  # noqa: E402
from plp_inputs import make_config, draw_U, draw_uniforms, permute_graph  # noqa: E402


def main():
    cfg, n, k, sched = sys.argv[1], sys.argv[2], int(sys.argv[3]), [float(x) for x in sys.argv[4].split(",")]
    n = None if n == "None" else int(n)
    order = sys.argv[sys.argv.index("--order") + 1] if "--order" in sys.argv else "tile"
    g = make_config(cfg, n=n)
    if order == "tile":
        g = permute_graph(g, plp.tile_order(g.row_ptr, g.col))
    Z = draw_U(g.n, k, 0)
    u = draw_uniforms(10, k)
    ctx = plp.Context(0)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), sched)
    kern = plp.last_edge_kernel()
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    Uo, tro = osol.continuation_solve(g, Z, sched)
    lab_o, _, sse_o, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    for r in tr.records:
        print(json.dumps({"who": "gpu", "p": r.p, "it": r.it, "F": r.F, "g": r.gradnorm, "delta": r.delta,
                          "tcg": r.tcg_iters, "st": r.tcg_status, "rho": r.rho, "acc": r.accepted}))
    for t in tro:
        print(json.dumps({"who": "orc", "p": t[0], "it": t[1], "F": t[2], "g": t[3], "delta": t[4], "tcg": t[5],
                          "st": t[6], "rho": t[7], "acc": t[8]}))
    a, b = lab.cpu().numpy(), lab_o
    C = np.zeros((k, k), dtype=np.int64)
    np.add.at(C, (a, b), 1)
    mism = int(g.n - C.max(axis=1).sum())
    Uh = U.cpu().numpy()
    # subspace distance between the two solutions (U^T Uo singular values)
    sv = np.linalg.svd(Uh.T @ Uo, compute_uv=False)
    print(json.dumps({"kernel": kern, "rcut_gpu": rc, "rcut_oracle": rc_o, "sse_gpu": sse, "sse_oracle": sse_o,
                      "label_mismatch": mism, "F_gpu": float(oracle.objective(g, Uh, sched[-1])[0]),
                      "F_oracle": float(oracle.objective(g, Uo, sched[-1])[0]),
                      "max_abs_U_diff_colwise": float(np.max(np.abs(np.abs(Uh) - np.abs(Uo)))),
                      "subspace_sv_min": float(sv.min())}))


if __name__ == "__main__":
    main()
