"""End-to-end p-spectral clustering on a config (GPU solver through libplp, and the oracle solver):
continuation solve, k-means discretisation, RCut; prints a JSON line per arm.

  python tools/solver_e2e.py C2 [n] [--no-oracle]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from plp_inputs import make_config, draw_U, draw_uniforms  # noqa: E402

SCHED = {"C1": [2.0, 1.8, 1.5, 1.2], "C2": [2.0, 1.1], "C4": [2.0, 1.2]}
K = {"C1": 3, "C2": 2, "C4": 20}


def main():
    cfg = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else None
    g = make_config(cfg, n=n)
    k = K[cfg]
    Z = draw_U(g.n, k, 0)
    u = draw_uniforms(10, k)
    from paper_2605_26975_b200 import plp, solver
    ctx = plp.Context(0)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    t = time.time()
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), SCHED[cfg])
    torch.cuda.synchronize()
    t_solve = time.time() - t
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    out = {"arm": "gpu", "cfg": cfg, "n": g.n, "nnz": g.nnz, "solve_s": t_solve, "outer": len(tr.records),
           "tcg": sum(r.tcg_iters for r in tr.records), "F_final": tr.records[-1].F, "rcut": rc, "sse": sse}
    print(json.dumps(out), flush=True)
    np.save(os.path.join(ROOT, "gpurun_out", f"e2e_{cfg}_gpu_labels.npy"), lab.cpu().numpy())
    if "--no-oracle" in sys.argv:
        return
    import oracle
    from oracle import solver as osol
    t = time.time()
    Uo, tro = osol.continuation_solve(g, Z, SCHED[cfg])
    t_o = time.time() - t
    lab_o, _, sse_o, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    out = {"arm": "oracle", "cfg": cfg, "n": g.n, "solve_s": t_o, "outer": len(tro),
           "tcg": sum(r[5] for r in tro), "F_final": tro[-1][2], "rcut": rc_o, "sse": sse_o}
    print(json.dumps(out), flush=True)
    lg = lab.cpu().numpy()
    C = np.zeros((k, k), dtype=np.int64)
    np.add.at(C, (lg, lab_o), 1)
    perm_ok = bool(np.all((C > 0).sum(axis=1) == 1) and np.all((C > 0).sum(axis=0) == 1))
    print(json.dumps({"labels_equal_up_to_permutation": perm_ok,
                      "rcut_rel": abs(rc - rc_o) / max(abs(rc_o), 1e-300)}), flush=True)


if __name__ == "__main__":
    main()
