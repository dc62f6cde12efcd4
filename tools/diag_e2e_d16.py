"""D16 end-to-end diagnostic: GPU vs oracle continuation solve and k-means (label mismatch, RCut, stop reasons)."""
import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle
from oracle import solver as osol
from paper_2605_26975_b200 import plp, solver
from plp_inputs import make_config, draw_U, draw_uniforms
ctx = plp.Context(0)
for cfg, n, k, sched in (("D16", 8192, 4, [2.0, 1.5]), ("D16", 4096, 8, [2.0, 1.5])):
    g = make_config(cfg, n=n)
    Z = draw_U(g.n, k, 0); u = draw_uniforms(10, k)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), sched)
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    Uo, tro = osol.continuation_solve(g, Z, sched)
    lab_o, _, _, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    C = np.zeros((k, k), dtype=np.int64); np.add.at(C, (lab.cpu().numpy(), lab_o), 1)
    mis = g.n - C.max(axis=1).sum()
    gr = [r for r in tr.records if r.p == sched[-1]]; o = [t for t in tro if t[0] == sched[-1]]
    print(cfg, n, k, "mismatch", int(mis), "rc", rc, rc_o, "rel", abs(rc - rc_o) / rc_o, "gpu_stop", gr[-1].tcg_status, "oracle_stop", o[-1][6],
          "outer", len(gr), len(o), "kernel", plp.last_edge_kernel(), "maxdiffU", float(np.max(np.abs(np.abs(U.cpu().numpy()) - np.abs(Uo)))), flush=True)
