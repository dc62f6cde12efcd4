"""Tile-ordered D16 end-to-end diagnostic at two max_outer values (GPU vs oracle solve, labels, RCut, stop reasons)."""
import sys, time, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle
from oracle import solver as osol
from paper_2605_26975_b200 import plp, solver
from plp_inputs import make_config, draw_U, draw_uniforms, permute_graph
ctx = plp.Context(0)
for cfg, n, k, sched in (("D16", 8192, 4, [2.0, 1.5]), ("D16", 8192, 8, [2.0, 1.2])):
  g0 = make_config(cfg, n=n); g = permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))
  for mo in (200, 800):
    Z = draw_U(g.n, k, 0); u = draw_uniforms(10, k)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    t0 = time.time()
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), sched, solver.SolverConfig(max_outer=mo))
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    t1 = time.time()
    Uo, tro = osol.continuation_solve(g, Z, sched, max_outer=mo)
    t2 = time.time()
    lab_o, _, _, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    C = np.zeros((k, k), dtype=np.int64); np.add.at(C, (lab.cpu().numpy(), lab_o), 1)
    mis = g.n - C.max(axis=1).sum()
    gr = [r for r in tr.records if r.p == sched[-1]]; o = [t for t in tro if t[0] == sched[-1]]
    print(cfg, k, sched, "max_outer", mo, "mismatch", int(mis), "rc", rc, rc_o, "rel", abs(rc - rc_o) / rc_o, "stop", gr[-1].tcg_status, o[-1][6],
          "outer", len(gr), len(o), "t_gpu", round(t1 - t0, 1), "t_oracle", round(t2 - t1, 1), flush=True)
