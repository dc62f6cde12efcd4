"""Launch a few fused tCG iterations at a config (for ncu launch lists of the NEXT-2 passes).

  python tools/prof_tcg.py [--config C5] [--iters 4] [--unfused]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import get_graph, CONFIG_KP  # noqa: E402
from paper_2605_26975_b200 import plp, solver  # noqa: E402
from plp_inputs import draw_U  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--time", type=int, default=0, help="also time this many reps (CUDA events)")
    a = ap.parse_args()
    k, p = CONFIG_KP[a.config]
    g = get_graph(a.config, "tile")
    ctx = plp.Context(0)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U = plp.retract(ctx, torch.from_numpy(draw_U(g.n, k, 0)).cuda(), torch.zeros(g.n, k, dtype=torch.float64,
                                                                                   device="cuda"))
    cfg = solver.SolverConfig(tcg_kappa=0.0, tcg_max_iters=a.iters)
    tr = solver.GrassmannTR(ctx, G, k, cfg)
    st = solver._State(tr, U, p)
    tr.tcg_device(st, p, 1e6)
    eta, Heta, r, dlt, Hd, scal, status = tr._tcg_buf
    Hacc = Heta if a.unfused else None  # the solver's fused path accumulates no H step
    plp.tcg_init(ctx, st.grad, 1e6, 0.0, 1.0, eta, Hacc, r, dlt, scal, status)
    plp.tcg_run(ctx, G, st.U, st.AB, None, st.S, p, cfg.eps, plp.HESS_SPARSE, eta, Hacc, r, dlt, Hd, scal, status,
                1 << 30, a.iters, fused=not a.unfused)
    torch.cuda.synchronize()
    print("ok", status.cpu().tolist())
    if a.time:
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(a.time):
            plp.tcg_run(ctx, G, st.U, st.AB, None, st.S, p, cfg.eps, plp.HESS_SPARSE, eta, Hacc, r, dlt, Hd,
                        scal, status, 1 << 30, a.iters, fused=not a.unfused)
        s1.record()
        torch.cuda.synchronize()
        print(f"ms_per_iter {s0.elapsed_time(s1) / (a.time * a.iters):.4f}")


if __name__ == "__main__":
    main()
