"""Tiny invocations of every kernel family for compute-sanitizer (race / sync /
memory checking of the warp-specialised mbarrier + TMA edge kernel, the ticketed tCG reductions,
k-means and the dense kernels).

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py [halo|staged|rows|tcg|dense|kmeans|all]
Sizes are small (a few tiles / CTAs) so that the sanitizers finish in seconds; each case checks
its result against the oracle so a run that "passes" the tool also computed the right thing.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2605_26975_b200 import plp, solver  # noqa: E402
from plp_inputs import make_config, permute_graph, draw_U, draw_eta, draw_uniforms  # noqa: E402


def rel(x, r):
    return float(np.max(np.abs(x - r)) / max(np.max(np.abs(r)), 1e-300))


def edge_case(ctx, k=8, p=1.2, n=3000):
    g0 = make_config("C5", n=n)
    g = permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U = draw_U(g.n, k, 1)
    eta = draw_eta(g.n, k, 1)
    Ut, Et = torch.from_numpy(U).cuda(), torch.from_numpy(eta).cuda()
    F0, AB, Gr0 = plp.fgrad(ctx, G, Ut, p)
    Hv0 = plp.hessvec(ctx, G, Ut, Et, p, AB)
    F, ABo, Gr, Hv = plp.fgrad_hessvec(ctx, G, Ut, Et, p, AB_in=AB)
    torch.cuda.synchronize()
    Fo, A, B, Gro, Hvo = oracle.fgrad_hessvec(g, U, eta, p)
    errs = (rel(Gr.cpu().numpy(), Gro), rel(Hv.cpu().numpy(), Hvo), rel(Hv0.cpu().numpy(), Hvo),
            rel(Gr0.cpu().numpy(), Gro))
    assert max(errs) < 1e-9, errs
    return f"{plp.last_edge_kernel()} errs {max(errs):.1e}"


def tcg_case(ctx):
    g = make_config("C2", n=2000)
    k = 8
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    Uo, _ = oracle.retract(draw_U(g.n, k, 5), np.zeros((g.n, k)))
    out = []
    for fused in (True, False):
        tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(tcg_fused=fused, tcg_graph=False))
        st = solver._State(tr, torch.from_numpy(Uo).cuda(), 1.5)
        eta, Heta, it, status = tr.tcg_device(st, 1.5, 0.3)
        out.append((it, status))
    return f"tcg fused/unfused {out}"


def dense_case(ctx):
    n, k = 5003, 8
    rng = np.random.default_rng(0)
    U = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, k)))[0]).cuda()
    X = torch.from_numpy(rng.standard_normal((n, k))).cuda()
    P = plp.project(ctx, U, X)
    Q = plp.retract(ctx, U, 0.1 * X)
    d = plp.dot(ctx, U, X)
    torch.cuda.synchronize()
    assert rel(P.cpu().numpy(), oracle.project(U.cpu().numpy(), X.cpu().numpy())) < 1e-9
    return f"dense ok (dot {d.item():.3e}, |Q| {Q.norm().item():.3f})"


def kmeans_case(ctx):
    rng = np.random.default_rng(1)
    X = rng.standard_normal((3000, 4))
    u = draw_uniforms(3, 4)
    lab, C, sse, _ = plp.kmeans(ctx, torch.from_numpy(X).cuda(), 4, u, restarts=3)
    lab_o, _, sse_o, _ = oracle.kmeans(X, 4, u, restarts=3)
    assert np.array_equal(lab.cpu().numpy(), lab_o)
    return f"kmeans ok sse {sse:.6g}"


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    ctx = plp.Context(0)
    if which in ("halo", "all"):
        print("halo:", edge_case(ctx), flush=True)
        print("halo k=4:", edge_case(ctx, k=4, p=1.5), flush=True)
    if which in ("staged", "rows"):  # env PLP_EDGE_STAGED / PLP_EDGE_ROWS selects the kernel
        print(which + ":", edge_case(ctx), flush=True)
    if which in ("tcg", "all"):
        print(tcg_case(ctx), flush=True)
    if which in ("dense", "all"):
        print(dense_case(ctx), flush=True)
    if which in ("kmeans", "all"):
        print(kmeans_case(ctx), flush=True)


if __name__ == "__main__":
    main()
