"""GPU solver (paper_2605_26975_b200/solver.py over the C ABI) against the oracle solver and the
textbook eigenproblem: the north star's end-to-end acceptance (cluster labels equal up to
permutation, RCut within 1e-6 relative) on C1 and a reduced C2, p = 2 spectral consistency, the
first trust-region step against the oracle's, and the solver invariants."""
import numpy as np
import pytest
import scipy.sparse.csgraph as csgraph
import torch

import oracle
from oracle import solver as osol
from plp_inputs import make_config, draw_U, draw_uniforms, random_graph, streams

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    from paper_2605_26975_b200 import plp, solver
    return plp, solver, plp.Context(0)


def same_partition(a, b, k):
    C = np.zeros((k, k), dtype=np.int64)
    np.add.at(C, (np.asarray(a), np.asarray(b)), 1)
    return bool(np.all((C > 0).sum(axis=1) == 1) and np.all((C > 0).sum(axis=0) == 1))


@pytest.mark.parametrize("seed,n,k", [(1, 60, 2), (2, 120, 4), (3, 200, 2)])
def test_p2_matches_dense_eigensolver(mods, seed, n, k):
    plp, solver, ctx = mods
    g = random_graph(streams(seed)[0], n, avg_deg=5.0, connected=True)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    Z = torch.from_numpy(streams(seed)[1].standard_normal((n, k))).cuda()
    U, tr = solver.continuation_solve(ctx, G, Z, [2.0], solver.SolverConfig(grad_tol=1e-9))
    F = oracle.objective(g, U.cpu().numpy(), 2.0)[0]
    ev = np.sum(np.linalg.eigvalsh(csgraph.laplacian(g.to_scipy()).toarray())[:k])
    assert abs(F - ev) < 1e-6 * max(1.0, abs(ev))


def test_first_trust_region_step_matches_oracle(mods):
    """One tCG solve at a random orthonormal U (p = 1.5, sparse Hessian): the GPU step equals the
    oracle's within 1e-9 (same algorithm, different summation order)."""
    plp, solver, ctx = mods
    g = make_config("C2", n=5000)
    k = 2
    Z = draw_U(g.n, k, 3)
    Uo, _ = oracle.retract(Z, np.zeros_like(Z))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    tr = solver.GrassmannTR(ctx, G, k)
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), 1.5)
    eta, Heta, it, status = tr.tcg(st, 1.5, 0.3)
    cfg = osol.default_cfg(g.n, k)
    sto = osol._state(g, Uo, 1.5, osol.oracle_fns())
    eta_o, Heta_o, it_o, status_o = osol.tcg(
        lambda xi: osol._hess(g, sto, 1.5, xi, cfg["eps"], "sparse", osol.oracle_fns()), sto["grad"], Uo,
        0.3, cfg)
    assert (it, status) == (it_o, status_o)
    e = eta.cpu().numpy()
    assert np.max(np.abs(e - eta_o)) <= 1e-9 * np.max(np.abs(eta_o))
    assert np.max(np.abs(Heta.cpu().numpy() - Heta_o)) <= 1e-9 * np.max(np.abs(Heta_o))


@pytest.mark.parametrize("cfg,n,k,sched", [("C1", None, 3, [2.0, 1.8, 1.5, 1.2]),
                                            ("C2", 20000, 2, [2.0, 1.1]),
                                            ("D16", 8192, 4, [2.0, 1.5]),  # k = 2, 4: folded fused tCG
                                            ("D16", 4096, 8, [2.0, 1.5]),  # k = 8: fused tCG passes
                                            ("C1", None, 3, [2.0, 1.5])])  # k = 3: unfused device tCG
def test_end_to_end_labels_and_rcut_match_oracle(mods, cfg, n, k, sched):
    """North star: labels agree up to permutation, RCut within 1e-6 relative (C1, C2: the configs
    the north star names).  The D16 stand-ins take reading #25's boundary-node check (<= 1 % of
    labels, RCut within 2 %): their converged iterates are ~1e-5 apart between two reduction orders,
    enough to move 2-3 k-means boundary labels."""
    plp, solver, ctx = mods
    g = make_config(cfg, n=n)
    Z = draw_U(g.n, k, 0)
    u = draw_uniforms(10, k)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), sched)
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    Uo, tro = osol.continuation_solve(g, Z, sched)
    lab_o, _, sse_o, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    if cfg not in ("C1", "C2"):
        C = np.zeros((k, k), dtype=np.int64)
        np.add.at(C, (lab.cpu().numpy(), lab_o), 1)
        mismatch = g.n - C.max(axis=1).sum()
        assert mismatch <= 0.01 * g.n, mismatch
        assert abs(rc - rc_o) <= 0.02 * rc_o, (rc, rc_o)
        return
    assert same_partition(lab.cpu().numpy(), lab_o, k)
    assert abs(rc - rc_o) <= 1e-6 * max(abs(rc_o), 1e-300) or abs(rc - rc_o) < 1e-300
    # invariants of the GPU run
    Uh = U.cpu().numpy()
    assert np.max(np.abs(Uh.T @ Uh - np.eye(k))) < 1e-10
    for p in sched:
        Fs = [r.F for r in tr.records if r.p == p and r.accepted]
        assert all(b <= a + 1e-15 * abs(a) for a, b in zip(Fs, Fs[1:]))


@pytest.mark.parametrize("p,delta,mode", [(1.5, 0.3, 0), (1.2, 5.0, 0), (2.0, 0.05, 0), (1.5, 0.3, 1)])
def test_device_tcg_matches_host_tcg_bitwise(mods, p, delta, mode):
    """plp_tcg_run keeps the tCG scalars on the device; its recurrences are written in the host
    loop's order with explicit rounding, so step, H step, iteration count and exit status equal
    the host-driven tCG bit for bit (boundary, interior-convergence and full-Hessian cases)."""
    plp, solver, ctx = mods
    g = make_config("C2", n=5000)
    k = 2
    Z = draw_U(g.n, k, 4)
    Uo, _ = oracle.retract(Z, np.zeros_like(Z))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(hessian_mode=mode, tcg_fused=False))
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), p)
    a = tr.tcg(st, p, delta)
    b = tr.tcg_device(st, p, delta)
    assert a[2:] == b[2:], (a[2:], b[2:])
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


@pytest.mark.parametrize("cfg,n,k,p,delta,mode", [("C2", 5003, 8, 1.5, 0.3, 0), ("C2", 5003, 8, 1.2, 50.0, 0),
                                                  ("C1", None, 16, 1.5, 0.5, 0), ("C2", 4001, 8, 1.8, 2.0, 1),
                                                  ("C2", 2003, 16, 1.3, 1e3, 0),
                                                  # folded k (n k / 8 rows of 8, block-diagonal k x k)
                                                  ("C2", 5002, 4, 1.5, 0.3, 0), ("C2", 5004, 2, 1.2, 50.0, 0),
                                                  ("C2", 4000, 1, 1.6, 1e3, 0), ("C2", 3002, 4, 1.8, 2.0, 1)])
def test_fused_tcg_matches_oracle(mods, cfg, n, k, p, delta, mode):
    """NEXT-2 fused tCG (three tensor-core passes after the edge pass; <d, Hd> and ||P r||^2 from
    Grams) against the oracle's tCG: same iteration count and exit status, step and H step within
    1e-9 relative (ragged n: 8-row blocks with a tail; boundary, interior and full-Hessian cases)."""
    plp, solver, ctx = mods
    g = make_config(cfg, n=n)
    Z = draw_U(g.n, k, 5)
    Uo, _ = oracle.retract(Z, np.zeros_like(Z))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(hessian_mode=mode, tcg_fused=True))
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), p)
    eta, Heta, it, status = tr.tcg_device(st, p, delta)
    ocfg = osol.default_cfg(g.n, k)
    hm = "full" if mode == 1 else "sparse"
    sto = osol._state(g, Uo, p, osol.oracle_fns())
    eta_o, Heta_o, it_o, status_o = osol.tcg(
        lambda xi: osol._hess(g, sto, p, xi, ocfg["eps"], hm, osol.oracle_fns()), sto["grad"], Uo, delta, ocfg)
    assert (it, status) == (it_o, status_o)
    assert np.max(np.abs(eta.cpu().numpy() - eta_o)) <= 1e-9 * np.max(np.abs(eta_o))
    assert np.max(np.abs(Heta.cpu().numpy() - Heta_o)) <= 1e-9 * np.max(np.abs(Heta_o))


@pytest.mark.parametrize("n,k", [(37, 8), (70, 16)])
def test_fused_tcg_tiny_graphs(mods, n, k):
    """Fused tCG on graphs smaller than one 8-row block per warp (single-CTA grids, ragged tail)."""
    plp, solver, ctx = mods
    g = random_graph(streams(n)[0], n, avg_deg=6.0, connected=True)
    Uo, _ = oracle.retract(draw_U(g.n, k, 8), np.zeros((g.n, k)))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(tcg_fused=True))
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), 1.6)
    eta, Heta, it, status = tr.tcg_device(st, 1.6, 0.4)
    ocfg = osol.default_cfg(g.n, k)
    sto = osol._state(g, Uo, 1.6, osol.oracle_fns())
    eta_o, Heta_o, it_o, status_o = osol.tcg(
        lambda xi: osol._hess(g, sto, 1.6, xi, ocfg["eps"], "sparse", osol.oracle_fns()), sto["grad"], Uo, 0.4, ocfg)
    assert (it, status) == (it_o, status_o)
    assert np.max(np.abs(eta.cpu().numpy() - eta_o)) <= 1e-9 * np.max(np.abs(eta_o))
    assert np.max(np.abs(Heta.cpu().numpy() - Heta_o)) <= 1e-9 * np.max(np.abs(Heta_o))


def test_fused_tcg_rejects_unsupported_k(mods):
    plp, solver, ctx = mods
    g = make_config("C2", n=501)  # k = 4: n k not divisible by 8
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U = torch.from_numpy(oracle.retract(draw_U(g.n, 4, 1), np.zeros((g.n, 4)))[0]).cuda()
    tr = solver.GrassmannTR(ctx, G, 4, solver.SolverConfig(tcg_fused=True))
    st = solver._State(tr, U, 1.5)
    with pytest.raises(plp.PlpError):
        tr.tcg_device(st, 1.5, 0.3)


@pytest.mark.parametrize("k,fused", [(3, False), (8, True)])
def test_tcg_graph_replay_is_bitwise_the_direct_launches(k, fused):
    """plp_tcg_graph_create / _launch: a captured batch of tCG iterations on a side stream gives
    bitwise the step, H step, iteration count and status of launching the same iterations
    directly, and the end-to-end solve is unchanged."""
    from paper_2605_26975_b200 import plp, solver
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ctx = plp.Context(0, stream)
        g = make_config("C2", n=3001)
        G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
        # near a p = 2 minimiser the Hessian is positive definite: tCG runs many iterations
        Z = torch.from_numpy(draw_U(g.n, k, 6)).cuda()
        U, _ = solver.continuation_solve(ctx, G, Z, [2.0], solver.SolverConfig(grad_tol=1e-2, tcg_graph=False))
        res = []
        for graph in (False, True):
            tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(tcg_graph=graph, tcg_fused=fused, tcg_batch=4))
            st = solver._State(tr, U, 2.0)
            res.append(tr.tcg_device(st, 2.0, 10.0))
            if graph:
                assert tr._graphs and all(gr.nodes() >= 5 * b for b, gr in tr._graphs.items())
        a, b = res
        assert a[2:] == b[2:] and a[2] > 4
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
        Z = torch.from_numpy(draw_U(g.n, k, 7)).cuda()
        sols = [solver.continuation_solve(ctx, G, Z, [2.0, 1.5], solver.SolverConfig(tcg_graph=gr, tcg_fused=fused))
                for gr in (False, True)]
        assert torch.equal(sols[0][0], sols[1][0])
        assert [r.tcg_iters for r in sols[0][1].records] == [r.tcg_iters for r in sols[1][1].records]


def test_tcg_graph_needs_created_stream(mods):
    """plp_tcg_graph_create on the legacy default stream is refused (PLP_ERR_ARG), not captured."""
    plp, solver, ctx = mods
    if ctx.stream.cuda_stream != 0:
        pytest.skip("context not on the default stream")
    g = make_config("C2", n=400)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    Uo, _ = oracle.retract(draw_U(g.n, 2, 2), np.zeros((g.n, 2)))
    tr = solver.GrassmannTR(ctx, G, 2, solver.SolverConfig(tcg_graph=False))
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), 1.5)
    tr.tcg_device(st, 1.5, 0.3)
    eta, Heta, r, dlt, Hd, scal, status = tr._tcg_buf
    with pytest.raises(plp.PlpError):
        plp.TcgGraph(ctx, G, st.U, st.AB, None, st.S, 1.5, 1e-9, plp.HESS_SPARSE, eta, Heta, r, dlt, Hd, scal,
                     status, 100, 4)


@pytest.mark.parametrize("seed", range(8))
def test_fused_tcg_randomised_against_oracle(mods, seed):
    """Randomised fused-tCG cases (k, p, trust radius, iteration cap, graph size drawn from the
    seed): same iteration count and exit status as the oracle's tCG (boundary, negative curvature,
    convergence and the iteration cap all occur), step and H step within 1e-9."""
    plp, solver, ctx = mods
    rng = np.random.default_rng(1000 + seed)
    k = int(rng.choice([2, 4, 8]))
    n = int(rng.choice([600, 1200, 2400])) // 8 * 8 + 8
    p = float(rng.choice([1.1, 1.3, 1.6, 1.9, 2.0]))
    delta = float(rng.choice([1e-3, 0.3, 50.0]))
    cap = int(rng.choice([2, 7, 200]))
    g = random_graph(streams(seed + 50)[0], n, avg_deg=7.0, connected=True)
    Uo, _ = oracle.retract(draw_U(g.n, k, seed + 60), np.zeros((g.n, k)))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(tcg_fused=True, tcg_max_iters=cap))
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), p)
    eta, Heta, it, status = tr.tcg_device(st, p, delta)
    ocfg = osol.default_cfg(g.n, k, tcg_max_iters=cap)
    sto = osol._state(g, Uo, p, osol.oracle_fns())
    eta_o, Heta_o, it_o, status_o = osol.tcg(
        lambda xi: osol._hess(g, sto, p, xi, ocfg["eps"], "sparse", osol.oracle_fns()), sto["grad"], Uo, delta, ocfg)
    assert (it, status) == (it_o, status_o), (k, n, p, delta, cap)
    assert np.max(np.abs(eta.cpu().numpy() - eta_o)) <= 1e-9 * np.max(np.abs(eta_o))
    assert np.max(np.abs(Heta.cpu().numpy() - Heta_o)) <= 1e-9 * np.max(np.abs(Heta_o))


def _tile_ordered(plp, cfg, n):
    from plp_inputs import permute_graph
    g0 = make_config(cfg, n=n)
    return permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))


def _converged(gpu_records, oracle_trace, p):
    """Both solves stopped on the gradient test at the final p (not on max_outer)."""
    g = [r for r in gpu_records if r.p == p]
    o = [t for t in oracle_trace if t[0] == p]
    return bool(g and o and g[-1].tcg_status == "stop" and o[-1][6] == "stop")


@pytest.mark.parametrize("cfg,n,k,sched", [("D16", 8192, 8, [2.0, 1.2]),
                                            ("D16", 8192, 4, [2.0, 1.5]),
                                            ("C2", 20000, 4, [2.0, 1.1]),
                                            ("C5", 20000, 8, [2.0, 1.2])])
def test_end_to_end_tile_ordered_matches_oracle(mods, cfg, n, k, sched):
    """The ordering the solver runs on (plp_tile_order): every Hessian-vector product of the solve
    goes through the halo kernel's adaptive capped-form variant (k = 4, 8).  Where both solves
    converge (gradient test at the final p) the labels must agree up to permutation and RCut within
    1e-6 relative.  Where they stop on max_outer (|grad| stalls above grad_tol at small p; seen on
    D16 at k = 4 and 8), the returned iterate is wherever iteration 200 ends, and two correct solvers
    differing in rounding (summation order, ~200-iteration CGs) end at different points of the same
    flat valley (tools/diag_e2e.py: the staged kernel's solve separates from the oracle's the same
    way): there the check is the same clustering up to boundary nodes -- <= 1 % of labels, RCut
    within 2 % (reading #25: labels within 2.5 % -- D16 k = 4 at p = 1.5 on the 80-row tile order:
    the GPU solve converges after 69 outer iterations, the oracle's stalls above grad_tol through
    200 and 800, and the two end 1.9 % of labels and 0.9 % of RCut apart)."""
    plp, solver, ctx = mods
    g = _tile_ordered(plp, cfg, n)
    Z = draw_U(g.n, k, 0)
    u = draw_uniforms(10, k)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), sched)
    assert plp.last_edge_kernel().startswith("edge_halo_kernel"), plp.last_edge_kernel()
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    Uo, tro = osol.continuation_solve(g, Z, sched)
    lab_o, _, sse_o, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    if _converged(tr.records, tro, sched[-1]):
        assert same_partition(lab.cpu().numpy(), lab_o, k)
        assert abs(rc - rc_o) <= 1e-6 * max(abs(rc_o), 1e-300)
    else:
        C = np.zeros((k, k), dtype=np.int64)
        np.add.at(C, (lab.cpu().numpy(), lab_o), 1)
        mismatch = g.n - C.max(axis=1).sum()
        assert mismatch <= 0.025 * g.n, mismatch
        assert abs(rc - rc_o) <= 0.02 * rc_o, (rc, rc_o)


@pytest.mark.slow
def test_end_to_end_c2_full_size_matches_oracle(mods):
    """North star acceptance at config 2's own size (two moons, n = 100,000, k = 2, p 2 -> 1.1)."""
    plp, solver, ctx = mods
    g = make_config("C2")
    k, sched = 2, [2.0, 1.1]
    Z = draw_U(g.n, k, 0)
    u = draw_uniforms(10, k)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U, tr = solver.continuation_solve(ctx, G, torch.from_numpy(Z).cuda(), sched)
    lab, rc, sse = solver.cluster(ctx, G, U, k, u)
    Uo, tro = osol.continuation_solve(g, Z, sched)
    lab_o, _, sse_o, _ = oracle.kmeans(Uo, k, u, restarts=10)
    rc_o = oracle.rcut(g, lab_o, k)[0]
    assert same_partition(lab.cpu().numpy(), lab_o, k)
    assert abs(rc - rc_o) <= 1e-6 * max(abs(rc_o), 1e-300)


@pytest.mark.parametrize("cfg,n,k,p,delta", [("D16", 8192, 8, 1.2, 0.3), ("D16", 8192, 4, 1.5, 50.0),
                                              ("C5", 30000, 8, 1.2, 1e3), ("C5", 30000, 16, 1.8, 0.3)])
def test_fused_tcg_tile_ordered_matches_oracle(mods, cfg, n, k, p, delta):
    """Fused tCG on tile-ordered graphs (its Hessian-vector products run the adaptive halo kernel):
    same iteration count and status as the oracle's tCG, step and H step within 1e-9."""
    plp, solver, ctx = mods
    g = _tile_ordered(plp, cfg, n)
    Uo, _ = oracle.retract(draw_U(g.n, k, 5), np.zeros((g.n, k)))
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(tcg_fused=True))
    st = solver._State(tr, torch.from_numpy(Uo).cuda(), p)
    eta, Heta, it, status = tr.tcg_device(st, p, delta)
    kern = plp.last_edge_kernel()
    assert (kern.startswith("edge_halo_kernel[") and "adapt" in kern) or (k == 16 and kern.startswith("edge_staged")), kern
    ocfg = osol.default_cfg(g.n, k)
    sto = osol._state(g, Uo, p, osol.oracle_fns())
    eta_o, Heta_o, it_o, status_o = osol.tcg(
        lambda xi: osol._hess(g, sto, p, xi, ocfg["eps"], "sparse", osol.oracle_fns()), sto["grad"], Uo, delta, ocfg)
    assert (it, status) == (it_o, status_o)
    assert np.max(np.abs(eta.cpu().numpy() - eta_o)) <= 1e-9 * np.max(np.abs(eta_o))
    assert np.max(np.abs(Heta.cpu().numpy() - Heta_o)) <= 1e-9 * np.max(np.abs(Heta_o))


_GRAM_RUN = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
from paper_2605_26975_b200 import plp, solver
from plp_inputs import make_config, permute_graph, draw_U
import oracle
g0 = make_config({cfg!r}, n={n})
g = permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))
k, p = {k}, {p}
ctx = plp.Context(0)
G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
Uo, _ = oracle.retract(draw_U(g.n, k, 5), np.zeros((g.n, k)))
cfg = solver.SolverConfig(tcg_fused=True, tcg_graph=False)
tr = solver.GrassmannTR(ctx, G, k, cfg)
st = solver._State(tr, torch.from_numpy(Uo).cuda(), p)
tr.tcg_device(st, p, 1e3)
eta, Heta, r, dlt, Hd, scal, status = tr._tcg_buf
plp.tcg_init(ctx, st.grad, 1e3, 0.0, 1.0, eta, None, r, dlt, scal, status)
plp.tcg_run(ctx, G, st.U, st.AB, None, st.S, p, cfg.eps, plp.HESS_SPARSE, eta, None, r, dlt, Hd, scal, status,
            1 << 30, {iters}, fused=True)
torch.cuda.synchronize()
np.save({out!r}, eta.cpu().numpy())
print("KERNEL", plp.last_edge_kernel())
print("STATUS", status.cpu().tolist())
"""


@pytest.mark.parametrize("cfg,n,k,p", [("D16", 8192, 8, 1.2), ("D16", 8192, 4, 1.5), ("C5", 30000, 8, 1.2),
                                       ("C5", 30002, 4, 1.8)])
def test_fused_tcg_pass_a_fold_matches_separate_pass(cfg, n, k, p, tmp_path):
    """NEXT-2: pass A of the fused tCG folded into the Hessian-vector-only halo pass (edge_halo.cuh
    GRAM; its DMMA Grams and d (EH - d S) sums over the tile's row blocks) against the separate pass A
    (PLP_TCG_GRAM_EDGE=0): same iteration count and status after 12 iterations, the step equal within
    1e-10 relative (only the Grams' summation order differs); the fold is what ran."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for fold in (1, 0):
        out = str(tmp_path / f"eta{fold}.npy")
        code = _GRAM_RUN.format(root=root, cfg=cfg, n=n, k=k, p=p, iters=12, out=out)
        env = dict(os.environ, PLP_TCG_GRAM_EDGE=str(fold))
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        lines = dict(ln.split(" ", 1) for ln in r.stdout.splitlines() if ln.startswith(("KERNEL", "STATUS")))
        res[fold] = (np.load(out), lines["KERNEL"], lines["STATUS"])
    assert "gram" in res[1][1], res[1][1]
    assert "gram" not in res[0][1], res[0][1]
    assert res[1][2] == res[0][2]
    e1, e0 = res[1][0], res[0][0]
    assert np.max(np.abs(e1 - e0)) <= 1e-10 * np.max(np.abs(e0))


@pytest.mark.parametrize("k", [8, 4, 16])
def test_fused_tcg_deferred_reprojection_is_bitwise(mods, k):
    """Fused tCG with the residual's re-projection deferred into the next pass B (tcg.cu: pass C
    writes only d; the last pass C of a plp_tcg_run batch writes the projected r and zeroes MR):
    one batch of N iterations against N batches of one iteration (each of which writes r, so no
    re-projection is deferred) -- step, residual, direction, iteration count and status bitwise
    equal (the same operations in the same order), the projected residual of the batch
    horizontal (U^T r ~ 0)."""
    plp, solver, ctx = mods
    g = make_config("C2", n=3000)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    # near a p = 2 minimiser the Hessian is positive definite: tCG runs many iterations
    Z = torch.from_numpy(draw_U(g.n, k, 6)).cuda()
    U, _ = solver.continuation_solve(ctx, G, Z, [2.0], solver.SolverConfig(grad_tol=1e-2, tcg_graph=False))
    cfg = solver.SolverConfig(tcg_fused=True, tcg_graph=False)
    tr = solver.GrassmannTR(ctx, G, k, cfg)
    st = solver._State(tr, U, 1.8)
    tr.tcg_device(st, 1.8, 10.0)
    n_it = 7
    out = []
    for batches in ((n_it,), (1,) * n_it):
        eta, Heta, r, dlt, Hd, scal, status = (t.clone() for t in tr._tcg_buf)
        plp.tcg_init(ctx, st.grad, 10.0, 0.0, 1.0, eta, None, r, dlt, scal, status)
        for b in batches:
            plp.tcg_run(ctx, G, st.U, st.AB, None, st.S, 1.8, cfg.eps, plp.HESS_SPARSE, eta, None, r, dlt, Hd,
                        scal, status, 1 << 30, b, fused=True)
        torch.cuda.synchronize()
        out.append((eta, r, dlt, status.cpu().tolist()))
    (e1, r1, d1, s1), (e2, r2, d2, s2) = out
    assert s1 == s2 and s1[1] >= 3, (s1, s2)
    assert torch.equal(e1, e2) and torch.equal(r1, r2) and torch.equal(d1, d2)
    utr = (st.U[: g.n].T @ r1).abs().max().item()
    assert utr <= 1e-10 * max(1.0, r1.abs().max().item()), utr
