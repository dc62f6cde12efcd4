"""The collective C ABI on one GPU ("on P ranks each call is collective"): a
context holding a one-rank NCCL communicator (plp_ctx_create with an id from
plp_get_nccl_unique_id) and a graph from plp_create_graph_dist run the multi-rank code path --
halo exchange (no peers at world = 1), in-library all-reduce of A, B, dots, Grams and dots, F from
the reduced A, B -- and must give bitwise the single-GPU results.  The multi-rank exchange logic is
covered by the gloo tests (tests/test_dist_gloo.py) on CPU."""
import numpy as np
import pytest
import torch

import oracle
from plp_inputs import make_config, draw_U, draw_eta, draw_uniforms, permute_graph
from helpers import TOL, colwise_relerr, scalar_relerr, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plp():
    from paper_2605_26975_b200 import plp as mod
    return mod


@pytest.fixture(scope="module")
def ctxs(plp):
    plain = plp.Context(0)
    coll = plp.Context(0, rank=0, world=1, nccl_id=plp.get_nccl_unique_id())
    return plain, coll


@pytest.fixture(scope="module")
def graph(plp):
    g0 = make_config("C5", n=60_000)
    return permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))


def test_comm_info(plp, ctxs):
    plain, coll = ctxs
    assert plain.comm_info() == (0, 1, False)
    assert coll.comm_info() == (0, 1, True)


def test_world_gt_one_needs_id(plp):
    with pytest.raises(plp.PlpError, match="PLP_ERR_ARG"):
        plp.Context(0, rank=0, world=2, nccl_id=None)


@pytest.mark.parametrize("k,p,mode", [(8, 1.2, 0), (4, 1.5, 1), (3, 1.8, 0), (8, 2.0, 1)])
def test_edge_calls_bitwise_equal_to_single_gpu(plp, ctxs, graph, k, p, mode):
    plain, coll = ctxs
    g = graph
    Gp = plp.Graph(plain, g.row_ptr, g.col, g.w)
    Gc = plp.DistGraph(coll, g.n, 0, g.n, g.row_ptr, g.col, g.w)
    assert Gc.n_halo == 0 and Gc.send_rows == 0 and Gc.n_cols == g.n
    U = torch.from_numpy(draw_U(g.n, k, 2)).cuda()
    eta = torch.from_numpy(draw_eta(g.n, k, 2)).cuda()
    res = []
    for ctx, G in ((plain, Gp), (coll, Gc)):
        F0, AB, Gr = plp.fgrad(ctx, G, U, p)
        Hv = plp.hessvec(ctx, G, U, eta, p, AB, mode=mode, G_in=Gr)
        Hv2 = plp.hessvec(ctx, G, U, eta, p, AB, mode=mode | plp.U_HALO_CURRENT, G_in=Gr)
        F, ABo, G2, Hv3 = plp.fgrad_hessvec(ctx, G, U, eta, p, AB_in=AB, mode=mode)
        Fn, ABn, G3, Hv4 = plp.fgrad_hessvec(ctx, G, U, eta, p, AB_in=None, mode=mode)
        torch.cuda.synchronize()
        res.append([F0, AB, Gr, Hv, Hv2, F, ABo, G2, Hv3, Fn, ABn, G3, Hv4])
    for a, b in zip(*res):
        assert torch.equal(a, b)
    # and the collective results are the oracle's
    F, A, B, Gro, Hvo = oracle.fgrad_hessvec(g, U.cpu().numpy(), eta.cpu().numpy(), p, 1e-9,
                                             "full" if mode else "sparse")
    assert scalar_relerr(to_np(res[1][5])[0], F) < TOL
    assert colwise_relerr(to_np(res[1][7]), Gro) < TOL and colwise_relerr(to_np(res[1][8]), Hvo) < TOL


def test_dense_calls_bitwise_equal_to_single_gpu(plp, ctxs):
    plain, coll = ctxs
    n, k = 50_001, 8
    rng = np.random.default_rng(3)
    U = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, k)))[0]).cuda()
    X = torch.from_numpy(rng.standard_normal((n, k))).cuda()
    out = []
    for ctx in (plain, coll):
        out.append([plp.gram(ctx, U, X), plp.project(ctx, U, X), plp.retract(ctx, U, 0.1 * X),
                    plp.dot(ctx, U, X)])
    torch.cuda.synchronize()
    for a, b in zip(*out):
        assert torch.equal(a, b)


def test_rcut_and_allreduce(plp, ctxs, graph):
    plain, coll = ctxs
    g = graph
    k = 5
    lab = torch.from_numpy((np.arange(g.n) * 7 // g.n % k).astype(np.int32)).cuda()
    Gp = plp.Graph(plain, g.row_ptr, g.col, g.w)
    Gc = plp.DistGraph(coll, g.n, 0, g.n, g.row_ptr, g.col, g.w)
    a = plp.rcut(plain, Gp, k, lab)
    b = plp.rcut(coll, Gc, k, lab)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    rc_o = oracle.rcut(g, lab.cpu().numpy(), k)[0]
    assert abs(float(b[0].item()) - rc_o) <= 1e-12 * rc_o
    x = torch.arange(10, dtype=torch.float64, device="cuda")
    y = x.clone()
    plp.allreduce_sum(coll, y)
    torch.cuda.synchronize()
    assert torch.equal(x, y)


def test_device_tcg_on_collective_context(plp, ctxs):
    """The unfused device tCG calls the collective entry points (plp_hessvec, plp_project, plp_dot):
    on the one-rank communicator it gives bitwise the plain context's iterates."""
    from paper_2605_26975_b200 import solver
    plain, coll = ctxs
    g = make_config("C2", n=4000)
    k = 2
    Z = torch.from_numpy(draw_U(g.n, k, 4)).cuda()
    outs = []
    for ctx, mk in ((plain, lambda c: plp.Graph(c, g.row_ptr, g.col, g.w)),
                    (coll, lambda c: plp.DistGraph(c, g.n, 0, g.n, g.row_ptr, g.col, g.w))):
        G = mk(ctx)
        with torch.cuda.stream(ctx.stream):
            U, tr = solver.continuation_solve(ctx, G, Z, [2.0, 1.5],
                                              solver.SolverConfig(tcg_fused=False, tcg_graph=False))
        outs.append((U, [r.tcg_iters for r in tr.records]))
    assert outs[0][1] == outs[1][1]
    assert torch.equal(outs[0][0], outs[1][0])


_SPLIT_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from paper_2605_26975_b200 import plp
from plp_inputs import make_config, draw_U, draw_eta, permute_graph
g0 = make_config("C5", n=60_000)
g = permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))
plain = plp.Context(0)
coll = plp.Context(0, rank=0, world=1, nccl_id=plp.get_nccl_unique_id())
out = {{}}
for k, p, mode in ((8, 1.2, 0), (4, 1.5, 1)):
    U = torch.from_numpy(draw_U(g.n, k, 2)).cuda()
    eta = torch.from_numpy(draw_eta(g.n, k, 2)).cuda()
    Gp = plp.Graph(plain, g.row_ptr, g.col, g.w)
    Gc = plp.DistGraph(coll, g.n, 0, g.n, g.row_ptr, g.col, g.w)
    for name, ctx, G in (("p", plain, Gp), ("c", coll, Gc)):
        F0, AB, Gr = plp.fgrad(ctx, G, U, p)
        Hv = plp.hessvec(ctx, G, U, eta, p, AB, mode=mode, G_in=Gr)
        F, ABo, G2, Hv3 = plp.fgrad_hessvec(ctx, G, U, eta, p, AB_in=AB, mode=mode)
        torch.cuda.synchronize()
        kern = plp.last_edge_kernel()
        for key, v in (("Hv", Hv), ("F", F), ("AB", ABo), ("G", G2), ("Hv3", Hv3)):
            out[f"{{name}}_{{k}}_{{key}}"] = v.cpu().numpy()
        out[f"{{name}}_{{k}}_kern"] = np.array(kern)
np.savez({path!r}, **out)
"""


def test_interior_boundary_split_path(plp, tmp_path):
    """The overlapped collective pass (interior tiles while the halo exchange is in flight on the
    comm stream, then the boundary tiles; two launches whose CTA partials are reduced together).
    PLP_DEBUG_SPLIT=1 marks every third tile a boundary tile so the path runs on one GPU: rows (G,
    Hv) are bitwise those of the single launch, A, B and F equal up to the partial grouping."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    path = str(tmp_path / "split.npz")
    script = tmp_path / "split.py"
    script.write_text(_SPLIT_SCRIPT.format(root=os.path.dirname(here), tests=here, path=path))
    subprocess.check_call([sys.executable, str(script)], env=dict(os.environ, PLP_DEBUG_SPLIT="1"))
    z = np.load(path)
    for k in (8, 4):
        assert str(z[f"c_{k}_kern"]).startswith("edge_halo_kernel"), str(z[f"c_{k}_kern"])
        for key in ("Hv", "G", "Hv3"):
            if k == 8:  # sparse mode: rows bitwise
                assert np.array_equal(z[f"p_{k}_{key}"], z[f"c_{k}_{key}"]), (k, key)
            else:  # full mode: the rank-two epilogue uses the reduced dots (partial grouping)
                assert colwise_relerr(z[f"c_{k}_{key}"], z[f"p_{k}_{key}"]) < 1e-13, (k, key)
        for key in ("F", "AB"):
            assert scalar_relerr(z[f"c_{k}_{key}"], z[f"p_{k}_{key}"]) < 1e-14, (k, key)


@pytest.mark.parametrize("n,dim,K,seed", [(30_000, 8, 8, 0), (20_011, 4, 5, 1), (5_000, 3, 3, 2),
                                          (40_000, 12, 10, 3)])
def test_kmeans_dist_one_rank_bitwise_equal_to_kmeans(plp, ctxs, n, dim, K, seed):
    """plp_kmeans_dist on a one-rank communicator (the collective seeding / Lloyd / reseed code
    path: sums all-reduced, picks by the owning rank and broadcast) is bitwise plp_kmeans, and
    plp_kmeans_dist on a context without a communicator is too; labels equal the oracle's."""
    plain, coll = ctxs
    rng = np.random.default_rng(seed)
    C = rng.uniform(-6, 6, size=(K, dim))
    X = C[rng.integers(0, K, n)] + rng.standard_normal((n, dim))
    Xt = torch.from_numpy(X).cuda()
    u = draw_uniforms(4, K)
    ref = plp.kmeans(plain, Xt, K, u, restarts=4)
    for ctx in (coll, plain):
        got = plp.kmeans_dist(ctx, Xt, K, u, restarts=4)
        assert torch.equal(got[0], ref[0])
        assert torch.equal(got[1], ref[1])
        assert got[2] == ref[2] and got[3] == ref[3]
    lab_o, _, sse_o, _ = oracle.kmeans(X, K, u, restarts=4)
    assert np.array_equal(ref[0].cpu().numpy(), lab_o)


def test_kmeans_dist_empty_cluster_reseed_one_rank(plp, ctxs):
    """Duplicate points force empty clusters: the farthest-point reseed through the collective
    path equals plp_kmeans bitwise."""
    plain, coll = ctxs
    rng = np.random.default_rng(7)
    X = np.repeat(rng.standard_normal((6, 4)), 500, axis=0)
    X[:10] += 1e-3 * rng.standard_normal((10, 4))
    Xt = torch.from_numpy(X).cuda()
    u = draw_uniforms(3, 8)
    ref = plp.kmeans(plain, Xt, 8, u, restarts=3)
    got = plp.kmeans_dist(coll, Xt, 8, u, restarts=3)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1]) and got[2] == ref[2]


@pytest.mark.parametrize("cfg,n,k,p,delta", [("C2", 4003, 16, 1.5, 0.3), ("C2", 4000, 2, 1.2, 50.0),
                                              ("C5", 30000, 8, 1.2, 1e3)])
def test_fused_tcg_on_collective_context(plp, ctxs, cfg, n, k, p, delta):
    """The fused device tCG on a collective context (k x k and scalar totals all-reduced, then the
    scalar step in tcg_step_kernel): on the one-rank communicator bitwise the plain context's tCG
    where neither folds pass A into the edge pass (k = 16; k = 2 on a graph without halo tiles),
    and at k = 8 on a tile-ordered graph (plain: pass A folded) the same iteration count and status
    with the step within 1e-10; the oracle's tCG agrees within 1e-9."""
    from oracle import solver as osol
    from paper_2605_26975_b200 import solver
    plain, coll = ctxs
    g = make_config(cfg, n=n)
    if cfg == "C5":
        g = permute_graph(g, plp.tile_order(g.row_ptr, g.col))
    Uo, _ = oracle.retract(draw_U(g.n, k, 5), np.zeros((g.n, k)))
    res = []
    for ctx, mk in ((plain, lambda c: plp.Graph(c, g.row_ptr, g.col, g.w)),
                    (coll, lambda c: plp.DistGraph(c, g.n, 0, g.n, g.row_ptr, g.col, g.w))):
        G = mk(ctx)
        with torch.cuda.stream(ctx.stream):
            tr = solver.GrassmannTR(ctx, G, k, solver.SolverConfig(tcg_fused=True, tcg_graph=False))
            st = solver._State(tr, torch.from_numpy(Uo).cuda(), p)
            eta, Heta, it, status = tr.tcg_device(st, p, delta)
        torch.cuda.synchronize()
        res.append((eta.cpu().numpy(), it, status))
    (e0, it0, s0), (e1, it1, s1) = res
    assert (it0, s0) == (it1, s1)
    if k == 8:
        assert np.max(np.abs(e0 - e1)) <= 1e-10 * np.max(np.abs(e0))
    else:
        assert np.array_equal(e0, e1)
    ocfg = osol.default_cfg(g.n, k)
    sto = osol._state(g, Uo, p, osol.oracle_fns())
    eta_o, _, it_o, status_o = osol.tcg(
        lambda xi: osol._hess(g, sto, p, xi, ocfg["eps"], "sparse", osol.oracle_fns()), sto["grad"], Uo, delta, ocfg)
    assert (it1, s1) == (it_o, status_o)
    assert np.max(np.abs(e1 - eta_o)) <= 1e-9 * np.max(np.abs(eta_o))
