"""GPU-vs-oracle parity of plp_hessvec on tile-ordered graphs: the Hessian-vector product every
tCG iteration of the solver runs (Alg. 1; sparse and full mode).

On a tile-ordered graph plp_hessvec runs the halo kernel's adaptive variant (edge_halo.cuh,
ADAPT): rows whose differences leave the fast power domain (mostly |d| < eps, the degenerate
regime of flattened p-Laplacian iterates) are recomputed from shared memory in the capped form
s_cap = min(s_raw, eps^{p-2}), and a warp whose previous row needed that form goes there directly.
These tests hold that path to the oracle (1e-9, north star), including the degenerate regime
(piecewise-constant columns + 1e-12 noise, eps = 1e-9 and 0.3, exact zero rows), and check that
the adaptive halo kernel is what ran."""
import numpy as np
import pytest
import torch

import oracle
from plp_inputs import make_config, draw_U, draw_eta, permute_graph, streams
from helpers import TOL, colwise_relerr, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plp():
    from paper_2605_26975_b200 import plp as mod
    return mod


@pytest.fixture(scope="module")
def ctx(plp):
    return plp.Context(0)


_G = {}


def tgraph(name):
    """Tile-ordered graphs (plp_tile_order: the ordering the solver runs on)."""
    if name not in _G:
        from paper_2605_26975_b200 import plp as mod
        base = {"C5t": ("C5", 100_000), "C3t": ("C3", 40 ** 3), "D16t": ("D16", None),
                "C2t": ("C2", 30_000)}[name]
        g0 = make_config(base[0], n=base[1])
        _G[name] = permute_graph(g0, mod.tile_order(g0.row_ptr, g0.col))
    return _G[name]


def degenerate_U(g, k, seed, noise=1e-12, zero_rows=True, half=True):
    """Columns piecewise constant on blocks of ~300 consecutive (tile-ordered) nodes plus `noise`
    (most neighbour differences fall below eps), exact zero rows, and (half=True) random values on
    the second half of the nodes so that warps switch between the capped and the fast form."""
    rng = streams(seed)[1]
    blk = np.arange(g.n) // 300
    lv = rng.standard_normal((blk.max() + 1, k))
    U = lv[blk] + noise * rng.standard_normal((g.n, k))
    if half:
        U[g.n // 2:] = rng.standard_normal((g.n - g.n // 2, k))
    if zero_rows:
        U[rng.choice(g.n, size=max(4, g.n // 500), replace=False)] = 0.0
    return U


def assert_adaptive_path(kern, k, name=""):
    """k = 4, 8: the halo kernel's adaptive variant.  Where a tile's halo does not fit in shared
    memory (k = 16 tiles; C3's 3-D grid with random long-range edges has tiles with ~1000 halo
    rows) the staged kernel (libdevice row recompute) runs instead."""
    ok = (kern.startswith("edge_halo_kernel[") and "adapt" in kern) or \
        ((k == 16 or name.startswith("C3")) and kern.startswith("edge_staged_kernel"))
    assert ok, kern


def gpu_hessvec(plp, ctx, g, U, eta, p, mode, eps):
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=plp.VALIDATE_SYMMETRIC)
    Ut = torch.from_numpy(U).cuda()
    Et = torch.from_numpy(eta).cuda()
    F, AB, Gr = plp.fgrad(ctx, Gh, Ut, p, want_grad=(mode == plp.HESS_FULL))
    Hv = plp.hessvec(ctx, Gh, Ut, Et, p, AB, mode=mode, eps=eps, G_in=Gr)
    torch.cuda.synchronize()
    kern = plp.last_edge_kernel()
    return to_np(Hv), to_np(AB), kern


def oracle_hessvec(g, U, eta, p, mode, eps):
    _, A, B = oracle.objective(g, U, p)
    return oracle.hessvec(g, U, eta, p, eps, "full" if mode == 1 else "sparse", AB=(A, B)), A, B


CASES = [("C5t", 8, 1.2), ("C5t", 4, 1.5), ("C5t", 16, 1.8), ("C5t", 8, 1.37), ("C5t", 8, 2.0),
         ("D16t", 8, 1.2), ("D16t", 4, 1.1), ("D16t", 16, 1.5),
         ("C3t", 8, 1.5), ("C3t", 4, 1.2), ("C3t", 16, 1.37), ("C2t", 4, 1.1)]


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name,k,p", CASES)
def test_hessvec_tile_ordered_random(plp, ctx, name, k, p, mode):
    g = tgraph(name)
    U, eta = draw_U(g.n, k, 12), draw_eta(g.n, k, 12)
    Hv, AB, kern = gpu_hessvec(plp, ctx, g, U, eta, p, mode, 1e-9)
    assert_adaptive_path(kern, k, name)
    ref, A, B = oracle_hessvec(g, U, eta, p, mode, 1e-9)
    assert colwise_relerr(AB[:k], A) < TOL and colwise_relerr(AB[k:], B) < TOL
    e = colwise_relerr(Hv, ref)
    assert e < TOL, e


@pytest.mark.parametrize("eps", [1e-9, 0.3])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("name,k,p", [("C5t", 8, 1.2), ("C5t", 4, 1.5), ("C5t", 16, 1.1),
                                      ("D16t", 8, 1.2), ("D16t", 4, 1.8), ("C3t", 8, 1.37),
                                      ("C5t", 8, 2.0)])
def test_hessvec_degenerate_regime(plp, ctx, name, k, p, mode, eps):
    """Piecewise-constant columns + 1e-12 noise (|d| < eps on most edges of the first half of the
    nodes), exact zero rows (node cap), random values on the second half (warps switch forms)."""
    g = tgraph(name)
    U = degenerate_U(g, k, 5)
    eta = draw_eta(g.n, k, 5)
    Hv, AB, kern = gpu_hessvec(plp, ctx, g, U, eta, p, mode, eps)
    assert_adaptive_path(kern, k, name)
    ref, A, B = oracle_hessvec(g, U, eta, p, mode, eps)
    assert colwise_relerr(AB[:k], A) < TOL and colwise_relerr(AB[k:], B) < TOL
    e = colwise_relerr(Hv, ref)
    assert e < TOL, e


@pytest.mark.parametrize("name,k,p", [("C5t", 8, 1.2), ("D16t", 4, 1.5)])
def test_hessvec_fully_degenerate_and_exact_ties(plp, ctx, name, k, p):
    """Every node degenerate (no random half): exact ties (noise 0) within blocks and 1e-13 noise;
    the capped form runs on every warp for the whole launch."""
    g = tgraph(name)
    for noise in (0.0, 1e-13):
        U = degenerate_U(g, k, 9, noise=noise, half=False)
        eta = draw_eta(g.n, k, 9)
        for mode in (0, 1):
            Hv, AB, kern = gpu_hessvec(plp, ctx, g, U, eta, p, mode, 1e-9)
            assert kern.startswith("edge_halo_kernel[") and "adapt" in kern, kern
            ref, A, B = oracle_hessvec(g, U, eta, p, mode, 1e-9)
            e = colwise_relerr(Hv, ref)
            assert e < TOL, (noise, mode, e)


def test_hessvec_out_of_fast_domain_on_halo_path(plp, ctx):
    """|d| below 2^-120 (nonzero) and above 2^120 on the adaptive halo path: libdevice for what
    the capped form flags, still equal to the oracle."""
    g = tgraph("C5t")
    k = 8
    U = draw_U(g.n, k, 21)
    U[:, 1] = (1.0 + np.arange(g.n) * 1e-2) * 1e-38
    U[:7, 0] *= 1e125
    eta = draw_eta(g.n, k, 21)
    for eps in (1e-300, 1e-9):
        Hv, AB, kern = gpu_hessvec(plp, ctx, g, U, eta, 1.5, 0, eps)
        assert kern.startswith("edge_halo_kernel[") and "adapt" in kern, kern
        ref, _, _ = oracle_hessvec(g, U, eta, 1.5, 0, eps)
        assert colwise_relerr(Hv, ref) < TOL


def test_hessvec_repeated_calls_bitwise(plp, ctx):
    """Two calls on the same inputs (the tCG calls Hv thousands of times at fixed U) are bitwise
    equal, in the degenerate regime too (the capped-form carry-over is per launch)."""
    g = tgraph("C5t")
    U = degenerate_U(g, 8, 3)
    eta = draw_eta(g.n, 8, 3)
    a = gpu_hessvec(plp, ctx, g, U, eta, 1.2, 0, 1e-9)[0]
    b = gpu_hessvec(plp, ctx, g, U, eta, 1.2, 0, 1e-9)[0]
    assert np.array_equal(a, b)
