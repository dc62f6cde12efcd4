"""Full-size parity at BASELINE.json's headline config (C5: 8,388,608 nodes, k = 8, p = 1.2, tile
order), in the launch configuration bench.py times: the GPU's A, B (hence F) against the oracle's
full sums, and G, Hv on sampled rows the oracle computes one by one.  Also the sharded (P-rank)
row layout of the multi-GPU path, emulated on one GPU shard by shard (no inter-kernel waits)."""
import os
import sys

import numpy as np
import pytest
import torch

import oracle
from plp_inputs import draw_U, draw_eta, make_config, permute_graph
from helpers import TOL, colwise_relerr, scalar_relerr, to_np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def plp():
    from paper_2605_26975_b200 import plp as mod
    return mod


@pytest.fixture(scope="module")
def c5():
    from bench import get_graph
    return get_graph("C5", "tile")


def test_c5_fullsize_sampled_parity(plp, c5):
    g = c5
    k, p, eps = 8, 1.2, 1e-9
    U = draw_U(g.n, k, 0)
    eta = draw_eta(g.n, k, 0)
    ctx = plp.Context(0)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=plp.VALIDATE)
    Ut = torch.from_numpy(U).cuda()
    Et = torch.from_numpy(eta).cuda()
    F0, AB_in, _ = plp.fgrad(ctx, G, Ut, p, want_grad=False)
    F, AB, Gr, Hv = plp.fgrad_hessvec(ctx, G, Ut, Et, p, AB_in=AB_in, eps=eps)
    torch.cuda.synchronize()
    oracle.set_threads(os.cpu_count() or 1)
    Fo, A, B = oracle.objective(g, U, p)
    assert scalar_relerr(to_np(AB)[:k], A) < TOL and scalar_relerr(to_np(AB)[k:], B) < TOL
    assert scalar_relerr(to_np(F)[0], Fo) < TOL and scalar_relerr(to_np(F0)[0], Fo) < TOL
    rows = np.unique(np.concatenate([np.random.default_rng(0).integers(0, g.n, 3000),
                                     [0, 1, g.n - 1, g.n // 2]]))
    Go = oracle.euc_grad(g, U, p, A, B, rows=rows)
    Ho = oracle.hessvec(g, U, eta, p, eps, "sparse", (A, B), rows=rows)
    assert colwise_relerr(to_np(Gr)[rows], Go) < TOL
    assert colwise_relerr(to_np(Hv)[rows], Ho) < TOL


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_rows_equal_single_gpu(plp, world):
    """Each rank's local CSR (owned rows + halo columns) through the same C ABI gives the rows of
    the single-GPU call; partial A, B sum to the global values."""
    from paper_2605_26975_b200.dist import HaloPlan
    g0 = make_config("C5", n=200_000)
    g = permute_graph(g0, plp.tile_order(g0.row_ptr, g0.col))
    k, p = 8, 1.2
    U, eta = draw_U(g.n, k, 3), draw_eta(g.n, k, 3)
    ctx = plp.Context(0)
    Gg = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    Ut, Et = torch.from_numpy(U).cuda(), torch.from_numpy(eta).cuda()
    _, AB, _ = plp.fgrad(ctx, Gg, Ut, p, want_grad=False)
    _, _, G1, H1 = plp.fgrad_hessvec(ctx, Gg, Ut, Et, p, AB_in=AB)
    AB_sum = torch.zeros_like(AB)
    for r in range(world):
        pl = HaloPlan(g.row_ptr, g.col, g.w, r, world, k)
        ext = np.concatenate([np.arange(pl.r0, pl.r1), pl.halo])
        Gl = plp.Graph(ctx, pl.rp_loc, pl.col_loc, pl.w_loc, n_cols=ext.size, flags=0)
        Ue = torch.from_numpy(U[ext]).cuda()
        Ee = torch.from_numpy(eta[ext]).cuda()
        Gr = torch.empty(pl.n_loc, k, dtype=torch.float64, device="cuda")
        Hr = torch.empty_like(Gr)
        ABp = torch.empty_like(AB)
        plp.edge_pass(ctx, Gl, Ue, Ee, p, 1e-9, AB_in=AB, AB_out=ABp, G=Gr, Hv=Hr)
        AB_sum += ABp
        assert colwise_relerr(to_np(Gr), to_np(G1)[pl.r0:pl.r1]) < 1e-13
        assert colwise_relerr(to_np(Hr), to_np(H1)[pl.r0:pl.r1]) < 1e-13
    assert scalar_relerr(to_np(AB_sum), to_np(AB)) < 1e-12
