"""GPU-vs-oracle parity of the tall-skinny Grassmann kernels (projection, Cholesky-QR2 retraction,
Gram, dot, axpby, gathers), k-means and RCut, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle
from plp_inputs import make_config, streams, draw_uniforms, permute_graph
from helpers import TOL, colwise_relerr, scalar_relerr, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plp():
    from paper_2605_26975_b200 import plp as mod
    return mod


@pytest.fixture(scope="module")
def ctx(plp):
    return plp.Context(0)


def orthonormal(rng, n, k):
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q


@pytest.mark.parametrize("n,k", [(100_003, 8), (50_001, 20), (7, 3), (200_000, 2), (3001, 32), (999, 1)])
def test_project_parity(plp, ctx, n, k):
    rng = streams(n)[1]
    U = orthonormal(rng, n, k)
    G = rng.standard_normal((n, k))
    out = to_np(plp.project(ctx, torch.from_numpy(U).cuda(), torch.from_numpy(G).cuda()))
    assert colwise_relerr(out, oracle.project(U, G)) < TOL
    assert np.max(np.abs(U.T @ out)) < 1e-12 * np.sqrt(n)


def test_project_in_place(plp, ctx):
    rng = streams(1)[1]
    U = orthonormal(rng, 5000, 8)
    G = rng.standard_normal((5000, 8))
    Gt = torch.from_numpy(G).cuda()
    plp.project(ctx, torch.from_numpy(U).cuda(), Gt, out=Gt)
    assert colwise_relerr(to_np(Gt), oracle.project(U, G)) < TOL


@pytest.mark.parametrize("n,k", [(100_003, 8), (50_001, 20), (9, 3), (3001, 32), (400, 1)])
def test_retract_parity(plp, ctx, n, k):
    rng = streams(n + 1)[1]
    U = orthonormal(rng, n, k)
    xi = oracle.project(U, 0.5 * rng.standard_normal((n, k)) / np.sqrt(n))
    R = torch.empty(k, k, dtype=torch.float64, device="cuda")
    Q = to_np(plp.retract(ctx, torch.from_numpy(U).cuda(), torch.from_numpy(xi).cuda(), R=R))
    Qo, Ro = oracle.retract(U, xi)
    assert colwise_relerr(Q, Qo) < TOL
    assert colwise_relerr(to_np(R), Ro) < TOL
    assert np.max(np.abs(Q.T @ Q - np.eye(k))) < 1e-13


def test_retract_rank_deficient_raises(plp, ctx):
    rng = streams(2)[1]
    U = orthonormal(rng, 1000, 4)
    xi = -U.copy()
    xi[:, 0] += 0.0  # U + xi = 0 -> Gram = 0
    with pytest.raises(plp.PlpError, match="PLP_ERR_RANK"):
        plp.retract(ctx, torch.from_numpy(U).cuda(), torch.from_numpy(xi).cuda())


def test_gram_dot_axpby_gather(plp, ctx):
    rng = streams(3)[1]
    n, k = 77_777, 8
    X, Y = rng.standard_normal((2, n, k))
    Xt, Yt = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    assert colwise_relerr(to_np(plp.gram(ctx, Xt, Yt)), X.T @ Y) < 1e-12
    d = to_np(plp.dot(ctx, Xt, Yt))[0]
    assert abs(d - oracle.dense.dot(X, Y)) < 1e-12 * np.sum(np.abs(X * Y))
    plp.axpby(ctx, 0.5, Xt, -2.0, Yt)
    assert colwise_relerr(to_np(Yt), 0.5 * X - 2.0 * Y) < 1e-15
    idx = rng.integers(0, n, 1000)
    out = to_np(plp.gather_rows(ctx, torch.from_numpy(idx).cuda(), Xt))
    assert np.array_equal(out, X[idx])


def test_cholesky_and_apply_rinv(plp, ctx):
    rng = streams(4)[1]
    n, k = 20_000, 6
    Y = rng.standard_normal((n, k))
    C = Y.T @ Y
    R, info = plp.cholesky(ctx, torch.from_numpy(C).cuda())
    assert int(to_np(info)[0]) == 0
    Rr = np.linalg.cholesky(C).T
    assert colwise_relerr(to_np(R), Rr) < 1e-13
    Q = to_np(plp.apply_rinv(ctx, torch.from_numpy(Y).cuda(), R))
    assert colwise_relerr(Q, Y @ np.linalg.inv(Rr)) < 1e-12
    U = rng.standard_normal((n, k))
    M = rng.standard_normal((k, k))
    out = to_np(plp.apply_sub(ctx, torch.from_numpy(U).cuda(), torch.from_numpy(M).cuda(),
                              torch.from_numpy(Y).cuda()))
    assert colwise_relerr(out, Y - U @ M) < 1e-13


# ----------------------------------------------------------------------------------- k-means ---
@pytest.mark.parametrize("n,dim,K,restarts", [(1000, 3, 3, 10), (100_000, 2, 2, 3), (60_000, 8, 8, 2),
                                              (4, 1, 2, 10), (20_000, 20, 20, 1), (5000, 5, 7, 4),
                                              # > 1024 x 256 points: the D^2 pick's per-thread chunk
                                              # ranges hold several chunks (second scan level)
                                              (600_077, 8, 8, 2), (300_001, 4, 6, 1)])
def test_kmeans_parity(plp, ctx, n, dim, K, restarts):
    rng = streams(n + dim)[1]
    if n == 4:
        X = np.array([[0.0], [0.1], [10.0], [10.1]])
    else:
        centers = rng.uniform(-5, 5, (K, dim))
        X = centers[rng.integers(0, K, n)] + rng.standard_normal((n, dim))
    u = draw_uniforms(restarts, K, seed=n)
    lab_o, C_o, sse_o, it_o = oracle.kmeans(X, K, u, restarts=restarts)
    lab, C, sse, it = plp.kmeans(ctx, torch.from_numpy(X).cuda(), K, u, restarts=restarts)
    assert np.array_equal(to_np(lab), lab_o)  # integer decisions identical (same fp64 rounding)
    assert colwise_relerr(to_np(C), C_o) < TOL
    assert scalar_relerr(sse, sse_o) < TOL
    assert it == it_o


def test_kmeans_identical_points_and_empty_repair(plp, ctx):
    X = np.ones((50, 2))
    u = draw_uniforms(2, 3, seed=1)
    lab_o, C_o, sse_o, _ = oracle.kmeans(X, 3, u, restarts=2)
    lab, C, sse, _ = plp.kmeans(ctx, torch.from_numpy(X).cuda(), 3, u, restarts=2)
    assert sse == sse_o == 0.0 and np.array_equal(to_np(lab), lab_o)
    # two far clusters + K=3 forces an empty cluster during Lloyd with some seeds
    rng = streams(7)[1]
    X = np.concatenate([rng.standard_normal((300, 2)) * 0.01, 100 + rng.standard_normal((3, 2)) * 0.01])
    u = draw_uniforms(5, 3, seed=3)
    lab_o, C_o, sse_o, it_o = oracle.kmeans(X, 3, u, restarts=5)
    lab, C, sse, it = plp.kmeans(ctx, torch.from_numpy(X).cuda(), 3, u, restarts=5)
    assert np.array_equal(to_np(lab), lab_o) and scalar_relerr(sse, sse_o) < TOL


# -------------------------------------------------------------------------------------- RCut ---
@pytest.mark.parametrize("name,K", [("C1", 3), ("C2", 2), ("C5", 8)])
def test_rcut_parity(plp, ctx, name, K):
    g = make_config(name) if name != "C5" else make_config("C5", n=50_000)
    lab = streams(K)[1].integers(0, K, g.n).astype(np.int32)
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    rc, cut, sizes = plp.rcut(ctx, Gh, K, torch.from_numpy(lab).cuda())
    rc_o, cut_o, sizes_o = oracle.rcut(g, lab, K)
    assert np.array_equal(to_np(sizes), sizes_o)
    assert scalar_relerr(to_np(cut), cut_o) < 1e-12
    assert scalar_relerr(to_np(rc)[0], rc_o) < 1e-12


def test_rcut_empty_cluster_is_nan(plp, ctx):
    g = make_config("C1")
    lab = np.zeros(g.n, np.int32)
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    rc, _, sizes = plp.rcut(ctx, Gh, 2, torch.from_numpy(lab).cuda())
    assert np.isnan(to_np(rc)[0]) and to_np(sizes)[1] == 0


def test_end_to_end_p2_labels_and_rcut_c1(plp, ctx):
    """p = 2 on C1: the exact minimiser spans the 3 smallest Laplacian eigenvectors (numpy eigh,
    textbook); its F at p=2 is their sum, k-means labels on both sides are identical, and RCut
    from identical labels agrees to 1e-12."""
    g = make_config("C1")
    L = np.diag(np.asarray(g.to_scipy().sum(1)).ravel()) - g.to_scipy().toarray()
    lam, V = np.linalg.eigh(L)
    U = V[:, :3]
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    F, AB, Gr = plp.fgrad(ctx, Gh, torch.from_numpy(U).cuda(), 2.0)
    assert abs(to_np(F)[0] - lam[:3].sum()) < 1e-10
    assert np.max(np.abs(to_np(Gr))) < 1e-10
    u = draw_uniforms(10, 3)
    lab_o, _, _, _ = oracle.kmeans(U, 3, u)
    lab, _, _, _ = plp.kmeans(ctx, torch.from_numpy(U).cuda(), 3, u)
    assert np.array_equal(to_np(lab), lab_o)
    rc, _, _ = plp.rcut(ctx, Gh, 3, lab)
    rc_o, _, _ = oracle.rcut(g, lab_o, 3)
    assert scalar_relerr(to_np(rc)[0], rc_o) < 1e-12
