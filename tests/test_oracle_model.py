"""Pins of the oracle's F / Delta_p / EucGrad / EucHessianEta against things other than itself:
closed forms (textbook Laplacian, path/cycle spectra), worked examples, exact
identities (Euler homogeneity), finite differences and symmetry.  No GPU needed."""
import math

import numpy as np
import pytest
import scipy.sparse.csgraph as csgraph

import oracle
from plp_inputs import (cycle_graph, path_graph, random_graph, single_edge, csr_from_undirected,
                        streams, make_config)

PS = [2.0, 1.8, 1.5, 1.2, 1.1]


def relerr(x, ref):
    x, ref = np.asarray(x, float), np.asarray(ref, float)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


def lap(g):
    return csgraph.laplacian(g.to_scipy()).toarray()


def separated_U(rng, n, k, gap=0.05):
    """Random U with every |u_i - u_j| and every |u_i| above `gap` (FD needs smoothness)."""
    while True:
        U = rng.standard_normal((n, k))
        ok = np.min(np.abs(U)) > gap
        for l in range(k):
            s = np.sort(U[:, l])
            ok = ok and np.min(np.diff(s)) > gap
        if ok:
            return U


def small_graph(seed, n=10):
    return random_graph(streams(seed)[0], n, avg_deg=4.0, name=f"r{seed}")


# ------------------------------------------------------------------------------------ phi_p ---
def test_phi_worked_examples():
    for x in (-3.0, 0.0, 5.0):
        assert oracle.phi(x, 2.0) == x
    assert oracle.phi(-4.0, 1.5) == -2.0
    assert oracle.phi(0.0, 1.1) == 0.0


# --------------------------------------------------------------------------------- Delta_p ---
def test_plaplacian_examples():
    g = single_edge()
    L = oracle.plaplacian(g, np.array([[0.0], [1.0]]), 2.0)
    assert np.array_equal(L[:, 0], [-1.0, 1.0])
    gg = small_graph(3)
    assert np.all(oracle.plaplacian(gg, np.full((gg.n, 2), 0.7), 1.3) == 0.0)


@pytest.mark.parametrize("seed", range(5))
def test_plaplacian_p2_is_textbook_laplacian(seed):
    g = small_graph(seed, 15)
    U = streams(seed)[1].standard_normal((g.n, 3))
    assert relerr(oracle.plaplacian(g, U, 2.0), lap(g) @ U) < 1e-14


# ---------------------------------------------------------------------------------- F_p ---
def test_objective_single_edge():
    F, A, B = oracle.objective(single_edge(), np.array([[1.0], [-1.0]]), 2.0)
    assert F == 2.0 and A[0] == 4.0 and B[0] == 2.0


@pytest.mark.parametrize("seed", range(4))
def test_objective_p2_rayleigh_quotients(seed):
    """p=2: A = u^T L u (textbook L = D - W, which pins the 1/2 of Eq. (1)), B = u^T u."""
    g = small_graph(seed, 12)
    U = streams(seed)[1].standard_normal((g.n, 3))
    F, A, B = oracle.objective(g, U, 2.0)
    L = lap(g)
    Ar = np.einsum("il,ij,jl->l", U, L, U)
    assert relerr(A, Ar) < 1e-14
    assert relerr(B, np.sum(U * U, axis=0)) < 1e-15
    assert abs(F - np.sum(Ar / np.sum(U * U, axis=0))) < 1e-13 * abs(F)


@pytest.mark.parametrize("p", PS)
def test_objective_invariances(p):
    g = small_graph(7, 14)
    rng = streams(7)[1]
    U = rng.standard_normal((g.n, 3))
    F, A, B = oracle.objective(g, U, p)
    c = np.array([3.7, -0.2, 11.0])
    F2, _, _ = oracle.objective(g, U * c[None, :], p)
    assert abs(F2 - F) < 1e-13 * F  # degree-0 homogeneity per column
    U[:, 1] = 0.42  # constant column -> A_1 = 0
    _, A3, _ = oracle.objective(g, U, p)
    assert A3[1] == 0.0


@pytest.mark.parametrize("p", PS)
def test_euler_identity_u_dot_plaplacian_equals_A(p):
    """<u, Delta_p u> = 1/2 sum w (u_i-u_j) phi_p(u_i-u_j) = A exactly (symmetric W)."""
    g = small_graph(11, 20)
    U = streams(11)[1].standard_normal((g.n, 4))
    A = oracle.numerators(g, U, p)
    L = oracle.plaplacian(g, U, p)
    assert relerr(np.sum(U * L, axis=0), A) < 1e-13


def test_objective_brute_force_dense_tiny():
    """Direct ordered double sum over a dense W (catches CSR traversal errors)."""
    g = small_graph(5, 7)
    W = g.to_scipy().toarray()
    U = streams(5)[1].standard_normal((g.n, 2))
    p = 1.37
    F, A, B = oracle.objective(g, U, p)
    Fd = 0.0
    for l in range(2):
        num = sum(W[i, j] * abs(U[i, l] - U[j, l]) ** p for i in range(g.n) for j in range(g.n))
        den = sum(abs(U[i, l]) ** p for i in range(g.n))
        Fd += num / (2.0 * den)
    assert abs(F - Fd) < 1e-14 * Fd


def path_eigvecs(m, ks):
    i = np.arange(m)
    return np.stack([np.cos(j * math.pi * (i + 0.5) / m) for j in ks], axis=1), \
        np.array([2.0 - 2.0 * math.cos(j * math.pi / m) for j in ks])


def test_path_graph_spectrum_p2():
    """P_m: lambda_j = 2 - 2cos(j pi/m), v_j(i) = cos(j pi (i+1/2)/m) -> F = sum lambda, grad = 0."""
    m = 9
    g = path_graph(m)
    V, lam = path_eigvecs(m, [0, 1, 2])
    F, _, _ = oracle.objective(g, V, 2.0)
    assert abs(F - lam.sum()) < 1e-14
    G = oracle.euc_grad(g, V, 2.0)
    assert np.max(np.abs(G)) < 1e-14


def test_cycle_graph_spectrum_p2():
    m = 12
    g = cycle_graph(m)
    i = np.arange(m)
    V = np.stack([np.ones(m), np.cos(2 * math.pi * i / m), np.sin(2 * math.pi * 2 * i / m)], axis=1)
    lam = np.array([0.0, 2 - 2 * math.cos(2 * math.pi / m), 2 - 2 * math.cos(4 * math.pi / m)])
    F, _, _ = oracle.objective(g, V, 2.0)
    assert abs(F - lam.sum()) < 1e-14
    assert np.max(np.abs(oracle.euc_grad(g, V, 2.0))) < 1e-14


# ------------------------------------------------------------------------------ gradient ---
def test_grad_single_edge_is_zero():
    G = oracle.euc_grad(single_edge(), np.array([[1.0], [-1.0]]), 2.0)
    assert np.all(G == 0.0)


def fd_grad(g, U, p, h=1e-4):
    G = np.zeros_like(U)
    for i in range(U.shape[0]):
        for l in range(U.shape[1]):
            def f(t):
                V = U.copy()
                V[i, l] += t
                return oracle.objective(g, V, p)[0]
            G[i, l] = (-f(2 * h) + 8 * f(h) - 8 * f(-h) + f(-2 * h)) / (12 * h)
    return G


@pytest.mark.parametrize("p", PS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_grad_finite_differences(p, seed):
    g = small_graph(seed, 10)
    U = separated_U(streams(seed)[1], g.n, 2)
    G = oracle.euc_grad(g, U, p)
    assert relerr(G, fd_grad(g, U, p)) < 1e-7  # SPEC.md:244 asks 1e-5


@pytest.mark.parametrize("p", PS)
def test_grad_tangency(p):
    g = small_graph(21, 30)
    U = streams(21)[1].standard_normal((g.n, 3))
    G = oracle.euc_grad(g, U, p)
    for l in range(3):
        assert abs(G[:, l] @ U[:, l]) < 1e-13 * np.linalg.norm(G[:, l]) * np.linalg.norm(U[:, l])


def test_grad_p2_closed_form():
    g = small_graph(4, 16)
    U = streams(4)[1].standard_normal((g.n, 3))
    F, A, B = oracle.objective(g, U, 2.0)
    Gr = (2.0 / B) * (lap(g) @ U - (A / B) * U)
    assert relerr(oracle.euc_grad(g, U, 2.0), Gr) < 1e-13


def test_grad_rows_subset_matches_full():
    g = small_graph(9, 25)
    U = streams(9)[1].standard_normal((g.n, 2))
    rows = np.array([3, 0, 24, 7])
    assert np.array_equal(oracle.euc_grad(g, U, 1.4, rows=rows), oracle.euc_grad(g, U, 1.4)[rows])


# ------------------------------------------------------------------------------- Hessian ---
@pytest.mark.parametrize("p", PS)
@pytest.mark.parametrize("seed", [0, 1])
def test_sparse_hessian_euler_identity(p, seed):
    """H_sparse u = (p-1) grad exactly (HessA u = (p-1) grad A, HessB u = (p-1) grad B by Euler),
    valid when no cap fires (random U)."""
    g = small_graph(seed, 30)
    U = streams(seed)[1].standard_normal((g.n, 3))
    Hu = oracle.hessvec(g, U, U, p, eps=1e-12, mode="sparse")
    assert relerr(Hu, (p - 1.0) * oracle.euc_grad(g, U, p)) < 1e-12


@pytest.mark.parametrize("p", PS)
def test_full_hessian_euler_identity(p):
    """Exact Hessian of a degree-0 homogeneous f: Hess f . u = -grad f."""
    g = small_graph(13, 30)
    U = streams(13)[1].standard_normal((g.n, 3))
    Hu = oracle.hessvec(g, U, U, p, eps=1e-12, mode="full")
    assert relerr(Hu, -oracle.euc_grad(g, U, p)) < 1e-12


@pytest.mark.parametrize("p", PS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_full_hessian_finite_differences(p, seed):
    g = small_graph(seed + 40, 10)
    rng = streams(seed)[1]
    U = separated_U(rng, g.n, 2)
    eta = rng.standard_normal(U.shape)
    h = 1e-4
    gp = [oracle.euc_grad(g, U + t * eta, p) for t in (2 * h, h, -h, -2 * h)]
    fd = (-gp[0] + 8 * gp[1] - 8 * gp[2] + gp[3]) / (12 * h)
    assert relerr(oracle.hessvec(g, U, eta, p, mode="full"), fd) < 1e-6  # SPEC.md:266 asks 1e-4


@pytest.mark.parametrize("mode", ["sparse", "full"])
@pytest.mark.parametrize("p", [2.0, 1.5, 1.1])
def test_hessian_symmetry_and_linearity(mode, p):
    g = small_graph(17, 25)
    rng = streams(17)[1]
    U = rng.standard_normal((g.n, 2))
    v, w = rng.standard_normal((2, g.n, 2))
    Hv = oracle.hessvec(g, U, v, p, mode=mode)
    Hw = oracle.hessvec(g, U, w, p, mode=mode)
    for l in range(2):
        a, b = Hv[:, l] @ w[:, l], Hw[:, l] @ v[:, l]
        assert abs(a - b) < 1e-12 * (np.linalg.norm(Hv[:, l]) * np.linalg.norm(w[:, l]))
    H2 = oracle.hessvec(g, U, 2.5 * v - w, p, mode=mode)
    assert relerr(H2, 2.5 * Hv - Hw) < 1e-13
    assert np.all(oracle.hessvec(g, U, np.zeros_like(v), p, mode=mode) == 0.0)


def test_sparse_hessian_p2_closed_form():  # 2L/B - (2A/B^2) I
    g = small_graph(23, 18)
    rng = streams(23)[1]
    U = rng.standard_normal((g.n, 3))
    eta = rng.standard_normal((g.n, 3))
    F, A, B = oracle.objective(g, U, 2.0)
    ref = 2.0 * (lap(g) @ eta) / B - (2.0 * A / B ** 2) * eta
    assert relerr(oracle.hessvec(g, U, eta, 2.0), ref) < 1e-13


def test_sparse_hessian_edgeless():  # W = 0 -> A = 0, H = 0
    g = csr_from_undirected(4, np.zeros(0, int), np.zeros(0, int), np.zeros(0), "empty")
    U = np.array([[1.0], [2.0], [-1.0], [0.5]])
    assert np.all(oracle.hessvec(g, U, U[::-1].copy(), 1.5) == 0.0)


def test_hessian_parts_reconstruct_dense_operator():
    """Alg. 1 reconstruction: D (.) eta - eta H equals the dense H^l eta, where the
    dense operator is assembled from the row/column loops independently."""
    g = small_graph(29, 8)
    rng = streams(29)[1]
    U = rng.standard_normal((g.n, 1))
    p, eps = 1.3, 1e-9
    F, A, B = oracle.objective(g, U, p)
    Dd, H = oracle.hessian_parts(g, U, p, eps, A, B)
    W = g.to_scipy().toarray()
    u = U[:, 0]
    Wt = W * np.maximum(np.abs(u[:, None] - u[None, :]), eps) ** (p - 2.0)
    HA = p * (p - 1) * (np.diag(Wt.sum(1)) - Wt)
    HB = p * (p - 1) * np.diag(np.maximum(np.abs(u), eps) ** (p - 2.0))
    Hd = HA / B[0] - (A[0] / B[0] ** 2) * HB
    assert relerr(Dd[:, 0], np.diag(Hd)) < 1e-14
    eta = rng.standard_normal((g.n, 1))
    assert relerr(oracle.euc_hessian_eta(g, Dd, H, eta)[:, 0], Hd @ eta[:, 0]) < 1e-13


# ------------------------------------------------------------------------------ eps rule ---
def test_eps_cap_worked_example_tie():
    """Single edge, exact tie u_0 = u_1 = 0.5, p = 1.5: A = 0 and the curvature weight is
    w * eps^{p-2}; row 0 of Hv = p(p-1) w eps^{-1/2} (eta_0 - eta_1) / B (reading #6)."""
    g = single_edge()
    U = np.array([[0.5], [0.5]])
    eta = np.array([[1.0], [-1.0]])
    eps = 1e-9
    Hv = oracle.hessvec(g, U, eta, 1.5, eps=eps)
    B = 2 * 0.5 ** 1.5
    ref0 = 0.75 * eps ** -0.5 * 2.0 / B
    assert abs(Hv[0, 0] - ref0) < 1e-15 * abs(ref0)
    assert abs(Hv[1, 0] + ref0) < 1e-15 * abs(ref0)


def test_eps_cap_continuity_and_p2_independence():
    g = path_graph(4)
    eta = np.array([[1.0], [0.3], [-2.0], [0.7]])
    eps = 1e-6
    U_tie = np.array([[0.2], [0.2], [1.0], [0.0]])  # tie on edge (0,1), zero at node 3
    U_at = np.array([[0.2], [0.2 + eps], [1.0], [0.0]])
    h1 = oracle.hessvec(path_graph(4), U_tie, eta, 1.5, eps=eps)
    h2 = oracle.hessvec(path_graph(4), U_at, eta, 1.5, eps=eps)
    # a = eps exactly vs a = 0: same capped weight; only A/B shift by O(eps^1.5)
    assert relerr(h1, h2) < 1e-5
    # p = 2: the cap is irrelevant (weight exactly w), result = plain Laplacian formula
    for e in (1e-9, 1e-3, 0.5):
        F, A, B = oracle.objective(g, U_tie, 2.0)
        ref = 2.0 * (lap(g) @ eta) / B - (2.0 * A / B ** 2) * eta
        assert relerr(oracle.hessvec(g, U_tie, eta, 2.0, eps=e), ref) < 1e-14


def test_sharded_rows_with_halo_match_global():
    """Local CSR (owned rows, columns into owned+halo rows of U) gives the same row outputs and
    partial sums; used by the multi-GPU path."""
    g = make_config("C1", n=300)
    rng = streams(1)[1]
    U = rng.standard_normal((g.n, 3))
    p = 1.5
    F, A, B = oracle.objective(g, U, p)
    G = oracle.euc_grad(g, U, p, A, B)
    r0, r1 = 100, 220
    rp = g.row_ptr[r0:r1 + 1] - g.row_ptr[r0]
    cols = g.col[g.row_ptr[r0]:g.row_ptr[r1]].astype(np.int64)
    halo = np.unique(cols[(cols < r0) | (cols >= r1)])
    ext = np.concatenate([np.arange(r0, r1), halo])
    remap = {int(v): t for t, v in enumerate(ext)}
    lc = np.array([remap[int(c)] for c in cols], dtype=np.int32)

    class Loc:
        row_ptr, col, w = rp, lc, g.w[g.row_ptr[r0]:g.row_ptr[r1]]

    Gl = oracle.euc_grad(Loc, U[ext], p, A, B)
    assert np.array_equal(Gl, G[r0:r1])
    Al = oracle.numerators(Loc, U[ext], p)
    assert np.all(Al <= A + 1e-12)


def test_delaunay_generator_is_a_triangulation():
    """The NEXT-3 stand-in for delaunay_n<r>: symmetric, connected, planar
    (undirected edges <= 3n - 6, Euler), ~6n stored nonzeros, unit weights."""
    from plp_inputs import delaunay_graph
    g = delaunay_graph(streams(11)[0], 5000)
    A = g.to_scipy()
    assert (A != A.T).nnz == 0
    assert csgraph.connected_components(A)[0] == 1
    und = g.nnz // 2
    assert und <= 3 * g.n - 6 and 5.5 * g.n < g.nnz < 6.0 * g.n
    assert np.all(g.w == 1.0)


@pytest.mark.parametrize("p", [1.05, 1.2, 1.5, 1.8, 1.99])
def test_capped_weight_is_min_of_raw_and_cap(p):
    """The edge passes' capped form uses cap(|d|)^{p-2} = min(|d|^{p-2}, eps^{p-2}):
    exact because x^{p-2} is decreasing for p < 2 (checked on values spanning the cap, in the
    oracle's own arithmetic)."""
    eps = 1e-9
    rng = np.random.default_rng(int(p * 100))
    x = np.concatenate([10.0 ** rng.uniform(-14, 1, 2000), [eps, eps * (1 - 1e-15), eps * (1 + 1e-15)]])
    capped = np.maximum(x, eps) ** (p - 2.0)
    via_min = np.minimum(x ** (p - 2.0), eps ** (p - 2.0))
    assert np.max(np.abs(capped - via_min) / capped) <= 4e-16


@pytest.mark.parametrize("k", [1, 2, 4])
def test_folded_gram_and_apply_identities(k):
    """The folded fused tCG (k = 1, 2, 4) reads n x k arrays as n k / 8 rows of 8:
    the sum of the 8 / k diagonal k x k blocks of the 8 x 8 Gram is the true Gram, and applying the
    block-diagonal expansion of M equals X M row by row."""
    rng = np.random.default_rng(k)
    n = 8 * 37
    X, Y = rng.standard_normal((n, k)), rng.standard_normal((n, k))
    M = rng.standard_normal((k, k))
    Xf, Yf = X.reshape(n * k // 8, 8), Y.reshape(n * k // 8, 8)
    G8 = Xf.T @ Yf
    folded = sum(G8[b * k:(b + 1) * k, b * k:(b + 1) * k] for b in range(8 // k))
    assert np.allclose(folded, X.T @ Y, rtol=1e-13, atol=1e-12)
    Mbd = np.kron(np.eye(8 // k), M)
    assert np.allclose((Xf @ Mbd).reshape(n, k), X @ M, rtol=1e-13, atol=1e-12)
    # the Frobenius norm of the folded Gram is what ||P r||^2 subtracts
    assert np.isclose(np.sum(folded * folded), np.sum((X.T @ Y) ** 2), rtol=1e-12)


def test_fused_tcg_reformulations():
    """The fused tCG's reformulations against the definitions on random data:
    <d, P(EH) - d S> = sum d (EH - d S) - <U^T d, U^T EH>_F, and with U^T U = I,
    ||P r||^2 = ||r||^2 - ||U^T r||_F^2 and P(r + c Hd') = P(r + c Hd) for Hd' = EH - d S."""
    rng = np.random.default_rng(7)
    n, k = 500, 4
    U, _ = np.linalg.qr(rng.standard_normal((n, k)))
    A = rng.standard_normal((k, k))
    S = (A + A.T) / 2
    d, EH, r = (rng.standard_normal((n, k)) for _ in range(3))
    P = lambda X: X - U @ (U.T @ X)  # noqa: E731
    Hd = P(EH) - d @ S
    lhs = np.sum(d * Hd)
    rhs = np.sum(d * (EH - d @ S)) - np.sum((U.T @ d) * (U.T @ EH))
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))
    assert np.isclose(np.sum(P(r) ** 2), np.sum(r ** 2) - np.sum((U.T @ r) ** 2), rtol=1e-12)
    c = 0.37
    assert np.allclose(P(r + c * (EH - d @ S)), P(r + c * Hd), rtol=1e-12, atol=1e-12)


def test_node_cap_exact_zero_worked_example():
    """Exact zero node u_0 = 0 (reading #6, the node cap): single edge, u = (0, 1), p = 1.5.
    By hand: A = w |0 - 1|^p = w, B = |0|^p + |1|^p = 1, the edge weight w~ = w |1|^{p-2} = w, so
    HA eta = p(p-1) w (eta_0 - eta_1, eta_1 - eta_0) and HB eta = p(p-1)(eps^{p-2} eta_0, eta_1);
    Hv = HA eta / B - (A/B^2) HB eta."""
    w, p, eps = 0.7, 1.5, 1e-4
    g = single_edge(w)
    U = np.array([[0.0], [1.0]])
    eta = np.array([[0.3], [-0.2]])
    c = p * (p - 1)
    ref = np.array([c * w * (0.3 + 0.2) - w * c * eps ** (p - 2) * 0.3,
                    c * w * (-0.2 - 0.3) - w * c * (-0.2)])
    Hv = oracle.hessvec(g, U, eta, p, eps=eps)
    assert relerr(Hv[:, 0], ref) < 1e-14


@pytest.mark.parametrize("p", [1.8, 1.5, 1.2, 1.1])
@pytest.mark.parametrize("eps", [1e-9, 1e-2])
def test_hessvec_dense_assembly_with_zero_nodes_and_ties(p, eps):
    """Exact zero rows u_i = 0 and exact ties u_i = u_j in several columns: the oracle's sparse
    Hessian-vector product equals the dense operator HessA/B - (A/B^2) HessB assembled from the
    matrix definitions (SURVEY.md §8(c) formula 3; Alg. 1), column by column,
    with A, B from Eq. (1) written as dense sums."""
    g = small_graph(41, 14)
    rng = streams(41)[1]
    k = 3
    U = np.round(rng.standard_normal((g.n, k)) * 2.0) / 2.0  # ties and zeros
    U[3, :] = 0.0
    U[7, :] = 0.0  # two exact zero rows
    U[:, 0] += np.arange(g.n) * 1e-3  # keep column 0 tie-free as a control
    eta = rng.standard_normal((g.n, k))
    W = g.to_scipy().toarray()
    ref = np.zeros_like(eta)
    for l in range(k):
        u = U[:, l]
        Dm = np.abs(u[:, None] - u[None, :])
        A = 0.5 * np.sum(W * Dm ** p)
        B = np.sum(np.abs(u) ** p)
        Wt = W * np.maximum(Dm, eps) ** (p - 2.0)
        HA = p * (p - 1) * (np.diag(Wt.sum(1)) - Wt)
        HB = p * (p - 1) * np.diag(np.maximum(np.abs(u), eps) ** (p - 2.0))
        ref[:, l] = (HA / B - (A / B ** 2) * HB) @ eta[:, l]
    assert np.sum(U == 0.0) >= 2 * k
    got = oracle.hessvec(g, U, eta, p, eps=eps)
    for l in range(k):
        assert relerr(got[:, l], ref[:, l]) < 1e-12, l
