"""Pins of the oracle's k-means, RCut, projection and retraction (no GPU)."""
import math

import numpy as np
import pytest

import oracle
from plp_inputs import four_cycle, two_triangles, make_config, streams, draw_uniforms, path_graph


# ----------------------------------------------------------------------------------- k-means ---
def test_kmeans_1d_worked_example():
    X = np.array([[0.0], [0.1], [10.0], [10.1]])
    lab, C, sse, _ = oracle.kmeans(X, 2, draw_uniforms(10, 2, seed=3), restarts=10)
    assert lab[0] == lab[1] and lab[2] == lab[3] and lab[0] != lab[2]
    assert abs(sse - 0.01) < 1e-15
    assert sorted(C[:, 0].round(12)) == [0.05, 10.05]


def test_kmeans_identical_points():
    X = np.ones((6, 2))
    lab, C, sse, _ = oracle.kmeans(X, 2, draw_uniforms(3, 2, seed=1), restarts=3)
    assert sse == 0.0 and np.all(C == 1.0) and set(lab) <= {0, 1}


def brute_best_2partition(X):
    n = X.shape[0]
    best = math.inf
    for mask in range(1, 2 ** (n - 1)):
        a = np.array([(mask >> i) & 1 for i in range(n)], bool)
        s = 0.0
        for part in (X[a], X[~a]):
            s += np.sum((part - part.mean(0)) ** 2)
        best = min(best, s)
    return best


@pytest.mark.parametrize("seed", range(5))
def test_kmeans_exhaustive_n8(seed):
    X = streams(seed)[0].standard_normal((8, 2))
    _, _, sse, _ = oracle.kmeans(X, 2, draw_uniforms(50, 2, seed=seed), restarts=50)
    assert abs(sse - brute_best_2partition(X)) < 1e-12


def test_kmeans_fixed_point_and_blobs():
    pts = np.concatenate([np.array([[5.0 * math.cos(2 * math.pi * c / 3),
                                     5.0 * math.sin(2 * math.pi * c / 3)]]) for c in range(3)])
    rng = streams(0)[0]
    X = np.repeat(pts, 50, axis=0) + 0.3 * rng.standard_normal((150, 2))
    truth = np.repeat(np.arange(3), 50)
    lab, C, sse, _ = oracle.kmeans(X, 3, draw_uniforms(10, 3), restarts=10)
    # labels equal the generator's blobs up to permutation
    perm = {a: b for a, b in zip(lab, truth)}
    assert np.array_equal(np.vectorize(perm.get)(lab), truth)
    # fixed point: nearest-centroid assignment (ties lowest) and centroids are the means
    d = ((X[:, None, :] - C[None, :, :]) ** 2).sum(-1)
    assert np.array_equal(lab, np.argmin(d, axis=1))
    for c in range(3):
        assert np.allclose(C[c], X[lab == c].mean(0), rtol=0, atol=1e-14)
    assert abs(sse - d.min(1).sum()) < 1e-12 * sse


def test_kmeans_sse_nonincreasing():
    X = streams(4)[0].standard_normal((200, 3))
    u = draw_uniforms(1, 5, seed=4)
    prev = math.inf
    for it in range(0, 12):
        _, _, sse, _ = oracle.kmeans(X, 5, u, restarts=1, max_iters=it, rel_tol=0.0)
        assert sse <= prev + 1e-12
        prev = sse


def test_kmeans_seeding_rule():
    """k-means++ with supplied uniforms: centre 0 = floor(u0 n); with max_iters=0 the returned
    centroids are the seeds.  Points on a line make D^2 cumsum hand-checkable."""
    X = np.array([[0.0], [1.0], [2.0], [3.0]])
    u = np.array([[0.3, 0.5]])  # c0 = floor(1.2) = 1 -> D2 = [1,0,1,4], S=6, target 3 -> i=3
    lab, C, sse, _ = oracle.kmeans(X, 2, u, restarts=1, max_iters=0)
    assert C[0, 0] == 1.0 and C[1, 0] == 3.0
    assert list(lab) == [0, 0, 0, 1] and sse == 2.0  # point 2 ties (1 vs 1) -> lowest index


# -------------------------------------------------------------------------------------- RCut ---
def test_rcut_worked_examples():
    rc, cut, sizes = oracle.rcut(four_cycle(), np.array([0, 0, 1, 1]), 2)
    assert rc == 2.0 and list(cut) == [2.0, 2.0]
    rc, _, _ = oracle.rcut(two_triangles(), np.array([0, 0, 0, 1, 1, 1]), 2)
    assert rc == 0.0


def test_rcut_invariances_and_brute_force():
    g = make_config("C1", n=120)
    rng = streams(2)[0]
    lab = rng.integers(0, 4, g.n).astype(np.int32)
    rc, cut, sizes = oracle.rcut(g, lab, 4)
    perm = np.array([2, 0, 3, 1])
    rc2, _, _ = oracle.rcut(g, perm[lab], 4)
    assert abs(rc - rc2) < 1e-13 * rc
    W = g.to_scipy().toarray()
    ref = sum(W[np.ix_(lab == c, lab != c)].sum() / np.sum(lab == c) for c in range(4))
    assert abs(rc - ref) < 1e-12 * ref
    # cut(S) = cut(complement) for a bipartition
    lab2 = (lab >= 2).astype(np.int32)
    _, cut2, _ = oracle.rcut(g, lab2, 2)
    assert abs(cut2[0] - cut2[1]) < 1e-12 * cut2[0]


def test_rcut_path_graph_closed_form():
    # P_6 split in half: one cut edge of weight 1 -> 1/3 + 1/3
    rc, _, _ = oracle.rcut(path_graph(6), np.array([0, 0, 0, 1, 1, 1]), 2)
    assert abs(rc - 2.0 / 3.0) < 1e-15


# --------------------------------------------------------------------------- projection / QR ---
def rand_orthonormal(rng, n, k):
    Q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return Q


def test_projection_properties():
    rng = streams(5)[0]
    U = rand_orthonormal(rng, 300, 5)
    G = rng.standard_normal((300, 5))
    P = oracle.project(U, G)
    assert np.max(np.abs(U.T @ P)) < 1e-13
    assert np.max(np.abs(oracle.project(U, U @ rng.standard_normal((5, 5))))) < 1e-13
    assert np.max(np.abs(oracle.project(U, P) - P)) < 1e-13
    H = G - U @ (U.T @ G)
    assert np.max(np.abs(oracle.project(U, H) - H)) < 1e-13


def test_retraction_properties():
    rng = streams(6)[0]
    U = rand_orthonormal(rng, 400, 4)
    xi = oracle.project(U, 0.3 * rng.standard_normal((400, 4)))
    Q, R = oracle.retract(U, xi)
    assert np.max(np.abs(Q.T @ Q - np.eye(4))) < 1e-13
    assert np.max(np.abs(Q @ R - (U + xi))) < 1e-13
    assert np.all(np.diag(R) > 0) and np.allclose(np.tril(R, -1), 0)
    Q0, _ = oracle.retract(U * np.sign(np.diag(np.linalg.qr(U)[1]))[None, :], np.zeros_like(U))
    # xi = 0 -> U (for the representative with positive R diagonal)
    Us = U * np.sign(np.diag(np.linalg.qr(U)[1]))[None, :]
    assert np.max(np.abs(Q0 - Us)) < 1e-14
    # n = 2, k = 1: U = e1, xi = t e2 -> (e1 + t e2)/sqrt(1+t^2)
    t = 0.75
    Q1, _ = oracle.retract(np.array([[1.0], [0.0]]), np.array([[0.0], [t]]))
    assert np.allclose(Q1[:, 0], np.array([1.0, t]) / math.sqrt(1 + t * t), rtol=0, atol=1e-16)
    # uniqueness: equals Gram-Schmidt (Cholesky-QR) on a well-conditioned Y
    Y = U + xi
    Rc = np.linalg.cholesky(Y.T @ Y).T
    assert np.max(np.abs(Y @ np.linalg.inv(Rc) - Q)) < 1e-12
