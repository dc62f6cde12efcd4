"""Pins of the oracle solver (oracle/solver.py: trust-region Newton + truncated CG on the Grassmann
manifold with p-continuation) against things other than itself: the textbook eigenvalue problem at
p = 2 (dense eigensolver), the SPEC's worked tCG examples, and the solver invariants of SPEC.md:369-374
(orthonormal iterates, monotone accepted F, non-negative model decrease, horizontal gradient)."""
import math

import numpy as np
import pytest
import scipy.sparse.csgraph as csgraph

import oracle
from oracle import solver as osol
from oracle import dense
from plp_inputs import path_graph, random_graph, streams, csr_from_undirected


def eig_sum(g, k):
    L = csgraph.laplacian(g.to_scipy()).toarray()
    return float(np.sum(np.linalg.eigvalsh(L)[:k]))


def test_tcg_zero_gradient_gives_zero_step():
    cfg = osol.default_cfg(4, 1)
    eta, Heta, it, status = osol.tcg(lambda x: x, np.zeros((4, 1)), None, 1.0, cfg)
    assert it == 0 and status == "interior" and not np.any(eta)


def test_tcg_identity_operator_gives_newton_step():
    """H = identity, delta >= ||g|| -> step = -g within 1e-12."""
    rng = streams(3)[0]
    g = rng.standard_normal((6, 2))
    cfg = osol.default_cfg(6, 2)
    eta, Heta, it, status = osol.tcg(lambda x: x, g, None, 10.0 * np.linalg.norm(g), cfg)
    assert status == "converged" and np.max(np.abs(eta + g)) < 1e-12


def test_tcg_negative_curvature_moves_to_boundary():
    """a 2 x 2 diagonal operator with a negative eigenvalue along the initial direction
    -> ||step|| = delta exactly, status negative curvature."""
    D = np.array([[-1.0], [2.0]])
    g = np.array([[1.0], [0.0]])
    cfg = osol.default_cfg(2, 1)
    eta, Heta, it, status = osol.tcg(lambda x: D * x, g, None, 0.7, cfg)
    assert status == "negative_curvature"
    assert abs(np.linalg.norm(eta) - 0.7) < 1e-14
    assert eta[0, 0] < 0  # descent direction


def test_tcg_model_decrease_nonnegative_and_bounded():
    rng = streams(4)[0]
    for trial in range(20):
        n = 8
        A = rng.standard_normal((n, n))
        H = A + A.T  # indefinite symmetric
        g = rng.standard_normal((n, 1))
        delta = rng.uniform(0.1, 3.0)
        cfg = osol.default_cfg(n, 1)
        eta, Heta, it, status = osol.tcg(lambda x: H @ x, g, None, delta, cfg)
        dec = -float(np.sum(g * eta)) - 0.5 * float(np.sum(eta * Heta))
        assert dec >= -1e-14
        assert np.linalg.norm(eta) <= delta * (1 + 1e-12)
        assert np.max(np.abs(Heta - H @ eta)) < 1e-10


def test_path3_p2_reaches_sum_of_two_smallest_eigenvalues():
    """path P3, k = 2, p = 2, random U0 -> F* = 1 (eigenvalues 0 and 1) within 1e-8."""
    g = path_graph(3)
    Z = streams(0)[1].standard_normal((3, 2))
    U, tr = osol.continuation_solve(g, Z, [2.0])
    assert abs(oracle.objective(g, U, 2.0)[0] - 1.0) < 1e-8


@pytest.mark.parametrize("seed,n,k", [(1, 60, 2), (2, 120, 4), (3, 200, 2), (4, 150, 4), (5, 90, 3)])
def test_p2_matches_dense_eigensolver(seed, n, k):
    """SPEC.md:348 / acceptance 4: at p = 2, F* = sum of the k smallest Laplacian eigenvalues."""
    g = random_graph(streams(seed)[0], n, avg_deg=5.0, connected=True)
    Z = streams(seed)[1].standard_normal((n, k))
    U, tr = osol.continuation_solve(g, Z, [2.0], grad_tol=1e-9)
    F = oracle.objective(g, U, 2.0)[0]
    assert abs(F - eig_sum(g, k)) < 1e-6 * max(1.0, abs(eig_sum(g, k)))


def test_solver_invariants_at_p_below_2():
    """iterates orthonormal within 1e-10, accepted F non-increasing at fixed p,
    and the returned gradient horizontal."""
    g = random_graph(streams(7)[0], 120, avg_deg=5.0, connected=True)
    k = 3
    Z = streams(7)[1].standard_normal((g.n, k))
    U, tr = osol.continuation_solve(g, Z, [2.0, 1.6, 1.3], max_outer=60)
    assert np.max(np.abs(U.T @ U - np.eye(k))) < 1e-10
    for p in (2.0, 1.6, 1.3):
        Fs = [r[2] for r in tr if r[0] == p and r[8]]
        assert all(b <= a + 1e-15 * abs(a) for a, b in zip(Fs, Fs[1:]))
    F, A, B = oracle.objective(g, U, 1.3)
    G = oracle.euc_grad(g, U, 1.3, A, B)
    grad = dense.project(U, G)
    assert np.max(np.abs(U.T @ grad)) < 1e-10


def test_continuation_improves_objective_on_ring_of_cliques():
    """SPEC.md:367 (shape of the example): on a ring of cliques, continuing to p_final lowers
    F_{p_final} below the p = 2 solution re-evaluated at p_final."""
    m, c = 5, 4
    ij, w = [], []
    for a in range(c):
        base = a * m
        for u in range(m):
            for v in range(u + 1, m):
                ij.append((base + u, base + v))
                w.append(1.0)
        ij.append((base + m - 1, ((a + 1) % c) * m))
        w.append(0.2)
    ij = np.array(ij)
    g = csr_from_undirected(m * c, ij[:, 0], ij[:, 1], np.array(w), name="ring")
    wins = 0
    for seed in range(6):
        Z = streams(seed)[1].standard_normal((g.n, c))
        U2, _ = osol.continuation_solve(g, Z, [2.0])
        Up, _ = osol.continuation_solve(g, Z, [2.0, 1.6, 1.3], max_outer=80)
        wins += oracle.objective(g, Up, 1.3)[0] <= oracle.objective(g, U2, 1.3)[0] * (1 + 1e-12)
    assert wins >= 5
