"""fp64 CPU oracle for the p-spectral-clustering hot path (arxiv 2605.26975).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  The product path (paper_2605_26975_b200) never
imports it, and it never imports the product path; both are fed by `plp_inputs` (seeded
generators with none of the method's arithmetic).

Edge-wise definitions (Eq. (1), Delta_p, EucGrad, Alg. 1, k-means, RCut) live in plain C
(`plp_oracle.c`, loops in the paper's order, fp64, -ffp-contract=off).  The tall-skinny Grassmann
steps use numpy library primitives (`dense.py`).  Every function is pinned by tests/test_oracle_*.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .dense import project, retract  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "plp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

OR_OK, OR_ERR_ARG, OR_ERR_DEGENERATE, OR_ERR_EMPTY = 0, 1, 4, 5


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
               "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
    return _lib


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def get_threads() -> int:
    return int(lib().oracle_get_threads())


# ----------------------------------------------------------------------------------------------
def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _csr(g):
    rp = np.ascontiguousarray(g.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(g.col, dtype=np.int32)
    w = _f64(g.w)
    return rp.size - 1, rp, col, w


def _rows(rows, n_rows):
    if rows is None:
        return 0, None, n_rows
    r = np.ascontiguousarray(rows, dtype=np.int64)
    return r.size, r, r.size


def _check(st, what):
    if st != OR_OK:
        raise RuntimeError(f"oracle {what} failed with status {st}")


D = ctypes.c_double
I64 = ctypes.c_int64


def phi(x: float, p: float) -> float:
    f = lib().oracle_phi
    f.restype = ctypes.c_double
    return float(f(D(x), D(p)))


def objective(g, U, p):
    """F_p(U) (Eq. (1)), with the per-column numerators A and p-norms B."""
    n_rows, rp, col, w = _csr(g)
    U = _f64(U)
    k = U.shape[1]
    A = np.zeros(k)
    B = np.zeros(k)
    F = np.zeros(1)
    _check(lib().oracle_objective(I64(n_rows), _p(rp), _p(col), _p(w), k, _p(U), D(p), _p(A), _p(B),
                                  _p(F)), "objective")
    return float(F[0]), A, B


def numerators(g, U, p):
    n_rows, rp, col, w = _csr(g)
    U = _f64(U)
    A = np.zeros(U.shape[1])
    _check(lib().oracle_numerators(I64(n_rows), _p(rp), _p(col), _p(w), U.shape[1], _p(U), D(p),
                                   _p(A)), "numerators")
    return A


def pnorms(U, p, n_rows=None):
    U = _f64(U)
    n_rows = U.shape[0] if n_rows is None else n_rows
    B = np.zeros(U.shape[1])
    _check(lib().oracle_pnorms(I64(n_rows), U.shape[1], _p(U), D(p), _p(B)), "pnorms")
    return B


def plaplacian(g, U, p, rows=None):
    n_rows, rp, col, w = _csr(g)
    U = _f64(U)
    k = U.shape[1]
    nsel, r, ns = _rows(rows, n_rows)
    L = np.zeros((ns, k))
    _check(lib().oracle_plaplacian(I64(n_rows), _p(rp), _p(col), _p(w), k, _p(U), D(p), I64(nsel),
                                   _p(r), _p(L)), "plaplacian")
    return L


def euc_grad(g, U, p, A=None, B=None, rows=None):
    n_rows, rp, col, w = _csr(g)
    U = _f64(U)
    k = U.shape[1]
    if A is None or B is None:
        _, A, B = objective(g, U, p)
    A, B = _f64(A), _f64(B)
    nsel, r, ns = _rows(rows, n_rows)
    G = np.zeros((ns, k))
    _check(lib().oracle_euc_grad(I64(n_rows), _p(rp), _p(col), _p(w), k, _p(U), D(p), _p(A), _p(B),
                                 I64(nsel), _p(r), _p(G)), "euc_grad")
    return G


def hessian_parts(g, U, p, eps, A, B, rows=None):
    """Alg. 1 inputs D[l] (n x k) and the off-diagonal values of H[l] (nnz_sel x k)."""
    n_rows, rp, col, w = _csr(g)
    U = _f64(U)
    k = U.shape[1]
    nsel, r, ns = _rows(rows, n_rows)
    sel = np.arange(n_rows) if r is None else r
    nnz_sel = int(np.sum(rp[sel + 1] - rp[sel]))
    Dd = np.zeros((ns, k))
    H = np.zeros((max(nnz_sel, 1), k))
    _check(lib().oracle_hessian_parts(I64(n_rows), _p(rp), _p(col), _p(w), k, _p(U), D(p), D(eps),
                                      _p(_f64(A)), _p(_f64(B)), I64(nsel), _p(r), _p(Dd), _p(H)),
           "hessian_parts")
    return Dd, H[:nnz_sel]


def euc_hessian_eta(g, Dd, H, eta, rows=None):
    """Alg. 1 literally: r = eta (.) D - vxm(eta, H)."""
    n_rows, rp, col, _ = _csr(g)
    eta = _f64(eta)
    k = eta.shape[1]
    nsel, r, ns = _rows(rows, n_rows)
    out = np.zeros((ns, k))
    Hc = _f64(H) if H.size else np.zeros((1, k))
    _check(lib().oracle_euc_hessian_eta(I64(n_rows), _p(rp), _p(col), k, _p(_f64(Dd)), _p(Hc),
                                        _p(eta), I64(nsel), _p(r), _p(out)), "euc_hessian_eta")
    return out


def dots_full(g, U, eta, p):
    n_rows, rp, col, w = _csr(g)
    U, eta = _f64(U), _f64(eta)
    k = U.shape[1]
    al, be = np.zeros(k), np.zeros(k)
    _check(lib().oracle_dots_full(I64(n_rows), _p(rp), _p(col), _p(w), k, _p(U), _p(eta), D(p),
                                  _p(al), _p(be)), "dots_full")
    return al, be


def rank_two(g, U, p, A, B, alpha, beta, r_in, rows=None):
    n_rows, rp, col, w = _csr(g)
    U = _f64(U)
    k = U.shape[1]
    nsel, r, ns = _rows(rows, n_rows)
    out = np.array(r_in, dtype=np.float64, copy=True)
    _check(lib().oracle_rank_two(I64(n_rows), _p(rp), _p(col), _p(w), k, _p(U), D(p), _p(_f64(A)),
                                 _p(_f64(B)), _p(_f64(alpha)), _p(_f64(beta)), I64(nsel), _p(r),
                                 _p(out)), "rank_two")
    return out


def hessvec(g, U, eta, p, eps=1e-9, mode="sparse", AB=None, rows=None, dots=None):
    """EucHessianEta: sparse mode = Alg. 1 with the parts of reading #5; full mode adds the
    rank-two terms of the exact Hessian of A/B (needs the global dots alpha, beta)."""
    if AB is None:
        _, A, B = objective(g, U, p)
    else:
        A, B = AB
    Dd, H = hessian_parts(g, U, p, eps, A, B, rows)
    r = euc_hessian_eta(g, Dd, H, eta, rows)
    if mode == "full":
        al, be = dots_full(g, U, eta, p) if dots is None else dots
        r = rank_two(g, U, p, A, B, al, be, r, rows)
    elif mode != "sparse":
        raise ValueError(mode)
    return r


def fgrad_hessvec(g, U, eta, p, eps=1e-9, mode="sparse", rows=None):
    """The benchmark unit's outputs: F, A, B, G, Hv (all rows, or the listed rows)."""
    F, A, B = objective(g, U, p)
    G = euc_grad(g, U, p, A, B, rows)
    Hv = hessvec(g, U, eta, p, eps, mode, (A, B), rows)
    return F, A, B, G, Hv


def kmeans(X, K, uniforms, restarts=10, max_iters=300, rel_tol=1e-9):
    X = _f64(X)
    n, dim = X.shape
    u = _f64(uniforms).reshape(-1)
    assert u.size >= restarts * K
    lab = np.zeros(n, dtype=np.int32)
    C = np.zeros((K, dim))
    sse = np.zeros(1)
    it = ctypes.c_int(0)
    _check(lib().oracle_kmeans(I64(n), dim, K, _p(X), _p(u), restarts, max_iters, D(rel_tol),
                               _p(lab), _p(C), _p(sse), ctypes.byref(it)), "kmeans")
    return lab, C, float(sse[0]), it.value


def rcut(g, labels, K):
    n_rows, rp, col, w = _csr(g)
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    cut = np.zeros(K)
    sizes = np.zeros(K, dtype=np.int64)
    rc = np.zeros(1)
    _check(lib().oracle_rcut(I64(n_rows), _p(rp), _p(col), _p(w), K, _p(lab), _p(cut), _p(sizes),
                             _p(rc)), "rcut")
    return float(rc[0]), cut, sizes
