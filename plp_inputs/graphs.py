"""Synthetic graph and input generators (BASELINE.json configs C1-C5 + tiny closed-form graphs).

Conventions (SURVEY.md §8(d) "Generator conventions"):
  * Euclidean distances in fp64, self excluded.
  * Union symmetrisation: edge {i,j} if j in kNN(i) or i in kNN(j).  d^2 is computed ONCE per
    undirected edge, so w_ij == w_ji bitwise.
  * Weights w = exp(-d^2 / (2 * median d^2)), median over the undirected edge set (numpy median).
  * Node order = generation order.  Reordering (RCM) is the library's job (plp_create_graph).
  * Random streams: numpy SeedSequence(seed).spawn(4) -> PCG64 streams for
    {points+graph, U, eta, k-means uniforms}.
Storage: CSR with both triangles, int64 row_ptr[n+1], int32 col[nnz] (sorted, unique per row),
float64 w[nnz]; zero diagonal; w > 0.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import scipy.sparse as sp
from scipy.spatial import cKDTree


@dataclasses.dataclass
class Graph:
    name: str
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col: np.ndarray  # int32 [nnz]
    w: np.ndarray  # float64 [nnz]
    labels: np.ndarray | None = None  # generator's ground-truth blob labels (sanity only)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_scipy(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.w, self.col, self.row_ptr), shape=(self.n, self.n))


def streams(seed: int = 0):
    """Four independent PCG64 generators: points+graph, U, eta, k-means uniforms."""
    ss = np.random.SeedSequence(seed).spawn(4)
    return [np.random.Generator(np.random.PCG64(s)) for s in ss]


# ----------------------------------------------------------------------------------------------
# CSR construction
# ----------------------------------------------------------------------------------------------
def csr_from_undirected(n: int, i: np.ndarray, j: np.ndarray, wu: np.ndarray, name: str,
                        labels=None) -> Graph:
    """Both triangles from a list of unique undirected edges (i != j); w_ij == w_ji bitwise."""
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    wu = np.asarray(wu, dtype=np.float64)
    assert np.all(i != j)
    rows = np.concatenate([i, j])
    cols = np.concatenate([j, i])
    vals = np.concatenate([wu, wu])
    m = sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
    m.sort_indices()
    assert m.nnz == rows.size, "duplicate undirected edges passed to csr_from_undirected"
    return Graph(name, n, m.indptr.astype(np.int64), m.indices.astype(np.int32),
                 m.data.astype(np.float64), labels)


def _unique_undirected(i: np.ndarray, j: np.ndarray, n: int):
    a = np.minimum(i, j).astype(np.int64)
    b = np.maximum(i, j).astype(np.int64)
    keep = a != b
    key = np.unique(a[keep] * n + b[keep])
    return key // n, key % n


def knn_graph(pts: np.ndarray, knn: int, name: str, labels=None, workers: int = -1) -> Graph:
    """Union-symmetrised kNN graph with Gaussian weights exp(-d^2/(2 median d^2))."""
    n = pts.shape[0]
    tree = cKDTree(pts)
    _, idx = tree.query(pts, k=knn + 1, workers=workers)
    src = np.repeat(np.arange(n, dtype=np.int64), knn + 1)
    dst = idx.reshape(-1).astype(np.int64)
    a, b = _unique_undirected(src, dst, n)  # drops self pairs
    diff = pts[a] - pts[b]
    d2 = np.einsum("ij,ij->i", diff, diff)  # once per undirected edge
    sigma2 = float(np.median(d2))
    wu = np.exp(-d2 / (2.0 * sigma2))
    # exp of a finite negative number can underflow to 0 only for absurd d2; guard w > 0
    wu = np.maximum(wu, np.finfo(np.float64).tiny)
    return csr_from_undirected(n, a, b, wu, name, labels)


# ----------------------------------------------------------------------------------------------
# Point clouds (BASELINE.json configs)
# ----------------------------------------------------------------------------------------------
def blobs_2d(rng, sizes=(334, 333, 333), radius=5.0, sigma=1.0):
    """C1: 3 isotropic Gaussian blobs, means at angles 0, 2pi/3, 4pi/3 on a radius-5 circle."""
    pts, lab = [], []
    for c, m in enumerate(sizes):
        ang = 2.0 * math.pi * c / len(sizes)
        mu = np.array([radius * math.cos(ang), radius * math.sin(ang)])
        pts.append(mu + sigma * rng.standard_normal((m, 2)))
        lab.append(np.full(m, c, dtype=np.int32))
    return np.concatenate(pts), np.concatenate(lab)


def two_moons(rng, n=100_000, noise=0.1):
    """C2: outer arc (cos t, sin t), inner arc (1-cos t, 1/2 - sin t), t ~ U[0, pi], + N(0, noise^2)."""
    h = n // 2
    t1 = rng.uniform(0.0, math.pi, h)
    t2 = rng.uniform(0.0, math.pi, n - h)
    outer = np.stack([np.cos(t1), np.sin(t1)], axis=1)
    inner = np.stack([1.0 - np.cos(t2), 0.5 - np.sin(t2)], axis=1)
    pts = np.concatenate([outer, inner]) + noise * rng.standard_normal((n, 2))
    lab = np.concatenate([np.zeros(h, np.int32), np.ones(n - h, np.int32)])
    return pts, lab


def gmm(rng, n=1_000_000, dim=10, clusters=20, sigma=1.0, box=10.0):
    """C4: equal-size Gaussian mixture, means ~ U[-box, box]^dim."""
    means = rng.uniform(-box, box, (clusters, dim))
    per = n // clusters
    lab = np.repeat(np.arange(clusters, dtype=np.int32), per)
    lab = np.concatenate([lab, np.full(n - lab.size, clusters - 1, np.int32)])
    pts = means[lab] + sigma * rng.standard_normal((n, dim))
    return pts, lab


def uniform_square(rng, n=8_388_608):
    """C5: uniform points in [0,1]^2 (stand-in for SuiteSparse delaunay_n23)."""
    return rng.uniform(0.0, 1.0, (n, 2))


def grid3d_longrange(rng, side=128, frac=0.01, w_long=0.1, name="C3"):
    """C3: side^3 grid in natural order i = x + side*(y + side*z), 7-point-stencil unit weights,
    plus round(frac * #stencil edges) uniform node pairs of weight w_long (self pairs and
    duplicates -- among themselves or with stencil edges -- dropped)."""
    n = side ** 3
    idx = np.arange(n, dtype=np.int64).reshape(side, side, side)  # [z, y, x]
    e_i, e_j = [], []
    for ax in range(3):
        sl_a = [slice(None)] * 3
        sl_b = [slice(None)] * 3
        sl_a[ax] = slice(0, side - 1)
        sl_b[ax] = slice(1, side)
        e_i.append(idx[tuple(sl_a)].reshape(-1))
        e_j.append(idx[tuple(sl_b)].reshape(-1))
    si = np.concatenate(e_i)
    sj = np.concatenate(e_j)
    n_stencil = si.size
    n_long = int(round(frac * n_stencil))
    pr = rng.integers(0, n, size=(n_long, 2), dtype=np.int64)
    a = np.minimum(pr[:, 0], pr[:, 1])
    b = np.maximum(pr[:, 0], pr[:, 1])
    keep = a != b
    a, b = a[keep], b[keep]
    lkey = np.unique(a * n + b)
    skey = np.minimum(si, sj) * n + np.maximum(si, sj)
    lkey = lkey[~np.isin(lkey, skey)]
    ii = np.concatenate([si, lkey // n])
    jj = np.concatenate([sj, lkey % n])
    ww = np.concatenate([np.ones(n_stencil), np.full(lkey.size, w_long)])
    return csr_from_undirected(n, ii, jj, ww, name)


# ----------------------------------------------------------------------------------------------
# Tiny closed-form graphs (for oracle pins)
# ----------------------------------------------------------------------------------------------
def path_graph(m: int, w: float = 1.0) -> Graph:
    i = np.arange(m - 1)
    return csr_from_undirected(m, i, i + 1, np.full(m - 1, w), f"P{m}")


def cycle_graph(m: int, w: float = 1.0) -> Graph:
    i = np.arange(m)
    return csr_from_undirected(m, i, (i + 1) % m, np.full(m, w), f"C{m}")


def single_edge(w: float = 1.0) -> Graph:
    return csr_from_undirected(2, [0], [1], [w], "K2")


def four_cycle() -> Graph:
    return cycle_graph(4)


def two_triangles() -> Graph:
    return csr_from_undirected(6, [0, 1, 2, 3, 4, 5], [1, 2, 0, 4, 5, 3], np.ones(6), "2xK3")


def random_graph(rng, n: int, avg_deg: float = 4.0, connected: bool = True, name="rand") -> Graph:
    """Erdos-Renyi-like random weighted graph (+ a path backbone when connected=True)."""
    m = int(avg_deg * n / 2)
    pr = rng.integers(0, n, size=(m, 2))
    ii, jj = [pr[:, 0]], [pr[:, 1]]
    if connected:
        perm = rng.permutation(n)
        ii.append(perm[:-1])
        jj.append(perm[1:])
    a, b = _unique_undirected(np.concatenate(ii), np.concatenate(jj), n)
    wu = rng.uniform(0.1, 1.0, a.size)
    return csr_from_undirected(n, a, b, wu, name)


def delaunay_graph(rng, n: int, name: str = "D") -> Graph:
    """Stand-in for the paper's SuiteSparse delaunay_n<r> graphs (SURVEY.md §8(f)
    NEXT-3): the Delaunay triangulation (scipy.spatial.Delaunay, Qhull) of n uniform points in the
    unit square, every triangle side an undirected edge, unit weights (the SuiteSparse matrices are
    patterns).  nnz ~ 6 n stored nonzeros, planar, connected."""
    from scipy.spatial import Delaunay
    pts = uniform_square(rng, n)
    tri = Delaunay(pts).simplices.astype(np.int64)
    a = np.concatenate([tri[:, 0], tri[:, 1], tri[:, 2]])
    b = np.concatenate([tri[:, 1], tri[:, 2], tri[:, 0]])
    a, b = _unique_undirected(a, b, n)
    return csr_from_undirected(n, a, b, np.ones(a.size), name)


# ----------------------------------------------------------------------------------------------
# Configs
# ----------------------------------------------------------------------------------------------
CONFIGS = {
    # name: (k, p schedule)
    "C1": dict(k=3, p=(2.0, 1.8, 1.5, 1.2)),
    "C2": dict(k=2, p=(2.0, 1.1)),
    "C3": dict(k=8, p=(1.5,)),
    "C4": dict(k=20, p=(2.0, 1.2)),
    "C5": dict(k=8, p=(1.2,)),
    # the paper's workload shape (NEXT-3): Delaunay graphs of 2^r uniform points, unit weights
    "D16": dict(k=4, p=(2.0, 1.5, 1.2)),
    "D20": dict(k=4, p=(2.0, 1.5, 1.2)),
    "D23": dict(k=8, p=(1.2,)),
}


def make_config(name: str, seed: int = 0, n: int | None = None) -> Graph:
    """Build the graph of config `name` (optionally at a reduced node count `n` for parity tests;
    the shape recipe -- dimension, kNN degree, weighting, structure -- is unchanged)."""
    rng = streams(seed)[0]
    if name == "C1":
        sizes = (334, 333, 333) if n is None else (n - 2 * (n // 3), n // 3, n // 3)
        pts, lab = blobs_2d(rng, sizes)
        return knn_graph(pts, 10, "C1", lab)
    if name == "C2":
        pts, lab = two_moons(rng, 100_000 if n is None else n)
        return knn_graph(pts, 10, "C2", lab)
    if name == "C3":
        side = 128 if n is None else max(4, int(round(n ** (1.0 / 3.0))))
        return grid3d_longrange(rng, side)
    if name == "C4":
        pts, lab = gmm(rng, 1_000_000 if n is None else n)
        return knn_graph(pts, 15, "C4", lab)
    if name == "C5":
        pts = uniform_square(rng, 8_388_608 if n is None else n)
        return knn_graph(pts, 6, "C5")
    if name.startswith("D") and name[1:].isdigit():  # D<r>: delaunay_n<r> shape, 2^r points
        r = int(name[1:])
        return delaunay_graph(rng, (1 << r) if n is None else n, name)
    raise KeyError(name)


def draw_U(n: int, k: int, seed: int = 0) -> np.ndarray:
    """U iid N(0,1), fp64, node-major n x k."""
    return streams(seed)[1].standard_normal((n, k))


def draw_eta(n: int, k: int, seed: int = 0) -> np.ndarray:
    return streams(seed)[2].standard_normal((n, k))


def draw_uniforms(restarts: int, clusters: int, seed: int = 0) -> np.ndarray:
    """k-means++ seeding uniforms in [0,1): restarts x clusters."""
    return streams(seed)[3].uniform(0.0, 1.0, (restarts, clusters))


# ----------------------------------------------------------------------------------------------
# Helpers for tests
# ----------------------------------------------------------------------------------------------
def validate_graph(g: Graph) -> None:
    """Graph invariants: symmetric bitwise, zero diagonal, w > 0, sorted cols."""
    rp, c, w = g.row_ptr, g.col, g.w
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == c.size == w.size
    assert np.all(w > 0)
    rows = np.repeat(np.arange(g.n), np.diff(rp))
    assert np.all(rows != c)
    for i in range(min(g.n, 1_000_000)):
        seg = c[rp[i]:rp[i + 1]]
        if seg.size > 1:
            assert np.all(np.diff(seg) > 0)
        if i > 2000:
            break
    m = g.to_scipy()
    d = (m - m.T)
    assert d.nnz == 0 or np.all(d.data == 0)


def permute_graph(g: Graph, perm: np.ndarray) -> Graph:
    """Relabel nodes: new node i is old node perm[i] (perm = new -> old)."""
    perm = np.asarray(perm, dtype=np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    m = g.to_scipy()[perm][:, perm].tocsr()
    m.sort_indices()
    lab = None if g.labels is None else g.labels[perm]
    return Graph(g.name + "_perm", g.n, m.indptr.astype(np.int64), m.indices.astype(np.int32),
                 m.data.astype(np.float64), lab)
