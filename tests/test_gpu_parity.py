"""GPU-vs-oracle parity of the fused F / EucGrad / EucHessianEta path, through the C ABI.

Inputs are seeded and synthetic (plp_inputs), at sizes the oracle finishes in seconds that still
span many CTA tiles and a ragged tail.  Tolerance: 1e-9 relative (north star), per column,
normwise (tests/helpers.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from plp_inputs import (make_config, draw_U, draw_eta, path_graph, single_edge, random_graph,
                        streams, permute_graph, csr_from_undirected)
from helpers import TOL, colwise_relerr, scalar_relerr, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def plp():
    from paper_2605_26975_b200 import plp as mod
    return mod


@pytest.fixture(scope="module")
def ctx(plp):
    return plp.Context(0)


_GRAPHS = {}


def graph(name):
    if name not in _GRAPHS:
        if name == "C1":
            g = make_config("C1")
        elif name == "C2":
            g = make_config("C2")
        elif name == "C3s":
            g = make_config("C3", n=40 ** 3)
        elif name == "C4s":
            g = make_config("C4", n=20000)
        elif name == "C5s":
            from paper_2605_26975_b200 import plp as mod
            g0 = make_config("C5", n=100_000)
            g = permute_graph(g0, mod.rcm_order(g0.row_ptr, g0.col))
        elif name in ("C5t", "C3t", "C2t", "D16t"):
            from paper_2605_26975_b200 import plp as mod
            base = {"C5t": ("C5", 100_000), "C3t": ("C3", 40 ** 3), "C2t": ("C2", None),
                    "D16t": ("D16", None)}[name]
            g0 = make_config(base[0], n=base[1])
            g = permute_graph(g0, mod.tile_order(g0.row_ptr, g0.col))
        elif name == "P5":
            g = path_graph(5)
        elif name == "K2":
            g = single_edge(0.7)
        elif name == "iso":
            g = random_graph(streams(5)[0], 3000, avg_deg=1.0, connected=False, name="iso")
        else:
            raise KeyError(name)
        _GRAPHS[name] = g
    return _GRAPHS[name]


def run_gpu(plp, ctx, g, U, eta, p, mode, eps, ab_from_fgrad=True):
    dev = torch.device("cuda:0")
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=plp.VALIDATE_SYMMETRIC)
    Ut = torch.from_numpy(U).to(dev)
    Et = torch.from_numpy(eta).to(dev)
    F0, AB0, G0 = plp.fgrad(ctx, G, Ut, p)
    AB_in = AB0 if ab_from_fgrad else None
    F, ABo, Gr, Hv = plp.fgrad_hessvec(ctx, G, Ut, Et, p, AB_in=AB_in, mode=mode, eps=eps)
    torch.cuda.synchronize()
    return dict(F0=to_np(F0)[0], AB0=to_np(AB0), G0=to_np(G0), F=to_np(F)[0], AB=to_np(ABo),
                G=to_np(Gr), Hv=to_np(Hv))


def check(res, g, U, eta, p, mode, eps):
    F, A, B, Gr, Hv = oracle.fgrad_hessvec(g, U, eta, p, eps, "full" if mode == 1 else "sparse")
    k = U.shape[1]
    assert scalar_relerr(res["F0"], F) < TOL
    assert scalar_relerr(res["F"], F) < TOL
    assert scalar_relerr(res["AB0"][:k], A) < TOL and scalar_relerr(res["AB0"][k:], B) < TOL
    assert scalar_relerr(res["AB"][:k], A) < TOL and scalar_relerr(res["AB"][k:], B) < TOL
    e_g0 = colwise_relerr(res["G0"], Gr)
    e_g = colwise_relerr(res["G"], Gr)
    e_h = colwise_relerr(res["Hv"], Hv)
    assert e_g0 < TOL and e_g < TOL and e_h < TOL, (e_g0, e_g, e_h)
    return e_g, e_h


CASES = [
    ("C1", 3, 2.0), ("C1", 3, 1.8), ("C1", 3, 1.5), ("C1", 3, 1.2),
    ("C2", 2, 2.0), ("C2", 2, 1.1),
    ("C3s", 8, 1.5), ("C4s", 20, 2.0), ("C4s", 20, 1.2), ("C5s", 8, 1.2),
    # generic (table-driven) power and other rational exponents
    ("C1", 3, 1.37), ("C1", 4, 1.62), ("C1", 2, 1.05), ("C1", 6, 1.999), ("C1", 8, 1.4),
    ("C1", 8, 1.9), ("C1", 8, 1.3), ("C1", 8, 1.7), ("C1", 8, 1.6),
    # odd and extreme k
    ("C1", 1, 1.5), ("C1", 5, 1.2), ("C1", 7, 1.1), ("C1", 16, 1.5), ("C1", 32, 1.2),
    ("C1", 31, 2.0), ("C1", 12, 1.8), ("P5", 2, 1.5), ("K2", 1, 1.2), ("iso", 3, 1.5),
    # tile-ordered graphs (halo kernel: every neighbour row from shared memory)
    ("C5t", 8, 1.2), ("C5t", 8, 2.0), ("C5t", 8, 1.37), ("C5t", 8, 1.5), ("C5t", 4, 1.1),
    ("C5t", 16, 1.8), ("C3t", 8, 1.5), ("C2t", 2, 1.1), ("iso", 4, 1.2), ("C1", 20, 1.2),
    # the paper's workload shape: Delaunay graph of 2^16 uniform points (NEXT-3), tile order
    ("D16t", 8, 1.2), ("D16t", 4, 1.5), ("D16t", 8, 2.0),
    # k = 20 (C4's width): the ring-gather kernel -- isolated nodes (degree 0: padded batches),
    # a 5-node path (one partial pass), generic power
    ("iso", 20, 1.5), ("P5", 20, 1.2), ("C4s", 20, 1.37), ("C1", 20, 1.8),
]


@pytest.mark.parametrize("name,k,p", CASES)
def test_fused_sparse_parity(plp, ctx, name, k, p):
    g = graph(name)
    U = draw_U(g.n, k, seed=11)
    eta = draw_eta(g.n, k, seed=11)
    res = run_gpu(plp, ctx, g, U, eta, p, plp.HESS_SPARSE, 1e-9)
    check(res, g, U, eta, p, 0, 1e-9)


@pytest.mark.parametrize("name,k,p", [("C1", 3, 1.5), ("C2", 2, 1.1), ("C4s", 20, 1.2),
                                      ("C1", 5, 1.37), ("C1", 8, 2.0), ("C5t", 8, 1.2),
                                      ("C3t", 8, 1.37)])
def test_fused_full_parity(plp, ctx, name, k, p):
    g = graph(name)
    U = draw_U(g.n, k, seed=3)
    eta = draw_eta(g.n, k, seed=3)
    res = run_gpu(plp, ctx, g, U, eta, p, plp.HESS_FULL, 1e-9)
    check(res, g, U, eta, p, 1, 1e-9)


def test_ab_in_null_runs_objective_first(plp, ctx):
    g = graph("C1")
    U, eta = draw_U(g.n, 3, 4), draw_eta(g.n, 3, 4)
    res = run_gpu(plp, ctx, g, U, eta, 1.5, plp.HESS_SPARSE, 1e-9, ab_from_fgrad=False)
    check(res, g, U, eta, 1.5, 0, 1e-9)


@pytest.mark.parametrize("p", [1.5, 1.2, 1.37, 2.0])
@pytest.mark.parametrize("eps", [1e-9, 0.3])
@pytest.mark.parametrize("name,k", [("C1", 3), ("C5t", 4)])
def test_ties_zeros_and_cap(plp, ctx, p, eps, name, k):
    """Exact ties u_i = u_j and exact zeros u_i = 0 (reading #6): the cap decision is taken on the
    same IEEE |u_i - u_j| on both sides; eps = 0.3 puts many edges below the cap.  k = 3 runs the
    row kernel, k = 4 on a tile-ordered graph the halo kernel."""
    g = graph(name)
    rng = streams(8)[1]
    U = np.round(rng.standard_normal((g.n, k)) * 2.0) / 4.0  # many ties and zeros
    U[:, 0] += 0.01  # keep every column nonzero
    eta = draw_eta(g.n, k, 8)
    for mode in (0, 1):
        res = run_gpu(plp, ctx, g, U, eta, p, mode, eps)
        check(res, g, U, eta, p, mode, eps)


def test_out_of_fast_domain_differences(plp, ctx):
    """|u_i - u_j| below 2^-120 (but nonzero) or above 2^120 leaves the fast power domain: the
    row / slot is recomputed with libdevice and still matches the oracle."""
    for name, k in (("C1", 3), ("C5t", 4)):
        g = graph(name)
        U = draw_U(g.n, k, 21)
        U[:, 1] = (1.0 + np.arange(g.n) * 1e-2) * 1e-38  # |u_i - u_j| ~ 1e-40 < 2^-120
        U[:7, 0] *= 1e125  # a few huge entries
        eta = draw_eta(g.n, k, 21)
        res = run_gpu(plp, ctx, g, U, eta, 1.5, 0, 1e-300)
        check(res, g, U, eta, 1.5, 0, 1e-300)


ALT_KERNELS = {"rows": "PLP_EDGE_ROWS", "staged": "PLP_EDGE_STAGED"}


@pytest.mark.parametrize("kernel", sorted(ALT_KERNELS))
def test_parity_suite_with_alternative_kernel(kernel):
    """Re-runs this module's oracle-parity cases in a subprocess with the staged kernel forced
    (PLP_EDGE_STAGED=1, edge_staged.cuh) or the unstaged row kernel (PLP_EDGE_ROWS=1,
    edge_kernel.cuh), so every edge kernel, not only the default one, is held to the oracle."""
    if any(os.environ.get(v) for v in ALT_KERNELS.values()):
        pytest.skip("already an alternative-kernel run")
    env = dict(os.environ, **{ALT_KERNELS[kernel]: "1"})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.abspath(__file__), "-k",
                        "fused_sparse_parity or fused_full_parity or ties or out_of_fast or "
                        "deterministic or misaligned or chunk_fallback"], env=env, capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("kernel", sorted(ALT_KERNELS))
def test_default_and_alternative_kernels_agree(plp, ctx, tmp_path, kernel):
    """The same call with the default (halo) kernel and, in a subprocess, with the staged or the
    unstaged row kernel: within 1e-12 of each other (summation association only)."""
    if any(os.environ.get(v) for v in ALT_KERNELS.values()):
        pytest.skip("already an alternative-kernel run")
    g = graph("C5t")
    U, eta = draw_U(g.n, 8, 31), draw_eta(g.n, 8, 31)
    res = run_gpu(plp, ctx, g, U, eta, 1.2, 0, 1e-9)
    script = tmp_path / "alt.py"
    script.write_text(
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.abspath(__file__))!r})\n"
        "from test_gpu_parity import graph, run_gpu\n"
        "from paper_2605_26975_b200 import plp\n"
        "from plp_inputs import draw_U, draw_eta\n"
        "g = graph('C5t'); U, eta = draw_U(g.n, 8, 31), draw_eta(g.n, 8, 31)\n"
        "r = run_gpu(plp, plp.Context(0), g, U, eta, 1.2, 0, 1e-9)\n"
        f"np.savez({str(tmp_path / 'alt.npz')!r}, G=r['G'], Hv=r['Hv'], AB=r['AB'])\n")
    env = dict(os.environ, **{ALT_KERNELS[kernel]: "1"})
    subprocess.check_call([sys.executable, str(script)], env=env)
    z = np.load(tmp_path / "alt.npz")
    assert colwise_relerr(res["G"], z["G"]) < 1e-12
    assert colwise_relerr(res["Hv"], z["Hv"]) < 1e-12
    assert scalar_relerr(res["AB"], z["AB"]) < 1e-12


@pytest.mark.parametrize("k", [8, 4, 6])
def test_chunk_fallback_high_degree(plp, ctx, k):
    """Rows of degree ~150 (a chunk of 32 rows then exceeds the staged kernel's shared-memory slot,
    so those chunks read col / w from global memory) mixed with low-degree rows (staged chunks):
    both paths against the oracle."""
    rng = streams(77)[0]
    n = 4000
    pairs = set()
    for i in range(n):
        deg = 150 if (i // 32) % 3 == 0 else 4
        for j in rng.integers(0, n, size=deg // 2):
            if j != i:
                pairs.add((min(i, int(j)), max(i, int(j))))
    ij = np.array(sorted(pairs))
    w = rng.uniform(0.1, 1.0, size=len(ij))
    g = csr_from_undirected(n, ij[:, 0], ij[:, 1], w, name="hub")
    U, eta = draw_U(g.n, k, 9), draw_eta(g.n, k, 9)
    res = run_gpu(plp, ctx, g, U, eta, 1.2, 0, 1e-9)
    check(res, g, U, eta, 1.2, 0, 1e-9)


def test_misaligned_views_use_scalar_path(plp, ctx):
    g = graph("C1")
    k = 8
    U = draw_U(g.n, k, 5)
    eta = draw_eta(g.n, k, 5)
    dev = torch.device("cuda:0")
    big = torch.zeros(g.n * k + 1, dtype=torch.float64, device=dev)
    Ut = big[1:].view(g.n, k)
    Ut.copy_(torch.from_numpy(U))
    assert Ut.data_ptr() % 16 == 8
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    F0, AB0, _ = plp.fgrad(ctx, Gh, Ut, 1.2, want_grad=False)
    F, ABo, Gr, Hv = plp.fgrad_hessvec(ctx, Gh, Ut, torch.from_numpy(eta).to(dev), 1.2, AB_in=AB0)
    Fo, A, B, Gro, Hvo = oracle.fgrad_hessvec(g, U, eta, 1.2)
    assert colwise_relerr(to_np(Gr), Gro) < TOL and colwise_relerr(to_np(Hv), Hvo) < TOL
    assert scalar_relerr(to_np(F)[0], Fo) < TOL


def test_deterministic_bitwise(plp, ctx):
    g = graph("C5s")
    U, eta = draw_U(g.n, 8, 1), draw_eta(g.n, 8, 1)
    a = run_gpu(plp, ctx, g, U, eta, 1.2, 0, 1e-9)
    b = run_gpu(plp, ctx, g, U, eta, 1.2, 0, 1e-9)
    for key in a:
        assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key


def test_degenerate_zero_column_gives_nonfinite_F(plp, ctx):
    g = graph("C1")
    U = draw_U(g.n, 2, 2)
    U[:, 1] = 0.0
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    F, AB, _ = plp.fgrad(ctx, Gh, torch.from_numpy(U).cuda(), 1.5, want_grad=False)
    assert not np.isfinite(to_np(F)[0]) and to_np(AB)[3] == 0.0


def test_domain_errors(plp, ctx):
    g = graph("K2")
    Gh = plp.Graph(ctx, g.row_ptr, g.col, g.w)
    U = torch.ones(2, 1, dtype=torch.float64, device="cuda")
    for p in (1.0, 2.5, 0.5):
        with pytest.raises(plp.PlpError, match="PLP_ERR_DOMAIN"):
            plp.fgrad(ctx, Gh, U, p)
    U33 = torch.ones(2, 33, dtype=torch.float64, device="cuda")
    with pytest.raises(plp.PlpError, match="PLP_ERR_DOMAIN"):
        plp.fgrad(ctx, Gh, U33, 1.5)
    with pytest.raises(plp.PlpError, match="PLP_ERR_DOMAIN"):
        plp.hessvec(ctx, Gh, U, U, 1.5, torch.ones(2, dtype=torch.float64, device="cuda"), eps=0.0)
    with pytest.raises(plp.PlpError, match="PLP_ERR_GRAPH"):
        bad = g.w.copy()
        bad[0] = 0.0
        plp.Graph(ctx, g.row_ptr, g.col, bad)


@pytest.mark.parametrize("p", [2.0, 1.8, 1.5, 1.2, 1.1, 1.9, 1.37, 1.62, 1.01, 1.999, 1.25])
def test_power_policies_accuracy(plp, ctx, p):
    """The custom fp64 powers (pow64.cuh) against numpy's pow: relative error
    <= 4e-15 over 1e-12 .. 1e3, and the cap / rare-branch semantics."""
    rng = streams(9)[1]
    a = np.concatenate([10.0 ** rng.uniform(-12, 3, 200_000), [0.0, 1e-9, 5e-10, 1.0, 2.0]])
    eps = 1e-9
    s, t = plp.debug_pow(ctx, torch.from_numpy(a).cuda(), p, eps)
    s, t = to_np(s), to_np(t)
    s_ref = np.maximum(a, eps) ** (p - 2.0)
    t_ref = np.where(a > 0, a ** (p - 1.0), 0.0)
    es = np.max(np.abs(s - s_ref) / s_ref)
    nz = t_ref > 0
    et = np.max(np.abs(t[nz] - t_ref[nz]) / t_ref[nz])
    print(f"p={p}: max rel err s {es:.2e} t {et:.2e}")
    assert es < 1e-14 and et < 1e-14
    assert np.all(t[~nz] == 0.0)
