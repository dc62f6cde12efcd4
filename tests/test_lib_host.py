"""CPU-only checks of libplp: the C-ABI library loads, exports every symbol include/plp.h declares,
and its host-side graph setup (validation, RCM, relabelling, partitioning, halo plans) is right.
No compute call touches a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest
import scipy.sparse as sp

from plp_inputs import (make_config, permute_graph, random_graph, streams, csr_from_undirected,
                        single_edge)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def plp():
    from paper_2605_26975_b200 import plp as mod
    return mod


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "plp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(plp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(plp):
    names = declared_symbols()
    assert len(names) >= 30
    lib = ctypes.CDLL(plp.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(plp.SYMBOLS) == names
    assert "sm_100a" in plp.version()


def test_library_is_sm100a_only(plp):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", plp.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


def test_validate_accepts_generator_graphs(plp):
    for g in (make_config("C1"), make_config("C3", n=20 ** 3), single_edge()):
        plp.validate_csr(g.row_ptr, g.col, g.w, symmetric=True)


def test_validate_rejects_bad_graphs(plp):
    g = make_config("C1", n=60)
    bad_w = g.w.copy()
    bad_w[5] = -1.0
    with pytest.raises(plp.PlpError, match="PLP_ERR_GRAPH"):
        plp.validate_csr(g.row_ptr, g.col, bad_w)
    asym = g.w.copy()
    asym[0] *= 1.0000001
    with pytest.raises(plp.PlpError, match="asymmetric"):
        plp.validate_csr(g.row_ptr, g.col, asym, symmetric=True)
    # diagonal entry
    rp = np.array([0, 2, 3], np.int64)
    col = np.array([0, 1, 0], np.int32)
    with pytest.raises(plp.PlpError, match="diagonal"):
        plp.validate_csr(rp, col, np.ones(3), symmetric=False)
    # unsorted / duplicate columns
    g2 = random_graph(streams(1)[0], 20)
    c2 = g2.col.copy()
    r = int(np.argmax(np.diff(g2.row_ptr)))
    s, e = g2.row_ptr[r], g2.row_ptr[r + 1]
    c2[s:e] = c2[s:e][::-1]
    with pytest.raises(plp.PlpError, match="strictly increasing"):
        plp.validate_csr(g2.row_ptr, c2, g2.w, symmetric=False)


def bandwidth(g):
    rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    return int(np.max(np.abs(rows - g.col)))


def test_rcm_is_a_deterministic_bandwidth_reducing_permutation(plp):
    g = make_config("C5", n=20000)
    perm = plp.rcm_order(g.row_ptr, g.col)
    assert np.array_equal(np.sort(perm), np.arange(g.n))
    assert np.array_equal(perm, plp.rcm_order(g.row_ptr, g.col))
    gp = permute_graph(g, perm)
    assert bandwidth(gp) < bandwidth(g) / 20
    # comparable to scipy's RCM (same algorithm family)
    from scipy.sparse.csgraph import reverse_cuthill_mckee
    ps = reverse_cuthill_mckee(g.to_scipy(), symmetric_mode=True)
    assert bandwidth(gp) < 2 * bandwidth(permute_graph(g, ps))


def test_rcm_handles_disconnected_and_isolated(plp):
    g = csr_from_undirected(7, [0, 1, 4], [1, 2, 5], [1.0, 1.0, 1.0], "parts")
    perm = plp.rcm_order(g.row_ptr, g.col)
    assert np.array_equal(np.sort(perm), np.arange(7))


def test_permute_csr_matches_scipy(plp):
    g = make_config("C1", n=300)
    perm = streams(3)[0].permutation(g.n)
    rp, col, w = plp.permute_csr(g.row_ptr, g.col, g.w, perm)
    ref = permute_graph(g, perm)
    assert np.array_equal(rp, ref.row_ptr) and np.array_equal(col, ref.col) and np.array_equal(w, ref.w)
    plp.validate_csr(rp, col, w, symmetric=True)


def test_partition_rows_balanced(plp):
    g = make_config("C4", n=5000)
    for parts in (1, 2, 4, 8):
        b = plp.partition_rows(g.row_ptr, parts, 32 * 20, 12)
        assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b) > 0)
        cost = 32 * 20 * np.diff(b) + 12 * np.diff(g.row_ptr[b])
        assert cost.max() / cost.mean() < 1.01


def test_halo_plan_matches_brute_force(plp):
    g = make_config("C1", n=400)
    r0, r1 = 120, 300
    halo, rp_loc, col_loc = plp.halo_plan(g.row_ptr, g.col, r0, r1)
    cols = g.col[g.row_ptr[r0]:g.row_ptr[r1]].astype(np.int64)
    ref = np.unique(cols[(cols < r0) | (cols >= r1)])
    assert np.array_equal(halo, ref)
    ext = np.concatenate([np.arange(r0, r1), halo])
    assert np.array_equal(ext[col_loc], cols)  # local ids map back to the global columns
    assert np.array_equal(rp_loc, g.row_ptr[r0:r1 + 1] - g.row_ptr[r0])


def test_halo_peer_slices_are_contiguous(plp):
    """Halo rows owned by one peer form one contiguous slice (received in place, plp.h)."""
    g = make_config("C5", n=30000)
    perm = plp.rcm_order(g.row_ptr, g.col)
    rp, col, w = plp.permute_csr(g.row_ptr, g.col, g.w, perm)
    b = plp.partition_rows(rp, 4, 256, 12)
    for r in range(4):
        halo, _, _ = plp.halo_plan(rp, col, b[r], b[r + 1])
        owner = np.searchsorted(b, halo, side="right") - 1
        assert np.all(np.diff(owner) >= 0)
        assert np.all(owner != r)
