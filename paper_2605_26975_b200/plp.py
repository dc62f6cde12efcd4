"""Thin Python binding of libplp (include/plp.h): argument marshalling only.

Every computation runs in libplp's sm_100a kernels; torch is used for device memory and streams.
There is no fallback: if libplp.so is missing or fails to load, importing this module raises.
Function names mirror the C ABI without the `plp_` prefix.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PLP_LIB") or os.path.join(_HERE, "libplp.so")  # PLP_LIB: tuning variants

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libplp.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; "
                      f"g.build()'` (no CPU fallback exists)")
_lib = ctypes.CDLL(LIB_PATH)

PLP_OK = 0
STATUS = {0: "PLP_OK", 1: "PLP_ERR_ARG", 2: "PLP_ERR_SHAPE", 3: "PLP_ERR_DOMAIN", 4: "PLP_ERR_GRAPH",
          5: "PLP_ERR_DEGENERATE", 6: "PLP_ERR_RANK", 7: "PLP_ERR_NONFINITE", 8: "PLP_ERR_CUDA",
          9: "PLP_ERR_OOM", 10: "PLP_ERR_EMPTY", 11: "PLP_ERR_NCCL"}
HESS_SPARSE, HESS_FULL = 0, 1
U_HALO_CURRENT = 16  # PLP_U_HALO_CURRENT: OR into mode when U's halo rows are already exchanged
VALIDATE, VALIDATE_SYMMETRIC = 1, 2

_lib.plp_last_error.restype = ctypes.c_char_p
_lib.plp_version.restype = ctypes.c_char_p
_lib.plp_last_edge_kernel.restype = ctypes.c_char_p

C_I64 = ctypes.c_int64
C_D = ctypes.c_double
VP = ctypes.c_void_p

# the exported symbol set (tests check every name declared in include/plp.h is exported)
SYMBOLS = [
    "plp_last_error", "plp_version", "plp_ctx_create", "plp_ctx_set_stream", "plp_ctx_destroy",
    "plp_ctx_info", "plp_validate_csr", "plp_rcm_order", "plp_permute_csr", "plp_partition_rows",
    "plp_halo_plan", "plp_create_graph", "plp_graph_info", "plp_destroy_graph", "plp_fgrad",
    "plp_hessvec", "plp_fgrad_hessvec", "plp_edge_pass", "plp_full_epilogue",
    "plp_objective_from_ab", "plp_gram", "plp_project", "plp_apply_sub", "plp_retract",
    "plp_cholesky", "plp_apply_rinv", "plp_dot", "plp_axpby", "plp_gather_rows", "plp_kmeans", "plp_kmeans_dist",
    "plp_rcut", "plp_debug_pow", "plp_tile_order", "plp_last_edge_kernel", "plp_halo_tile_rows", "plp_tcg_init",
    "plp_tcg_run", "plp_tcg_graph_create", "plp_tcg_graph_launch", "plp_tcg_graph_nodes",
    "plp_tcg_graph_destroy", "plp_get_nccl_unique_id", "plp_ctx_comm_info", "plp_allreduce_sum",
    "plp_create_graph_dist", "plp_graph_dist_info", "plp_halo_exchange", "plp_dist_recv_plan",
]
TCG_STATUS = {0: "running", 1: "boundary", 2: "negative_curvature", 3: "converged", 4: "maxiter",
              5: "interior"}
TILE_ROWS = 80  # PLP_TILE_ROWS in include/plp.h: plp_tile_order's default BFS tile
HALO_TILE = int(_lib.plp_halo_tile_rows())  # PLP_HALO_TILE: tile_order's default tile size
TCG_SCAL_LEN = 4160  # PLP_TCG_SCAL_LEN in include/plp.h


def last_edge_kernel() -> str:
    """plp_last_edge_kernel(): the last edge kernel launched (diagnostics)."""
    return _lib.plp_last_edge_kernel().decode()


class PlpError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.plp_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")


def _ck(st: int, where: str) -> None:
    if st != PLP_OK:
        raise PlpError(st, where)


def version() -> str:
    return _lib.plp_version().decode()


# ------------------------------------------------------------------------------------------------
# marshalling helpers
# ------------------------------------------------------------------------------------------------
def _dev(t, name, dtype=torch.float64, shape=None, nullable=False):
    if t is None:
        if nullable:
            return VP(0)
        raise ValueError(f"{name} is required")
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    return VP(t.data_ptr())


def _host(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a, VP(a.ctypes.data)


class Context:
    """plp_ctx: device workspaces + the CUDA stream work is enqueued on (torch's current stream
    unless given).  rank / world / nccl_id: a collective context (one process per GPU; nccl_id =
    plp_get_nccl_unique_id() from rank 0, broadcast by the caller -- see `Context.distributed`)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None, rank: int = 0,
                 world: int = 1, nccl_id: bytes | None = None):
        self.device = device
        torch.cuda.set_device(device)
        s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        self.rank, self.world = rank, world
        h = VP()
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        _ck(_lib.plp_ctx_create(device, VP(s.cuda_stream), int(rank), int(world),
                                idbuf if idbuf is not None else VP(0), ctypes.byref(h)), "plp_ctx_create")
        self.h = h
        self.scratch = {}

    @classmethod
    def distributed(cls, device: int, stream=None, group=None):
        """Collective context over torch.distributed's default group: rank 0 draws the NCCL id,
        torch broadcasts it (the only use of torch.distributed: plumbing), every rank creates its
        communicator inside libplp."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [get_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(device, stream, rank, world, obj[0])

    def comm_info(self):
        r, w, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _ck(_lib.plp_ctx_comm_info(self.h, ctypes.byref(r), ctypes.byref(w), ctypes.byref(c)), "plp_ctx_comm_info")
        return r.value, w.value, bool(c.value)

    def set_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        _ck(_lib.plp_ctx_set_stream(self.h, VP(stream.cuda_stream)), "plp_ctx_set_stream")

    def info(self):
        a, b = ctypes.c_int(), ctypes.c_int()
        _ck(_lib.plp_ctx_info(self.h, ctypes.byref(a), ctypes.byref(b)), "plp_ctx_info")
        return a.value, b.value

    def close(self):
        if getattr(self, "h", None):
            _lib.plp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """plp_graph: a device CSR (rows [0, n_rows), columns indexing n_cols rows of U/eta)."""

    def __init__(self, ctx: Context, row_ptr, col, w, n_cols: int | None = None, flags: int = VALIDATE):
        rp, rpp = _host(row_ptr, np.int64)
        c, cp = _host(col, np.int32)
        ww, wp = _host(w, np.float64)
        self.n_rows = rp.size - 1
        self.n_cols = self.n_rows if n_cols is None else int(n_cols)
        self.nnz = int(rp[-1])
        self.ctx = ctx
        h = VP()
        _ck(_lib.plp_create_graph(ctx.h, C_I64(self.n_rows), C_I64(self.n_cols), rpp, cp, wp,
                                  ctypes.c_uint32(flags), ctypes.byref(h)), "plp_create_graph")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _lib.plp_destroy_graph(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistGraph(Graph):
    """plp_create_graph_dist: this rank's rows [row_begin, row_end) of an n_global-node graph (host
    CSR of the owned rows, GLOBAL column ids).  Dense arrays of the graph have n_cols = n_own +
    n_halo rows (halo slots filled by the collective calls); outputs have n_own rows."""

    def __init__(self, ctx: Context, n_global: int, row_begin: int, row_end: int, row_ptr, col, w,
                 flags: int = VALIDATE):
        rp, rpp = _host(row_ptr, np.int64)
        c, cp = _host(col, np.int32)
        ww, wp = _host(w, np.float64)
        self.ctx = ctx
        h = VP()
        _ck(_lib.plp_create_graph_dist(ctx.h, C_I64(n_global), C_I64(row_begin), C_I64(row_end), rpp, cp, wp,
                                       ctypes.c_uint32(flags), ctypes.byref(h)), "plp_create_graph_dist")
        self.h = h
        a, b, c2, d = C_I64(), C_I64(), C_I64(), C_I64()
        _ck(_lib.plp_graph_dist_info(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c2), ctypes.byref(d)),
            "plp_graph_dist_info")
        self.n_rows, self.n_halo, self.row_begin, self.send_rows = a.value, b.value, c2.value, d.value
        self.n_cols = self.n_rows + self.n_halo
        self.row_end = self.row_begin + self.n_rows
        self.n_global = int(n_global)
        self.nnz = int(rp[-1] - rp[0])


def get_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _ck(_lib.plp_get_nccl_unique_id(buf), "plp_get_nccl_unique_id")
    return buf.raw


def allreduce_sum(ctx: Context, x):
    """In-place sum over the ranks of a device fp64 tensor (plp_allreduce_sum)."""
    _ck(_lib.plp_allreduce_sum(ctx.h, _dev(x, "x"), C_I64(x.numel())), "plp_allreduce_sum")
    return x


def halo_exchange(ctx: Context, g: Graph, X):
    """Fill the halo rows [n_own, n_cols) of X (n_cols x ..., any dtype with rows of 4k bytes)."""
    rb = X[0].numel() * X.element_size() if X.dim() > 1 else X.element_size()
    _ck(_lib.plp_halo_exchange(ctx.h, g.h, int(rb), VP(X.data_ptr())), "plp_halo_exchange")
    return X


def dist_recv_plan(bounds, halo):
    """Host part of the halo plan (no GPU): per rank q the (offset, count) slice of the sorted halo
    it owns, from the ranks' row bounds."""
    b, bp = _host(bounds, np.int64)
    h, hp = _host(halo, np.int64)
    world = b.size - 1
    off = np.zeros(world, np.int64)
    cnt = np.zeros(world, np.int64)
    _ck(_lib.plp_dist_recv_plan(int(world), bp, C_I64(h.size), hp, VP(off.ctypes.data), VP(cnt.ctypes.data)),
        "plp_dist_recv_plan")
    return off, cnt


def _empty(ctx, *shape):
    return torch.empty(*shape, dtype=torch.float64, device=f"cuda:{ctx.device}")


# ------------------------------------------------------------------------------------------------
# F_p, EucGrad, EucHessianEta
# ------------------------------------------------------------------------------------------------
def fgrad(ctx: Context, g: Graph, U, p: float, G=None, F=None, AB=None, want_grad: bool = True):
    """F (device [1]), AB (device [2k]) and, if want_grad, G (device n x k)."""
    k = U.shape[1]
    _dev(U, "U", shape=(g.n_cols, k))
    F = _empty(ctx, 1) if F is None else F
    AB = _empty(ctx, 2 * k) if AB is None else AB
    if want_grad and G is None:
        G = _empty(ctx, g.n_rows, k)
    _ck(_lib.plp_fgrad(ctx.h, g.h, k, _dev(U, "U"), C_D(p), _dev(F, "F", shape=(1,)),
                       _dev(AB, "AB", shape=(2 * k,)),
                       _dev(G, "G", shape=(g.n_rows, k), nullable=True) if want_grad else VP(0)),
        "plp_fgrad")
    return F, AB, (G if want_grad else None)


def hessvec(ctx: Context, g: Graph, U, eta, p: float, AB, mode: int = HESS_SPARSE, eps: float = 1e-9,
            G_in=None, Hv=None):
    k = U.shape[1]
    Hv = _empty(ctx, g.n_rows, k) if Hv is None else Hv
    _ck(_lib.plp_hessvec(ctx.h, g.h, k, _dev(U, "U", shape=(g.n_cols, k)),
                         _dev(eta, "eta", shape=(g.n_cols, k)), C_D(p), _dev(AB, "AB", shape=(2 * k,)),
                         int(mode), C_D(eps), _dev(G_in, "G_in", shape=(g.n_rows, k), nullable=True),
                         _dev(Hv, "Hv", shape=(g.n_rows, k))), "plp_hessvec")
    return Hv


def fgrad_hessvec(ctx: Context, g: Graph, U, eta, p: float, AB_in=None, mode: int = HESS_SPARSE,
                  eps: float = 1e-9, F=None, AB_out=None, G=None, Hv=None):
    """The benchmark unit: F, AB (recomputed), G and Hv in one edge pass (two if AB_in is None)."""
    k = U.shape[1]
    F = _empty(ctx, 1) if F is None else F
    AB_out = _empty(ctx, 2 * k) if AB_out is None else AB_out
    G = _empty(ctx, g.n_rows, k) if G is None else G
    Hv = _empty(ctx, g.n_rows, k) if Hv is None else Hv
    _ck(_lib.plp_fgrad_hessvec(ctx.h, g.h, k, _dev(U, "U", shape=(g.n_cols, k)),
                               _dev(eta, "eta", shape=(g.n_cols, k)), C_D(p),
                               _dev(AB_in, "AB_in", shape=(2 * k,), nullable=True), int(mode),
                               C_D(eps), _dev(F, "F", shape=(1,)), _dev(AB_out, "AB_out", shape=(2 * k,)),
                               _dev(G, "G", shape=(g.n_rows, k)), _dev(Hv, "Hv", shape=(g.n_rows, k))),
        "plp_fgrad_hessvec")
    return F, AB_out, G, Hv


def fgrad_hessvec_raw(ctx: Context, g: Graph, k: int, U, eta, p: float, AB_in, mode: int, eps: float,
                      F, AB_out, G, Hv):
    """Pre-validated variant for timing loops (pointers only; same C call)."""
    _ck(_lib.plp_fgrad_hessvec(ctx.h, g.h, k, VP(U.data_ptr()), VP(eta.data_ptr()), C_D(p),
                               VP(AB_in.data_ptr()) if AB_in is not None else VP(0), int(mode), C_D(eps),
                               VP(F.data_ptr()), VP(AB_out.data_ptr()), VP(G.data_ptr()),
                               VP(Hv.data_ptr())), "plp_fgrad_hessvec")


def edge_pass(ctx: Context, g: Graph, U, eta, p: float, eps: float, AB_in=None, AB_out=None,
              dots_out=None, G=None, Hv=None):
    k = U.shape[1]
    _ck(_lib.plp_edge_pass(ctx.h, g.h, k, _dev(U, "U", shape=(g.n_cols, k)),
                           _dev(eta, "eta", shape=(g.n_cols, k), nullable=True), C_D(p), C_D(eps),
                           _dev(AB_in, "AB_in", shape=(2 * k,), nullable=True),
                           _dev(AB_out, "AB_out", shape=(2 * k,), nullable=True),
                           _dev(dots_out, "dots_out", shape=(2 * k,), nullable=True),
                           _dev(G, "G", shape=(g.n_rows, k), nullable=True),
                           _dev(Hv, "Hv", shape=(g.n_rows, k), nullable=True)), "plp_edge_pass")


def full_epilogue(ctx: Context, n_rows: int, U, p: float, AB, dots, G, Hv):
    k = U.shape[1]
    _ck(_lib.plp_full_epilogue(ctx.h, C_I64(n_rows), k, _dev(U, "U"), C_D(p), _dev(AB, "AB"),
                               _dev(dots, "dots"), _dev(G, "G"), _dev(Hv, "Hv")), "plp_full_epilogue")


def objective_from_ab(ctx: Context, AB, F=None):
    k = AB.numel() // 2
    F = _empty(ctx, 1) if F is None else F
    _ck(_lib.plp_objective_from_ab(ctx.h, k, _dev(AB, "AB"), _dev(F, "F")), "plp_objective_from_ab")
    return F


# ------------------------------------------------------------------------------------------------
# tall-skinny Grassmann kernels
# ------------------------------------------------------------------------------------------------
def gram(ctx: Context, X, Y, out=None):
    n, k = X.shape
    out = _empty(ctx, k, k) if out is None else out
    _ck(_lib.plp_gram(ctx.h, C_I64(n), k, _dev(X, "X"), _dev(Y, "Y", shape=(n, k)), _dev(out, "out", shape=(k, k))),
        "plp_gram")
    return out


def project(ctx: Context, U, G, out=None):
    n, k = U.shape
    out = _empty(ctx, n, k) if out is None else out
    _ck(_lib.plp_project(ctx.h, C_I64(n), k, _dev(U, "U"), _dev(G, "G", shape=(n, k)),
                         _dev(out, "out", shape=(n, k))), "plp_project")
    return out


def apply_sub(ctx: Context, U, M, X, out=None):
    n, k = U.shape
    out = _empty(ctx, n, k) if out is None else out
    _ck(_lib.plp_apply_sub(ctx.h, C_I64(n), k, _dev(U, "U"), _dev(M, "M", shape=(k, k)),
                           _dev(X, "X", shape=(n, k)), _dev(out, "out", shape=(n, k))), "plp_apply_sub")
    return out


def retract(ctx: Context, U, xi, Q=None, R=None):
    n, k = U.shape
    Q = _empty(ctx, n, k) if Q is None else Q
    _ck(_lib.plp_retract(ctx.h, C_I64(n), k, _dev(U, "U"), _dev(xi, "xi", shape=(n, k)),
                         _dev(Q, "Q", shape=(n, k)), _dev(R, "R", shape=(k, k), nullable=True)),
        "plp_retract")
    return Q


def cholesky(ctx: Context, C, R=None, info=None):
    k = C.shape[0]
    R = _empty(ctx, k, k) if R is None else R
    info = torch.zeros(1, dtype=torch.int32, device=C.device) if info is None else info
    _ck(_lib.plp_cholesky(ctx.h, k, _dev(C, "C", shape=(k, k)), _dev(R, "R", shape=(k, k)),
                          _dev(info, "info", dtype=torch.int32)), "plp_cholesky")
    return R, info


def apply_rinv(ctx: Context, X, R, Y=None, Q=None):
    n, k = X.shape
    Q = _empty(ctx, n, k) if Q is None else Q
    _ck(_lib.plp_apply_rinv(ctx.h, C_I64(n), k, _dev(X, "X"), _dev(Y, "Y", shape=(n, k), nullable=True),
                            _dev(R, "R", shape=(k, k)), _dev(Q, "Q", shape=(n, k))), "plp_apply_rinv")
    return Q


def dot(ctx: Context, x, y, out=None):
    n, k = x.shape
    out = _empty(ctx, 1) if out is None else out
    _ck(_lib.plp_dot(ctx.h, C_I64(n), k, _dev(x, "x"), _dev(y, "y", shape=(n, k)), _dev(out, "out")),
        "plp_dot")
    return out


def axpby(ctx: Context, a: float, x, b: float, y):
    n, k = x.shape
    _ck(_lib.plp_axpby(ctx.h, C_I64(n), k, C_D(a), _dev(x, "x"), C_D(b), _dev(y, "y", shape=(n, k))),
        "plp_axpby")
    return y


def tcg_init(ctx: Context, grad, delta: float, kappa: float, theta: float, eta, Heta, r, dlt, scal, status):
    n, k = grad.shape
    _ck(_lib.plp_tcg_init(ctx.h, C_I64(n), k, _dev(grad, "grad"), C_D(delta), C_D(kappa), C_D(theta),
                          _dev(eta, "eta", shape=(n, k)), _dev(Heta, "Heta", shape=(n, k), nullable=True),
                          _dev(r, "r", shape=(n, k)), _dev(dlt, "dlt", shape=(n, k)),
                          _dev(scal, "scal", shape=(TCG_SCAL_LEN,)), _dev(status, "status", dtype=torch.int32)),
        "plp_tcg_init")


def _tcg_vectors(g: Graph, k: int, eta, Heta, r, dlt, Hd):
    """The tCG vectors have the graph's owned rows (n_rows x k); the direction dlt, a Hessian-vector
    input, has n_cols rows (halo slots on a multi-rank graph).  libplp writes n_rows x k doubles to
    each, so a mis-sized tensor is refused here."""
    for name, t in (("eta", eta), ("r", r), ("Hd", Hd)):
        _dev(t, name, shape=(g.n_rows, k))
    if Heta is not None:
        _dev(Heta, "Heta", shape=(g.n_rows, k))
    if tuple(dlt.shape) not in ((g.n_rows, k), (g.n_cols, k)):
        raise ValueError(f"dlt: shape {tuple(dlt.shape)}, expected ({g.n_rows} or {g.n_cols}, {k})")


def tcg_run(ctx: Context, g: Graph, U, AB, G_in, S, p: float, eps: float, mode: int, eta, Heta, r, dlt,
            Hd, scal, status, max_iters: int, iters: int, fused: bool = False):
    k = U.shape[1]
    _tcg_vectors(g, k, eta, Heta, r, dlt, Hd)
    _ck(_lib.plp_tcg_run(ctx.h, g.h, k, _dev(U, "U", shape=(g.n_cols, k)), _dev(AB, "AB", shape=(2 * k,)),
                         _dev(G_in, "G_in", shape=(g.n_rows, k), nullable=True), _dev(S, "S", shape=(k, k)),
                         C_D(p), C_D(eps), int(mode), _dev(eta, "eta"), _dev(Heta, "Heta", nullable=True), _dev(r, "r"),
                         _dev(dlt, "dlt"), _dev(Hd, "Hd"), _dev(scal, "scal", shape=(TCG_SCAL_LEN,)),
                         _dev(status, "status", dtype=torch.int32), int(max_iters), int(iters), int(fused)),
        "plp_tcg_run")


class TcgGraph:
    """plp_tcg_graph: a captured batch of `iters` tCG iterations (arguments baked in)."""

    def __init__(self, ctx: Context, g: Graph, U, AB, G_in, S, p: float, eps: float, mode: int, eta, Heta, r,
                 dlt, Hd, scal, status, max_iters: int, iters: int, fused: bool = False):
        k = U.shape[1]
        _tcg_vectors(g, k, eta, Heta, r, dlt, Hd)
        h = VP()
        self.ctx = ctx
        self.keep = (U, AB, G_in, S, eta, Heta, r, dlt, Hd, scal, status)  # pointers baked into the graph
        _ck(_lib.plp_tcg_graph_create(
            ctx.h, g.h, k, _dev(U, "U", shape=(g.n_cols, k)), _dev(AB, "AB", shape=(2 * k,)),
            _dev(G_in, "G_in", shape=(g.n_rows, k), nullable=True), _dev(S, "S", shape=(k, k)), C_D(p), C_D(eps),
            int(mode), _dev(eta, "eta"), _dev(Heta, "Heta", nullable=True), _dev(r, "r"), _dev(dlt, "dlt"), _dev(Hd, "Hd"),
            _dev(scal, "scal", shape=(TCG_SCAL_LEN,)), _dev(status, "status", dtype=torch.int32), int(max_iters),
            int(iters), int(fused), ctypes.byref(h)), "plp_tcg_graph_create")
        self.h = h

    def launch(self) -> None:
        _ck(_lib.plp_tcg_graph_launch(self.h), "plp_tcg_graph_launch")

    def nodes(self) -> int:
        v = ctypes.c_int()
        _ck(_lib.plp_tcg_graph_nodes(self.h, ctypes.byref(v)), "plp_tcg_graph_nodes")
        return v.value

    def close(self):
        if getattr(self, "h", None):
            _lib.plp_tcg_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gather_rows(ctx: Context, idx, X, out=None):
    m = idx.numel()
    k = X.shape[1]
    out = _empty(ctx, m, k) if out is None else out
    _ck(_lib.plp_gather_rows(ctx.h, C_I64(m), k, _dev(idx, "idx", dtype=torch.int64), _dev(X, "X"),
                             _dev(out, "out", shape=(m, k))), "plp_gather_rows")
    return out


# ------------------------------------------------------------------------------------------------
# k-means, RCut
# ------------------------------------------------------------------------------------------------
def kmeans(ctx: Context, X, clusters: int, uniforms, restarts: int = 10, max_iters: int = 300,
           rel_tol: float = 1e-9):
    n, dim = X.shape
    u, up = _host(uniforms, np.float64)
    if u.size < restarts * clusters:
        raise ValueError("uniforms must hold restarts x clusters values")
    labels = torch.empty(n, dtype=torch.int32, device=X.device)
    cent = _empty(ctx, clusters, dim)
    sse = ctypes.c_double()
    it = ctypes.c_int()
    _ck(_lib.plp_kmeans(ctx.h, C_I64(n), dim, clusters, _dev(X, "X"), up, restarts, max_iters,
                        C_D(rel_tol), _dev(labels, "labels", dtype=torch.int32), _dev(cent, "centroids"),
                        ctypes.byref(sse), ctypes.byref(it)), "plp_kmeans")
    return labels, cent, sse.value, it.value


def kmeans_dist(ctx: Context, X, clusters: int, uniforms, restarts: int = 10, max_iters: int = 300,
                rel_tol: float = 1e-9):
    """Collective k-means over the ranks' row blocks X (plp_kmeans_dist): labels of this rank's
    rows; centroids, sse and iterations identical on every rank."""
    n, dim = X.shape
    u, up = _host(uniforms, np.float64)
    if u.size < restarts * clusters:
        raise ValueError("uniforms must hold restarts x clusters values")
    labels = torch.empty(n, dtype=torch.int32, device=X.device)
    cent = _empty(ctx, clusters, dim)
    sse = ctypes.c_double()
    it = ctypes.c_int()
    xp = _dev(X, "X") if n > 0 else None
    lp = _dev(labels, "labels", dtype=torch.int32) if n > 0 else None
    _ck(_lib.plp_kmeans_dist(ctx.h, C_I64(n), dim, clusters, xp, up, restarts, max_iters, C_D(rel_tol), lp,
                             _dev(cent, "centroids"), ctypes.byref(sse), ctypes.byref(it)), "plp_kmeans_dist")
    return labels, cent, sse.value, it.value


def rcut(ctx: Context, g: Graph, clusters: int, labels, cut=None, sizes=None, out=None):
    cut = _empty(ctx, clusters) if cut is None else cut
    sizes = torch.empty(clusters, dtype=torch.int64, device=labels.device) if sizes is None else sizes
    out = _empty(ctx, 1) if out is None else out
    _ck(_lib.plp_rcut(ctx.h, g.h, clusters, _dev(labels, "labels", dtype=torch.int32), _dev(cut, "cut"),
                      _dev(sizes, "sizes", dtype=torch.int64), _dev(out, "rcut")), "plp_rcut")
    return out, cut, sizes


# ------------------------------------------------------------------------------------------------
# host-side graph utilities (no GPU needed)
# ------------------------------------------------------------------------------------------------
def validate_csr(row_ptr, col, w, n_cols=None, symmetric=True):
    rp, rpp = _host(row_ptr, np.int64)
    c, cp = _host(col, np.int32)
    ww, wp = _host(w, np.float64)
    n = rp.size - 1
    _ck(_lib.plp_validate_csr(C_I64(n), C_I64(n if n_cols is None else n_cols), rpp, cp, wp,
                              int(bool(symmetric))), "plp_validate_csr")


def rcm_order(row_ptr, col):
    rp, rpp = _host(row_ptr, np.int64)
    c, cp = _host(col, np.int32)
    perm = np.empty(rp.size - 1, dtype=np.int64)
    _ck(_lib.plp_rcm_order(C_I64(rp.size - 1), rpp, cp, VP(perm.ctypes.data)), "plp_rcm_order")
    return perm


def tile_order(row_ptr, col, tile: int = TILE_ROWS):
    """RCM sweep + BFS-grown tiles of `tile` nodes (perm[new] = old), rows of a tile by decreasing
    degree.  Default 80: three BFS tiles per 240-row halo-kernel tile.  Measured on the fused pass
    with 240-row kernel tiles (ms, C5 / D23): 60 -> 0.822 / 0.776, 80 -> 0.789 / 0.725,
    120 -> 0.812 / 0.748, 240 -> 0.798 / 0.712 (`profiles/r02l_order_tile.txt`)."""
    rp, rpp = _host(row_ptr, np.int64)
    c, cp = _host(col, np.int32)
    perm = np.empty(rp.size - 1, dtype=np.int64)
    _ck(_lib.plp_tile_order(C_I64(rp.size - 1), rpp, cp, int(tile), VP(perm.ctypes.data)), "plp_tile_order")
    return perm


def permute_csr(row_ptr, col, w, perm):
    rp, rpp = _host(row_ptr, np.int64)
    c, cp = _host(col, np.int32)
    ww, wp = _host(w, np.float64)
    pm, pmp = _host(perm, np.int64)
    n = rp.size - 1
    rpo = np.empty(n + 1, np.int64)
    co = np.empty(c.size, np.int32)
    wo = np.empty(ww.size, np.float64)
    _ck(_lib.plp_permute_csr(C_I64(n), rpp, cp, wp, pmp, VP(rpo.ctypes.data), VP(co.ctypes.data),
                             VP(wo.ctypes.data)), "plp_permute_csr")
    return rpo, co, wo


def partition_rows(row_ptr, parts: int, cost_row: float, cost_nnz: float):
    rp, rpp = _host(row_ptr, np.int64)
    b = np.empty(parts + 1, np.int64)
    _ck(_lib.plp_partition_rows(C_I64(rp.size - 1), rpp, int(parts), C_D(cost_row), C_D(cost_nnz),
                                VP(b.ctypes.data)), "plp_partition_rows")
    return b


def halo_plan(row_ptr, col, r0: int, r1: int):
    """-> (halo global ids int64[n_halo], local CSR (row_ptr int64, col int32) of rows [r0, r1))."""
    rp, rpp = _host(row_ptr, np.int64)
    c, cp = _host(col, np.int32)
    nh = C_I64(0)
    _ck(_lib.plp_halo_plan(rpp, cp, C_I64(r0), C_I64(r1), ctypes.byref(nh), VP(0), VP(0)), "plp_halo_plan")
    halo = np.empty(max(nh.value, 1), np.int64)
    nnz_loc = int(rp[r1] - rp[r0])
    cl = np.empty(max(nnz_loc, 1), np.int32)
    _ck(_lib.plp_halo_plan(rpp, cp, C_I64(r0), C_I64(r1), ctypes.byref(nh), VP(halo.ctypes.data),
                           VP(cl.ctypes.data)), "plp_halo_plan")
    rp_loc = (rp[r0:r1 + 1] - rp[r0]).astype(np.int64)
    return halo[:nh.value], rp_loc, cl[:nnz_loc]


def debug_pow(ctx: Context, a, p: float, eps: float = 1e-9):
    """(s, t) = (cap(a)^{p-2}, a^{p-1}) as the fused edge pass computes them (diagnostic)."""
    n = a.numel()
    s = torch.empty_like(a)
    t = torch.empty_like(a)
    _ck(_lib.plp_debug_pow(ctx.h, C_I64(n), _dev(a, "a"), C_D(p), C_D(eps), _dev(s, "s"), _dev(t, "t")),
        "plp_debug_pow")
    return s, t
