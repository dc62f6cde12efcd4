"""Riemannian trust-region Newton with truncated CG on the Grassmann manifold, with p-continuation
("Newton's method on the Grassmann manifold ... truncated
conjugate gradient scheme ... for progressively smaller values of p").

A host driver over the C ABI: every vector operation (F, EucGrad, EucHessianEta, projection,
curvature correction, dots, axpby, QR retraction, k-means, RCut) runs in libplp's kernels; Python
only holds the scalars of the trust-region and CG recurrences (read back once per step).  There is
no CPU fallback.

Geometry (readings, DESIGN.md §3 #21-#24): U in St(n, k) represents a point, the horizontal space is
{xi : U^T xi = 0} with the Euclidean metric, P(G) = G - U (U^T G), retraction = Q factor of
U + xi with R_ii > 0.  Riemannian gradient grad = P(G); Riemannian Hessian
H(xi) = P(EucHess[xi]) - xi sym(U^T G) (the Grassmann curvature term of SPEC.md:345, with the k x k
matrix symmetrised so that tCG sees a symmetric operator).  EucHess is Alg. 1's sparse Hessian by
default (plp_hessvec, HESS_SPARSE) or the exact one (HESS_FULL).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import torch

from . import plp


@dataclass
class SolverConfig:
    """SPEC.md:302 (defaults of SPEC.md:382-383; the trust radii are unstated: reading #22)."""
    grad_tol: float | None = None       # default 1e-6 sqrt(n k)
    max_outer: int = 200
    tr_delta0: float | None = None      # default tr_delta_max / 8
    tr_delta_max: float | None = None   # default sqrt(k)
    tr_rho_accept: float = 0.1
    tcg_kappa: float = 0.1
    tcg_theta: float = 1.0
    tcg_max_iters: int | None = None    # default min(2 n k, 1000)
    hessian_mode: int = plp.HESS_SPARSE
    eps: float = 1e-9
    device_tcg: bool = True            # tCG recurrences on the device (plp_tcg_run), no per-iteration D2H
    tcg_batch: int = 8                 # most iterations launched between two status reads
    # fused tCG passes (NEXT-2); default on for k = 8, 16 and (folded) k = 1, 2, 4 with n k % 8 = 0
    tcg_fused: bool | None = None
    tcg_graph: bool = True             # replay each batch as one CUDA graph (needs a non-default stream)

    def resolved(self, n: int, k: int) -> "SolverConfig":
        c = SolverConfig(**self.__dict__)
        if c.grad_tol is None:
            c.grad_tol = 1e-6 * math.sqrt(n * k)
        if c.tr_delta_max is None:
            c.tr_delta_max = math.sqrt(k)
        if c.tr_delta0 is None:
            c.tr_delta0 = c.tr_delta_max / 8.0
        if c.tcg_max_iters is None:
            c.tcg_max_iters = min(2 * n * k, 1000)
        if c.tcg_fused is None:
            c.tcg_fused = c.device_tcg and (k in (8, 16) or (k in (1, 2, 4) and (n * k) % 8 == 0))
        if not (0.0 < c.tr_rho_accept < 0.25 and c.grad_tol > 0 and c.tr_delta0 <= c.tr_delta_max):
            raise ValueError("invalid SolverConfig (SPEC.md:303)")
        return c


@dataclass
class IterRecord:
    p: float
    it: int
    F: float
    gradnorm: float
    delta: float
    tcg_iters: int
    tcg_status: str
    rho: float
    accepted: bool
    millis: float


@dataclass
class SolveTrace:
    records: list = field(default_factory=list)

    def csv(self) -> str:
        head = "p,iter,F,gradnorm,delta,tcg_iters,tcg_status,rho,accepted,millis"
        rows = [f"{r.p},{r.it},{r.F!r},{r.gradnorm!r},{r.delta!r},{r.tcg_iters},{r.tcg_status},"
                f"{r.rho!r},{int(r.accepted)},{r.millis:.3f}" for r in self.records]
        return "\n".join([head] + rows)


class _State:
    """Device state at the current iterate: U, F, AB, G, grad = P(G), S = sym(U^T G).

    On a multi-rank graph (plp.DistGraph) U has n_cols = n_own + n_halo rows (plp_fgrad fills the
    halo rows); every other vector has the n_own owned rows, and the Grams / dots / projections are
    collective (global) in libplp."""

    def __init__(self, solver: "GrassmannTR", U, p: float):
        s = solver
        self.U = U
        Uo = s.own(U)
        self.F, self.AB, self.G = plp.fgrad(s.ctx, s.g, U, p)
        self.grad = plp.project(s.ctx, Uo, self.G)
        # S = sym(U^T G) = (U^T G + G^T U) / 2, two Grams and an axpby in libplp
        self.S = plp.gram(s.ctx, Uo, self.G)
        plp.axpby(s.ctx, 0.5, plp.gram(s.ctx, self.G, Uo), 0.5, self.S)
        self.Fv = float(self.F.item())


class GrassmannTR:
    """Trust-region Newton for min F_p(U) over the Grassmann manifold (one graph, one context)."""

    def __init__(self, ctx: plp.Context, g: plp.Graph, k: int, cfg: SolverConfig | None = None):
        self.ctx, self.g, self.k = ctx, g, k
        # multi-rank (a DistGraph on a context with peers): global sizes for the defaults, no
        # CUDA-graph capture of the NCCL calls; the fused device tCG at k = 8, 16 (its k x k and
        # scalar totals all-reduced before each scalar step, tcg.cu), the unfused one otherwise (the
        # folded k = 1, 2, 4 view needs n_own k % 8 == 0 on every rank)
        self.n_own, self.n_cols = g.n_rows, g.n_cols
        self.multi = isinstance(g, plp.DistGraph) and ctx.world > 1
        n_glob = g.n_global if isinstance(g, plp.DistGraph) else g.n_rows
        cfg = cfg or SolverConfig()
        if self.multi:
            fused = cfg.tcg_fused if k in (8, 16) else False
            cfg = SolverConfig(**{**cfg.__dict__, "tcg_fused": fused, "tcg_graph": False})
        self.cfg = cfg.resolved(n_glob, k)
        self.hmode = self.cfg.hessian_mode | (plp.U_HALO_CURRENT if isinstance(g, plp.DistGraph) else 0)

    def own(self, X):
        """The owned rows of an n_cols-row array (a view)."""
        return X[:self.n_own] if X.shape[0] != self.n_own else X

    def ext(self, X):
        """An n_cols-row copy of an owned-row array (halo rows to be filled by libplp)."""
        if X.shape[0] == self.n_cols:
            return X
        Y = torch.zeros(self.n_cols, X.shape[1], dtype=X.dtype, device=X.device)
        Y[:self.n_own] = X
        return Y

    # -- operators --------------------------------------------------------------------------------
    def _hess(self, st: _State, p: float, xi):
        """H(xi) = P(EucHess[xi]) - xi S."""
        c = self.cfg
        EH = plp.hessvec(self.ctx, self.g, st.U, self.ext(xi), p, st.AB, mode=self.hmode, eps=c.eps,
                         G_in=st.G if c.hessian_mode == plp.HESS_FULL else None)
        PEH = plp.project(self.ctx, self.own(st.U), EH, out=EH)
        return plp.apply_sub(self.ctx, self.own(xi), st.S, PEH, out=PEH)

    def _dot(self, x, y) -> float:
        return float(plp.dot(self.ctx, x, y).item())

    # -- truncated CG on the device (plp_tcg_init / plp_tcg_run): same recurrences, no host sync
    # per iteration; the status is read once per `tcg_batch` iterations -------------------------
    def tcg_device(self, st: _State, p: float, delta: float):
        c = self.cfg
        ctx = self.ctx
        if not hasattr(self, "_tcg_buf") or self._tcg_buf[0].shape != st.grad.shape:
            z = lambda: torch.empty_like(st.grad)  # noqa: E731
            self._graphs, self._gin = {}, None
            # the direction is a Hessian-vector input: n_cols rows (halo slots on a DistGraph)
            dl = torch.zeros(self.n_cols, st.grad.shape[1], dtype=st.grad.dtype, device=st.grad.device)
            self._tcg_buf = (z(), z(), z(), dl, z(),
                             torch.zeros(plp.TCG_SCAL_LEN, dtype=torch.float64, device=st.grad.device),
                             torch.zeros(2, dtype=torch.int32, device=st.grad.device))
        eta, Heta, r, dlt, Hd, scal, status = self._tcg_buf
        # fused: no H step accumulated per iteration (16 n k bytes less per pass); H(eta) once at the end
        Hacc = None if c.tcg_fused else Heta
        plp.tcg_init(ctx, st.grad, delta, c.tcg_kappa, c.tcg_theta, eta, Hacc, r, self.own(dlt), scal, status)
        full = c.hessian_mode == plp.HESS_FULL
        use_graph = c.tcg_graph and ctx.stream.cuda_stream != 0
        if use_graph:
            self._refresh_graph_inputs(st, p)
        G_in = st.G if full else None
        done = 0
        batch = 1  # batches of 1, 2, 4, ... tcg_batch iterations: short solves waste little
        stv = status.cpu().tolist()
        while stv[0] == 0 and done < c.tcg_max_iters:
            if use_graph:
                self._graph_for(p, batch).launch()  # iterations past max_iters are no-ops (MAXITER)
            else:
                plp.tcg_run(ctx, self.g, st.U, st.AB, G_in, st.S, p, c.eps, c.hessian_mode, eta, Hacc, r, dlt,
                            Hd, scal, status, c.tcg_max_iters, min(batch, c.tcg_max_iters - done),
                            fused=c.tcg_fused)
            done += batch
            batch = min(2 * batch, c.tcg_batch)
            stv = status.cpu().tolist()
        if c.tcg_fused:
            return eta.clone(), self._hess(st, p, eta), int(stv[1]), plp.TCG_STATUS[int(stv[0])]
        return eta.clone(), Heta.clone(), int(stv[1]), plp.TCG_STATUS[int(stv[0])]

    def _refresh_graph_inputs(self, st: _State, p: float) -> None:
        """Copy the iterate into the persistent buffers the captured graphs read (their pointers
        are fixed); drop the graphs when p changes (p is baked in)."""
        full = self.cfg.hessian_mode == plp.HESS_FULL
        if getattr(self, "_gin", None) is None or self._gin[0].shape != st.U.shape:
            self._gin = (torch.empty_like(st.U), torch.empty_like(st.AB), torch.empty_like(st.S),
                         torch.empty_like(st.G) if full else None)
            self._graphs = {}
        U, AB, S, G = self._gin
        U.copy_(st.U)
        AB.copy_(st.AB)
        S.copy_(st.S)
        if full:
            G.copy_(st.G)
        if getattr(self, "_graph_p", None) != p:
            self._graphs, self._graph_p = {}, p

    def _graph_for(self, p: float, batch: int):
        """The captured batch of `batch` iterations for this p (one CUDA graph per batch size)."""
        c = self.cfg
        if batch not in self._graphs:
            U, AB, S, G = self._gin
            eta, Heta, r, dlt, Hd, scal, status = self._tcg_buf
            self._graphs[batch] = plp.TcgGraph(self.ctx, self.g, U, AB, G, S, p, c.eps, c.hessian_mode, eta,
                                               None if c.tcg_fused else Heta, r, dlt, Hd, scal, status,
                                               c.tcg_max_iters, batch, fused=c.tcg_fused)
        return self._graphs[batch]

    # -- truncated CG (Steihaug-Toint; Absil-Baker-Gallivan 2007, Alg. 2) ------------------------
    def tcg(self, st: _State, p: float, delta: float):
        c = self.cfg
        ctx = self.ctx
        eta = torch.zeros_like(st.grad)
        Heta = torch.zeros_like(st.grad)
        r = st.grad.clone()
        z_r = self._dot(r, r)
        r0 = math.sqrt(z_r)
        if r0 == 0.0:
            return eta, Heta, 0, "interior"
        dlt_ext = torch.zeros(self.n_cols, r.shape[1], dtype=r.dtype, device=r.device)
        dlt = self.own(dlt_ext)  # view: the owned rows of the Hessian-vector input
        plp.axpby(ctx, -1.0, r, 0.0, dlt)  # dlt = -r
        e_Pe, e_Pd, d_Pd = 0.0, 0.0, z_r
        stop_tol = r0 * min(r0 ** c.tcg_theta, c.tcg_kappa)
        status = "maxiter"
        j = 0
        for j in range(1, c.tcg_max_iters + 1):
            Hd = self._hess(st, p, dlt_ext)
            d_Hd = self._dot(dlt, Hd)
            alpha = z_r / d_Hd if d_Hd != 0.0 else math.inf
            e_Pe_new = e_Pe + 2.0 * alpha * e_Pd + alpha * alpha * d_Pd
            if d_Hd <= 0.0 or e_Pe_new >= delta * delta:
                tau = (-e_Pd + math.sqrt(e_Pd * e_Pd + d_Pd * (delta * delta - e_Pe))) / d_Pd
                plp.axpby(ctx, tau, dlt, 1.0, eta)
                plp.axpby(ctx, tau, Hd, 1.0, Heta)
                status = "negative_curvature" if d_Hd <= 0.0 else "boundary"
                break
            e_Pe = e_Pe_new
            plp.axpby(ctx, alpha, dlt, 1.0, eta)
            plp.axpby(ctx, alpha, Hd, 1.0, Heta)
            plp.axpby(ctx, alpha, Hd, 1.0, r)
            r = plp.project(ctx, self.own(st.U), r, out=r)  # keep the residual horizontal
            z_new = self._dot(r, r)
            if math.sqrt(z_new) <= stop_tol:
                status = "converged"
                break
            beta = z_new / z_r
            z_r = z_new
            plp.axpby(ctx, -1.0, r, beta, dlt)  # dlt = -r + beta dlt
            e_Pd = beta * (e_Pd + alpha * d_Pd)
            d_Pd = z_r + beta * beta * d_Pd
        return eta, Heta, j, status

    # -- outer loop ---------------------------------------------------------------------------------
    def solve(self, U0, p: float, trace: SolveTrace | None = None):
        """Trust-region solve at fixed p; torch work (buffers, scalar reads) is ordered on the
        context's stream."""
        with torch.cuda.stream(self.ctx.stream):
            return self._solve(U0, p, trace)

    def _solve(self, U0, p: float, trace: SolveTrace | None = None):
        c = self.cfg
        ctx = self.ctx
        trace = trace if trace is not None else SolveTrace()
        st = _State(self, U0, p)
        if not math.isfinite(st.Fv):
            raise FloatingPointError(f"non-finite objective at p={p}")
        delta = c.tr_delta0
        for it in range(c.max_outer):
            t0 = time.perf_counter()
            gnorm = math.sqrt(self._dot(st.grad, st.grad))
            if gnorm <= c.grad_tol or delta < 1e-14:
                trace.records.append(IterRecord(p, it, st.Fv, gnorm, delta, 0, "stop", math.nan, False,
                                                1e3 * (time.perf_counter() - t0)))
                break
            if c.device_tcg:
                eta, Heta, nit, status = self.tcg_device(st, p, delta)
            else:
                eta, Heta, nit, status = self.tcg(st, p, delta)
            model_dec = -self._dot(st.grad, eta) - 0.5 * self._dot(eta, Heta)
            try:
                U_new = self.ext(plp.retract(ctx, self.own(st.U), eta))
                cand = _State(self, U_new, p)
                F_new = cand.Fv
            except plp.PlpError:  # rank-deficient U + eta: a rejected step
                cand, F_new = None, math.inf
            if model_dec > 0.0:
                rho = (st.Fv - F_new) / model_dec
            else:
                rho = 1.0 if F_new <= st.Fv else -math.inf
            accepted = cand is not None and math.isfinite(F_new) and rho > c.tr_rho_accept
            if rho < 0.25:
                delta *= 0.5
            elif rho > 0.75 and status in ("boundary", "negative_curvature"):
                delta = min(2.0 * delta, c.tr_delta_max)
            trace.records.append(IterRecord(p, it, F_new if accepted else st.Fv, gnorm, delta, nit,
                                            status, rho, accepted, 1e3 * (time.perf_counter() - t0)))
            if accepted:
                st = cand
        return st.U, trace


def init_embedding(ctx: plp.Context, Z) -> torch.Tensor:
    """U0 = Q factor of a seeded Gaussian sample Z, by the QR retraction at 0."""
    return plp.retract(ctx, Z, torch.zeros_like(Z))


def continuation_solve(ctx: plp.Context, g: plp.Graph, Z, schedule, cfg: SolverConfig | None = None):
    """Solve at p = schedule[0] (= 2) from QR(Z), then warm-start each smaller p from the previous
    solution after QR re-orthonormalisation (reading #23).  On a multi-rank graph
    every rank passes its own rows of Z and gets its own rows of U back (the QR is collective)."""
    k = Z.shape[1]
    tr = GrassmannTR(ctx, g, k, cfg)
    trace = SolveTrace()
    U = tr.ext(init_embedding(ctx, tr.own(Z)))
    for j, p in enumerate(schedule):
        if j > 0:
            Uo = tr.own(U)
            U = tr.ext(plp.retract(ctx, Uo, torch.zeros_like(Uo)))
        U, trace = tr.solve(U, float(p), trace)
    return tr.own(U), trace


def _allgather_rows(X, group=None):
    """All ranks' owned rows of X, in rank order (= global row order of the contiguous blocks)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([X.shape[0]], dtype=torch.int64, device=X.device)
    ns = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    m = int(max(int(v.item()) for v in ns))
    pad = torch.zeros(m, *X.shape[1:], dtype=X.dtype, device=X.device)
    pad[:X.shape[0]] = X
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([pt[:int(v.item())] for pt, v in zip(parts, ns)])


def cluster(ctx: plp.Context, g: plp.Graph, U, k: int, uniforms, restarts: int = 10, kmeans: str = "sharded"):
    """Discretisation: k-means on the rows of U, then RCut of the labels.

    Multi-rank (a DistGraph): kmeans="sharded" (default) runs the collective k-means on each
    rank's own rows (plp_kmeans_dist: D^2 sums, per-cluster sums / counts / sse and the farthest
    point all-reduced; bitwise plp_kmeans on one rank); kmeans="gathered" all-gathers the n x k
    embedding and runs plp_kmeans on the whole of it on every GPU (identical labels everywhere,
    0.5 GB over NVLink at C5).  Each rank keeps its own rows' labels (+ halo slots) and RCut is
    collective (plp_rcut)."""
    if isinstance(g, plp.DistGraph):
        labels = torch.zeros(g.n_cols, dtype=torch.int32, device=U.device)
        if kmeans == "gathered" and ctx.world > 1:
            Ua = _allgather_rows(U[:g.n_rows].contiguous())
            lab_all, centroids, sse, _ = plp.kmeans(ctx, Ua, k, uniforms, restarts=restarts)
            labels[:g.n_rows] = lab_all[g.row_begin:g.row_end]
        else:
            lab, centroids, sse, _ = plp.kmeans_dist(ctx, U[:g.n_rows].contiguous(), k, uniforms, restarts=restarts)
            labels[:g.n_rows] = lab
        rc, cut, sizes = plp.rcut(ctx, g, k, labels)
        return labels[:g.n_rows], float(rc.item()), sse
    labels, centroids, sse, _ = plp.kmeans(ctx, U, k, uniforms, restarts=restarts)
    rc, cut, sizes = plp.rcut(ctx, g, k, labels)
    return labels, float(rc.item()), sse
