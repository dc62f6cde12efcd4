"""Multi-GPU plumbing.

The product path is the collective C ABI: `plp.Context.distributed` (each rank's libplp context
owns an NCCL communicator; torch.distributed only broadcasts the 128-byte NCCL id) and
`plp.DistGraph` (plp_create_graph_dist: the rank's halo plan, exchanged with its peers inside
libplp).  plp_fgrad / plp_hessvec / plp_fgrad_hessvec / plp_rcut then exchange the halo rows of
U and eta and all-reduce A, B, dots and Grams themselves.

This module holds
  * `row_bounds`: the contiguous row-block partition (balanced on 32 k bytes per row + 12 bytes per
    stored nonzero, plp_partition_rows) with interior boundaries aligned to the halo kernel's tiles
    (plp.HALO_TILE, the tiles of plp_tile_order), so each rank's tiles are the ordering's tiles;
  * `HaloPlan` / `HaloExchange`: the same plan as plp_create_graph_dist (recv slices from
    plp_dist_recv_plan, send counts from the all-gathered request-count matrix, request lists sent
    to the owners), written over torch.distributed so that tests/test_dist_gloo.py can check the
    multi-rank algorithm with gloo on CPU (no GPU, no NCCL);
  * `ShardedProblem`: one rank's share of the benchmark unit through the collective ABI.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def row_bounds(row_ptr, world: int, k: int, tile: int | None = None) -> np.ndarray:
    """bounds[0..world]: rank r owns rows [bounds[r], bounds[r+1])."""
    from . import plp
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    n = row_ptr.size - 1
    tile = plp.HALO_TILE if tile is None else tile
    b = plp.partition_rows(row_ptr, world, 32.0 * k, 12.0)
    if tile > 1:
        b[1:-1] = np.minimum(np.round(b[1:-1] / tile) * tile, n).astype(np.int64)
        b = np.maximum.accumulate(b)
    return np.asarray(b, np.int64)


class HaloPlan:
    """One rank's plan (host): owned rows, sorted halo, local CSR, recv slices and send lists --
    the algorithm of plp_create_graph_dist (comm.cu), over any torch.distributed backend."""

    def __init__(self, row_ptr, col, w, rank: int, world: int, k: int, bounds=None, group=None):
        from . import plp
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        self.bounds = row_bounds(row_ptr, world, k) if bounds is None else np.asarray(bounds, np.int64)
        self.rank, self.world, self.group = rank, world, group
        self.r0, self.r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.n_loc = self.r1 - self.r0
        self.halo, self.rp_loc, self.col_loc = plp.halo_plan(row_ptr, col, self.r0, self.r1)
        self.w_loc = np.ascontiguousarray(np.asarray(w)[row_ptr[self.r0]:row_ptr[self.r1]], np.float64)
        self.n_halo = int(self.halo.size)
        # recv: the slice of my halo owned by each peer (libplp's host plan)
        self.recv_off, self.recv_cnt = plp.dist_recv_plan(self.bounds, self.halo)
        assert self.recv_cnt[rank] == 0
        self.send_off = np.zeros(world, np.int64)
        self.send_cnt = np.zeros(world, np.int64)
        self.send_idx = np.zeros(0, np.int64)

    def exchange_lists(self) -> None:
        """Request-count matrix by all-gather, then each rank's request list to its owners (grouped
        send/recv), converted to local row ids -- as plp_create_graph_dist does over NCCL."""
        cnt = torch.from_numpy(self.recv_cnt.copy())
        M = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(M, cnt, group=self.group)
        M = torch.stack(M).numpy()  # M[r][q]: rows rank r needs from rank q
        self.send_cnt = M[:, self.rank].astype(np.int64)
        self.send_off = np.concatenate([[0], np.cumsum(self.send_cnt)[:-1]]).astype(np.int64)
        req = torch.zeros(int(self.send_cnt.sum()), dtype=torch.int64)
        ops = []
        for q in range(self.world):
            if self.recv_cnt[q]:
                o, c = int(self.recv_off[q]), int(self.recv_cnt[q])
                ops.append(dist.P2POp(dist.isend, torch.from_numpy(self.halo[o:o + c].copy()), q, group=self.group))
            if self.send_cnt[q]:
                o, c = int(self.send_off[q]), int(self.send_cnt[q])
                ops.append(dist.P2POp(dist.irecv, req[o:o + c], q, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        req = req.numpy()
        assert np.all((req >= self.r0) & (req < self.r1)), "peer requested a row this rank does not own"
        self.send_idx = req - self.r0


class HaloExchange:
    """Per-step halo exchange of an extended array X_ext [n_loc + n_halo, k]: pack the requested
    rows (`pack(idx, X, out)`), grouped send/recv, each peer's rows land in place."""

    def __init__(self, plan: HaloPlan, k: int, device, dtype=torch.float64, pack=None):
        self.plan, self.k = plan, k
        self.send_idx = torch.from_numpy(plan.send_idx.astype(np.int64)).to(device)
        self.sendbuf = torch.empty(max(int(plan.send_cnt.sum()), 1), k, dtype=dtype, device=device)
        self.pack = pack

    def __call__(self, X_ext: torch.Tensor) -> None:
        p = self.plan
        if self.send_idx.numel():
            self.pack(self.send_idx, X_ext, self.sendbuf[:self.send_idx.numel()])
        ops = []
        for q in range(p.world):
            if p.send_cnt[q]:
                o, c = int(p.send_off[q]), int(p.send_cnt[q])
                ops.append(dist.P2POp(dist.isend, self.sendbuf[o:o + c], q, group=p.group))
            if p.recv_cnt[q]:
                o, c = int(p.recv_off[q]), int(p.recv_cnt[q])
                ops.append(dist.P2POp(dist.irecv, X_ext[p.n_loc + o:p.n_loc + o + c], q, group=p.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


class ShardedProblem:
    """One rank's share of the benchmark unit through the collective C ABI (bench.py --gpus N)."""

    def __init__(self, ctx, g, k: int, rank: int, world: int, device):
        from . import plp
        self.plp, self.ctx, self.k, self.device = plp, ctx, k, device
        self.bounds = row_bounds(g.row_ptr, world, k)
        r0, r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        rp = np.ascontiguousarray(g.row_ptr[r0:r1 + 1], np.int64)
        col = np.ascontiguousarray(g.col[rp[0]:rp[-1]], np.int32)
        w = np.ascontiguousarray(g.w[rp[0]:rp[-1]], np.float64)
        self.graph = plp.DistGraph(ctx, g.n, r0, r1, rp, col, w, flags=0)
        self.r0, self.r1 = r0, r1
        self.nnz_local = self.graph.nnz

    def make_step(self, U_h, eta_h, p: float, eps: float, mode: int):
        """Returns step(): one collective plp_fgrad_hessvec (U and eta halos exchanged, A, B
        all-reduced, F from the global A, B) -- the benchmark unit with a fresh (U, eta) pair."""
        plp, G, k, dev = self.plp, self.graph, self.k, self.device
        self.U_ext = torch.zeros(G.n_cols, k, dtype=torch.float64, device=dev)
        self.eta_ext = torch.zeros_like(self.U_ext)
        self.U_ext[:G.n_rows] = torch.from_numpy(np.ascontiguousarray(U_h[self.r0:self.r1])).to(dev)
        self.eta_ext[:G.n_rows] = torch.from_numpy(np.ascontiguousarray(eta_h[self.r0:self.r1])).to(dev)
        self.G = torch.empty(G.n_rows, k, dtype=torch.float64, device=dev)
        self.Hv = torch.empty_like(self.G)
        self.F = torch.empty(1, dtype=torch.float64, device=dev)
        self.AB = torch.empty(2 * k, dtype=torch.float64, device=dev)
        self.AB_out = torch.empty_like(self.AB)
        # A, B at U (the solver's rho-test provides them): one collective plp_fgrad
        plp.fgrad(self.ctx, G, self.U_ext, p, F=self.F, AB=self.AB, want_grad=False)

        def step():
            plp.fgrad_hessvec_raw(self.ctx, G, k, self.U_ext, self.eta_ext, p, self.AB, mode, eps, self.F,
                                  self.AB_out, self.G, self.Hv)

        return step
