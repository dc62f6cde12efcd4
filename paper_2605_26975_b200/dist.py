"""Multi-GPU plumbing: contiguous row blocks, halo exchange, partial-sum reduction.

One process per GPU (torchrun).  The global graph is split into contiguous row blocks of the
(tile/RCM-ordered) node numbering, balanced on 32 k bytes per row + 12 bytes per stored nonzero
(plp_partition_rows) and aligned to whole tiles.  Each rank owns rows [r0, r1) and holds them
followed by its halo rows (columns outside [r0, r1), sorted; plp_halo_plan) in one extended array
U_ext = [U[r0:r1]; U[halo]], so its local CSR addresses the halo in place.  Because ownership
ranges are contiguous and the halo is sorted, the halo rows owned by one peer form one slice of
U_ext: a received message lands in place.  Per step:
  1. pack the rows each peer needs from this rank (plp_gather_rows kernel, one launch),
  2. exchange U (once per new iterate) and eta with grouped NCCL send/recv over NVLink,
  3. run the rank-local edge pass (plp_edge_pass / plp_fgrad_hessvec) on the extended arrays,
  4. all-reduce the 2k partial sums A, B (and 2k dots in full mode); F = sum A/B on the device.
Only the exchange of step 2 and the all-reduce of step 4 use torch.distributed; every arithmetic
step runs in libplp.  Row results (G, Hv) are bitwise those of one GPU: each row is summed in the
same CSR order.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


class HaloPlan:
    """Host-side plan for one rank (no GPU needed): row block, halo, local CSR, send/recv lists."""

    def __init__(self, row_ptr, col, w, rank: int, world: int, k: int, tile: int = 120,
                 bounds=None):
        from . import plp
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        n = row_ptr.size - 1
        if bounds is None:
            b = plp.partition_rows(row_ptr, world, 32.0 * k, 12.0)
            if tile > 1:  # align interior boundaries to whole tiles
                b[1:-1] = np.minimum(np.round(b[1:-1] / tile) * tile, n).astype(np.int64)
                b = np.maximum.accumulate(b)
            bounds = b
        self.bounds = np.asarray(bounds, np.int64)
        self.rank, self.world = rank, world
        self.r0, self.r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])
        self.n_loc = self.r1 - self.r0
        self.halo, self.rp_loc, self.col_loc = plp.halo_plan(row_ptr, col, self.r0, self.r1)
        self.w_loc = np.ascontiguousarray(np.asarray(w)[row_ptr[self.r0]:row_ptr[self.r1]], np.float64)
        self.n_halo = int(self.halo.size)
        # recv: the slice of my halo owned by each peer (contiguous because halo is sorted)
        owner = np.searchsorted(self.bounds, self.halo, side="right") - 1
        self.recv = {}
        for q in range(world):
            idx = np.nonzero(owner == q)[0]
            if idx.size:
                assert q != rank and np.all(np.diff(idx) == 1)
                self.recv[q] = (int(idx[0]), int(idx.size))
        self.send = {}  # filled by exchange_lists()

    def exchange_lists(self, group=None) -> None:
        """All-gather every rank's halo list once (host objects) and derive the send lists."""
        halos = [None] * self.world
        dist.all_gather_object(halos, self.halo.tolist(), group=group)
        for q in range(self.world):
            if q == self.rank:
                continue
            h = np.asarray(halos[q], dtype=np.int64)
            mine = h[(h >= self.r0) & (h < self.r1)]
            if mine.size:
                self.send[q] = mine - self.r0  # local row indices, in q's halo order


class HaloExchange:
    """Per-step halo exchange of an extended array X_ext [n_loc + n_halo, k] (rows [0, n_loc) are
    owned).  `pack(idx, X, out)` gathers rows (plp_gather_rows on GPU; index_select in CPU tests)."""

    def __init__(self, plan: HaloPlan, k: int, device, dtype=torch.float64, pack=None, group=None):
        self.plan, self.k, self.group = plan, k, group
        order = sorted(plan.send)
        self.send_peers = order
        idx = np.concatenate([plan.send[q] for q in order]) if order else np.zeros(0, np.int64)
        self.send_idx = torch.from_numpy(idx.astype(np.int64)).to(device)
        self.send_off = {}
        off = 0
        for q in order:
            self.send_off[q] = (off, plan.send[q].size)
            off += plan.send[q].size
        self.sendbuf = torch.empty(max(off, 1), k, dtype=dtype, device=device)
        self.pack = pack

    def __call__(self, X_ext: torch.Tensor) -> None:
        p = self.plan
        if self.send_idx.numel():
            self.pack(self.send_idx, X_ext, self.sendbuf[:self.send_idx.numel()])
        ops = []
        for q, (o, c) in self.send_off.items():
            ops.append(dist.P2POp(dist.isend, self.sendbuf[o:o + c], q, group=self.group))
        for q, (o, c) in p.recv.items():
            ops.append(dist.P2POp(dist.irecv, X_ext[p.n_loc + o:p.n_loc + o + c], q, group=self.group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()


class ShardedProblem:
    """One rank's share of the benchmark unit on its GPU (bench.py --gpus N)."""

    def __init__(self, ctx, g, k: int, rank: int, world: int, device, group=None):
        from . import plp
        self.plp, self.ctx, self.k, self.device, self.group = plp, ctx, k, device, group
        self.plan = HaloPlan(g.row_ptr, g.col, g.w, rank, world, k)
        self.plan.exchange_lists(group)
        pl = self.plan
        self.graph = plp.Graph(ctx, pl.rp_loc, pl.col_loc, pl.w_loc, n_cols=pl.n_loc + pl.n_halo, flags=0)
        self.nnz_local = int(pl.rp_loc[-1])

        def pack(idx, X, out):
            plp.gather_rows(ctx, idx, X, out)

        self.xchg = HaloExchange(pl, k, device, pack=pack, group=group)

    def make_step(self, U_h, eta_h, p: float, eps: float, mode: int):
        """Returns step(): exchange U and eta halos, fused pass, all-reduce A, B -> F."""
        plp, pl, k, dev = self.plp, self.plan, self.k, self.device
        ext = np.concatenate([np.arange(pl.r0, pl.r1), pl.halo])
        self.U = torch.from_numpy(np.ascontiguousarray(U_h[pl.r0:pl.r1])).to(dev)
        self.U_ext = torch.zeros(pl.n_loc + pl.n_halo, k, dtype=torch.float64, device=dev)
        self.eta_ext = torch.zeros_like(self.U_ext)
        self.U_ext[:pl.n_loc] = self.U
        self.eta_ext[:pl.n_loc] = torch.from_numpy(np.ascontiguousarray(eta_h[pl.r0:pl.r1])).to(dev)
        del ext
        self.G = torch.empty(pl.n_loc, k, dtype=torch.float64, device=dev)
        self.Hv = torch.empty_like(self.G)
        self.AB = torch.empty(2 * k, dtype=torch.float64, device=dev)
        self.AB_out = torch.empty_like(self.AB)
        self.F = torch.empty(1, dtype=torch.float64, device=dev)
        # A, B at U: objective pass + all-reduce (the solver's rho-test provides them)
        self.xchg(self.U_ext)
        plp.edge_pass(self.ctx, self.graph, self.U_ext, None, p, eps, AB_out=self.AB)
        dist.all_reduce(self.AB, group=self.group)

        def step():
            self.xchg(self.U_ext)
            self.xchg(self.eta_ext)
            plp.edge_pass(self.ctx, self.graph, self.U_ext, self.eta_ext, p, eps, AB_in=self.AB,
                          AB_out=self.AB_out, G=self.G, Hv=self.Hv)
            dist.all_reduce(self.AB_out, group=self.group)
            plp.objective_from_ab(self.ctx, self.AB_out, self.F)

        return step
