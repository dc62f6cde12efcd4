"""bench.py -- fused F / EucGrad / EucHessianEta throughput (GNNZ*k/s) on B200, BASELINE.json's metric.

A step = one plp_fgrad_hessvec call (SURVEY.md §8(a) a7 = a2..a5 fused, sparse-mode Hessian) on
the workload config (default C5: 8,388,608 uniform points in [0,1]^2, symmetrised 6-NN graph,
Gaussian weights, k = 8, p = 1.2, tile order = RCM + BFS-grown 120-row tiles), with A, B at U
supplied from a preceding plp_fgrad
(the trust-region rho-test always has them).  Inputs (CSR 0.71 GB + U, eta 1.07 GB)
exceed the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl plp|reference] [--config C5]

N > 1: launched by torchrun (or, without WORLD_SIZE in the environment, bench.py re-executes itself
under torch.distributed.run with N ranks); rows are split in contiguous blocks (RCM order), each step exchanges
the U and eta halos with NCCL and all-reduces A, B; time = max over ranks.
`--impl reference` times the fp64 CPU oracle (oracle/) on the same workload (generator order, from
plp_inputs alone) on this host's cores (the tier's reference arm); no product code runs on that arm.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_DESC = {
    "C5": "n=8,388,608 uniform points in [0,1]^2, symmetrised 6-NN, w=exp(-d^2/(2 median d^2)), k=8, p=1.2",
    "C3": "128^3 grid 7-point stencil + 1% long-range edges (w=0.1), k=8, p=1.5",
    "C4": "10-D GMM n=1,000,000, 20 clusters, symmetrised 15-NN, k=20, p=1.2",
    "C2": "two moons n=100,000, 10-NN, k=2, p=1.1",
    "D23": "Delaunay triangulation of 2^23 uniform points (the paper's delaunay_n23 shape), unit weights, k=8, p=1.2",
    "D20": "Delaunay triangulation of 2^20 uniform points, unit weights, k=8, p=1.2",
    "D16": "Delaunay triangulation of 2^16 uniform points, unit weights, k=8, p=1.2",
}
CONFIG_KP = {"C5": (8, 1.2), "C3": (8, 1.5), "C4": (20, 1.2), "C2": (2, 1.1), "C1": (3, 1.2),
             **{f"D{r}": (8, 1.2) for r in range(14, 24)}}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def get_graph(name: str, order: str):
    """Seeded synthetic graph (plp_inputs) in RCM order (libplp host code); cached under /tmp only
    to save generation time between runs (regenerated when absent)."""
    from plp_inputs import make_config, Graph
    from paper_2605_26975_b200 import plp
    from paper_2605_26975_b200.plp import TILE_ROWS
    tile = int(os.environ.get("PLP_ORDER_TILE", TILE_ROWS))  # BFS tile of the ordering (experiments)
    key = hashlib.sha1(f"{name}-{order}-{tile}-v5".encode()).hexdigest()[:12]
    cache = f"/tmp/plp_cache/{name}_{order}_{key}.npz"
    if os.path.exists(cache):
        try:
            z = np.load(cache)
            return Graph(name, int(z["n"]), z["rp"], z["col"], z["w"])
        except Exception:
            pass
    t0 = time.time()
    g = make_config(name)
    log(f"[bench] generated {name}: n={g.n} nnz={g.nnz} in {time.time() - t0:.1f}s")
    if order in ("rcm", "tile"):
        t0 = time.time()
        perm = plp.rcm_order(g.row_ptr, g.col) if order == "rcm" else plp.tile_order(g.row_ptr, g.col, tile)
        rp, col, w = plp.permute_csr(g.row_ptr, g.col, g.w, perm)
        g = Graph(name, g.n, rp, col, w)
        log(f"[bench] {order} reorder in {time.time() - t0:.1f}s")
    try:
        os.makedirs(os.path.dirname(cache), exist_ok=True)
        tmp = f"{cache}.{os.getpid()}.tmp.npz"  # one writer per process (ranks race on the cache)
        np.savez(tmp, n=g.n, rp=g.row_ptr, col=g.col, w=g.w)
        os.replace(tmp, cache)
    except Exception:
        pass
    return g


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes(n: int, nnz: int, k: int) -> int:
    """CSR once (12 nnz + 4(n+1)), U and eta read once, G and Hv written once."""
    return 12 * nnz + 4 * (n + 1) + 32 * n * k


# ------------------------------------------------------------------------------------------------
def row_block_sample(g, S: int):
    """Rows [0, S) of a CSR as a local CSR whose columns index an extended array [rows 0..S-1;
    halo] (the sorted distinct columns >= S), like one rank's shard.  numpy only: the oracle legs
    of this file execute no product code."""
    rp = np.ascontiguousarray(g.row_ptr[:S + 1], np.int64)
    cols = np.asarray(g.col[:rp[S]], np.int64)
    out = cols >= S
    halo = np.unique(cols[out])
    col_loc = cols.copy()
    col_loc[out] = S + np.searchsorted(halo, cols[out])
    return halo, rp, col_loc.astype(np.int32)


def cpu_oracle_sample(g, k, p, eps, rows_frac=0.25, reps=1, threads=None):
    """Time the fp64 oracle (as it stands) on rows [0, S) of the workload (a local CSR whose
    columns index an extended U, like one rank's shard).  Returns (GNNZ*k/s, seconds, desc, cores)."""
    import oracle
    from plp_inputs import draw_U, draw_eta
    S = max(1, min(g.n, int(round(g.n * rows_frac))))
    halo, rp_loc, col_loc = row_block_sample(g, S)
    ext = np.concatenate([np.arange(S), halo])

    class Loc:
        row_ptr, col, w = rp_loc, col_loc, g.w[:g.row_ptr[S]]

    U = draw_U(g.n, k, 0)[ext]
    eta = draw_eta(g.n, k, 0)[ext]
    nnz_s = int(rp_loc[-1])
    if threads is None:
        oracle.set_threads(os.cpu_count() or 1)
    else:
        oracle.set_threads(threads)
    cores = oracle.get_threads()
    t0 = time.time()
    for _ in range(reps):
        F, A, B = oracle.objective(Loc, U, p)
        Gr = oracle.euc_grad(Loc, U, p, A, B)
        Hv = oracle.hessvec(Loc, U, eta, p, eps, "sparse", (A, B))
    dt = (time.time() - t0) / reps
    what = "all rows" if S == g.n else f"rows [0,{S})"
    desc = (f"oracle F+grad+Hv (sparse) on {what} of the workload = {nnz_s} stored nonzeros "
            f"x k={k} (fraction {nnz_s / g.nnz:.3f} of nnz), {cores} OpenMP threads on {cpu_model()}")
    del Gr, Hv
    return nnz_s * k / dt / 1e9, dt, desc, cores


def get_graph_generator_order(name: str):
    """The workload in generator order from plp_inputs alone (no libplp): the reference arm's input.
    Same graph as get_graph's up to a node relabelling."""
    from plp_inputs import make_config, Graph
    cache = f"/tmp/plp_cache/{name}_gen_oracle.npz"
    if os.path.exists(cache):
        try:
            z = np.load(cache)
            return Graph(name, int(z["n"]), z["rp"], z["col"], z["w"])
        except Exception:
            pass
    g = make_config(name)
    try:
        os.makedirs(os.path.dirname(cache), exist_ok=True)
        tmp = f"{cache}.{os.getpid()}.tmp.npz"
        np.savez(tmp, n=g.n, rp=g.row_ptr, col=g.col, w=g.w)
        os.replace(tmp, cache)
    except Exception:
        pass
    return g


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_oracle_single_thread(g, k, p, eps, rows: int = 200_000):
    """the oracle on one thread too (rows [0, rows) of the workload)."""
    import oracle
    v, dt, desc, cores = None, None, None, None
    nthreads = oracle.get_threads()
    try:
        v, dt, desc, cores = cpu_oracle_sample(g, k, p, eps, rows_frac=rows / g.n, threads=1)
    finally:
        oracle.set_threads(nthreads)
    return v, dt


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle on the same config/metric, bounded sample per step."""
    if rank != 0:
        return
    k, p = CONFIG_KP[args.config]
    g = get_graph_generator_order(args.config)  # plp_inputs only: no product code on this arm
    vals, dts = [], []
    desc, cores = "", 0
    for s in range(args.warmup + args.steps):
        v, dt, desc, cores = cpu_oracle_sample(g, k, p, 1e-9, rows_frac=args.ref_frac)
        if s >= args.warmup:
            vals.append(v)
            dts.append(dt)
    val = float(np.median(vals))
    out = {"metric": "fused grad+Hv GNNZ*k/s", "value": val, "unit": "GNNZ*k/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.median(dts)),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": args.config, "desc": CONFIG_DESC.get(args.config, args.config),
                      "n": g.n, "nnz": g.nnz, "k": k, "p": p,
                      "order": "generator (the same graph as the plp arm's up to a relabelling)",
                      "rows": "all" if args.ref_frac >= 1.0 else f"fraction {args.ref_frac} of the rows"},
           "cpu_baseline": {"value": val, "unit": "GNNZ*k/s", "cores": cores, "kind": "oracle",
                            "sample": desc},
           "e2e": {"value": val, "unit": "GNNZ*k/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------------
def run_plp(args, rank, world):
    import torch
    from paper_2605_26975_b200 import plp
    from plp_inputs import draw_U, draw_eta

    dev = torch.device(f"cuda:{args.local_rank}")
    torch.cuda.set_device(dev)
    k, p = CONFIG_KP[args.config]
    eps = 1e-9
    mode = plp.HESS_FULL if args.mode == "full" else plp.HESS_SPARSE
    g = get_graph(args.config, args.order)
    n, nnz = g.n, g.nnz
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sharded = world > 1 or args.sharded
    # multi-rank: the collective ABI (libplp's own NCCL communicator; torch broadcasts its id)
    ctx = plp.Context.distributed(args.local_rank, stream) if sharded else plp.Context(args.local_rank, stream)
    U_h = draw_U(n, k, 0)
    eta_h = draw_eta(n, k, 0)

    if sharded:
        from paper_2605_26975_b200 import dist
        prob = dist.ShardedProblem(ctx, g, k, rank, world, device=dev)
        step = prob.make_step(U_h, eta_h, p, eps, mode)
        nnz_local = prob.nnz_local
    else:
        G = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=plp.VALIDATE)
        U = torch.from_numpy(U_h).to(dev)
        eta = torch.from_numpy(eta_h).to(dev)
        Fb = torch.empty(1, dtype=torch.float64, device=dev)
        AB_in = torch.empty(2 * k, dtype=torch.float64, device=dev)
        AB_out = torch.empty(2 * k, dtype=torch.float64, device=dev)
        Gr = torch.empty(n, k, dtype=torch.float64, device=dev)
        Hv = torch.empty(n, k, dtype=torch.float64, device=dev)
        plp.fgrad(ctx, G, U, p, F=Fb, AB=AB_in, want_grad=False)

        def step():
            plp.fgrad_hessvec_raw(ctx, G, k, U, eta, p, AB_in, mode, eps, Fb, AB_out, Gr, Hv)
        nnz_local = nnz

    def barrier():
        if sharded:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(args.local_rank) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = nnz * k / (ms * 1e-3) / 1e9  # whole-job GNNZ*k/s

    # ---- dominant kernel alone (edge pass without finalize), per-launch CUDA events ----
    roof = None
    if not sharded:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        torch.cuda.synchronize()
        evs[0].record(stream)
        for i in range(args.steps):
            plp.edge_pass(ctx, G, U, eta, p, eps, AB_in=AB_in, G=Gr, Hv=Hv)
            evs[i + 1].record(stream)
        torch.cuda.synchronize()
        kms = float(np.mean([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]))
        peak, peak_kind = load_peaks()
        byts = algorithmic_bytes(n, nnz, k)
        ach = byts / (kms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(f"{args.config}-{args.order}-{args.mode}")
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "kernel": plp.last_edge_kernel(),
                "kernel_ms": kms, "algorithmic_bytes": byts, "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}
    else:
        # rank-local edge pass alone (no halo exchange), per-launch events; whole job: the global
        # algorithmic bytes over the slowest rank's time against world x the per-GPU peak
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        barrier()
        evs[0].record(stream)
        for i in range(args.steps):
            plp.edge_pass(ctx, prob.graph, prob.U_ext, prob.eta_ext, p, eps, AB_in=prob.AB, G=prob.G, Hv=prob.Hv)
            evs[i + 1].record(stream)
        barrier()
        kms = float(np.mean([evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]))
        if world > 1:
            t = torch.tensor([kms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            kms = float(t.item())
        peak, peak_kind = load_peaks()
        byts = algorithmic_bytes(n, nnz, k)
        ach = byts / (kms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak * world, "unit": "GB/s",
                "frac": ach / (peak * world), "traffic": None, "kernel": plp.last_edge_kernel(),
                "kernel_ms": kms, "algorithmic_bytes": byts,
                "peak_kind": f"{peak_kind} x {world} GPUs (MEASURED_PEAKS.json hbm_gbs); kernel_ms = max over ranks"}

    # ---- end to end through the public API: pinned host inputs in, results out, every step ----
    e2e = None
    if not sharded and not args.no_e2e:
        # Streamed through the public API: every step uploads its U, eta from pinned host memory and
        # downloads its F, AB, G, Hv.  Uploads, the kernel and downloads run on three streams with
        # double-buffered device arrays, so step i + 1's upload overlaps step i's download (PCIe is
        # full duplex); every step's copies are inside the timed region.
        U_p = torch.from_numpy(U_h).pin_memory()
        E_p = torch.from_numpy(eta_h).pin_memory()
        nb = 2
        Ud = [U] + [torch.empty_like(U) for _ in range(nb - 1)]
        Ed = [eta] + [torch.empty_like(eta) for _ in range(nb - 1)]
        Gd = [Gr] + [torch.empty_like(Gr) for _ in range(nb - 1)]
        Hd = [Hv] + [torch.empty_like(Hv) for _ in range(nb - 1)]
        Fd = [Fb] + [torch.empty_like(Fb) for _ in range(nb - 1)]
        ABd = [AB_out] + [torch.empty_like(AB_out) for _ in range(nb - 1)]
        G_p = [torch.empty(n, k, dtype=torch.float64).pin_memory() for _ in range(nb)]
        H_p = [torch.empty(n, k, dtype=torch.float64).pin_memory() for _ in range(nb)]
        F_p = [torch.empty(1, dtype=torch.float64).pin_memory() for _ in range(nb)]
        AB_p = [torch.empty(2 * k, dtype=torch.float64).pin_memory() for _ in range(nb)]
        s_up, s_down = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        up_done = [torch.cuda.Event() for _ in range(nb)]
        comp_done = [torch.cuda.Event() for _ in range(nb)]
        down_done = [torch.cuda.Event() for _ in range(nb)]
        for b in range(nb):  # mark every buffer free
            comp_done[b].record(stream)
            down_done[b].record(stream)
        e_steps = max(4, min(args.steps, 10))

        def e2e_step(i):
            b = i % nb
            s_up.wait_event(comp_done[b])  # step i - nb finished reading Ud[b], Ed[b]
            with torch.cuda.stream(s_up):
                Ud[b].copy_(U_p, non_blocking=True)
                Ed[b].copy_(E_p, non_blocking=True)
            up_done[b].record(s_up)
            stream.wait_event(up_done[b])
            stream.wait_event(down_done[b])  # step i - nb's results are out of Gd[b], Hd[b]
            plp.fgrad_hessvec_raw(ctx, G, k, Ud[b], Ed[b], p, AB_in, mode, eps, Fd[b], ABd[b], Gd[b], Hd[b])
            comp_done[b].record(stream)
            s_down.wait_event(comp_done[b])
            with torch.cuda.stream(s_down):
                G_p[b].copy_(Gd[b], non_blocking=True)
                H_p[b].copy_(Hd[b], non_blocking=True)
                F_p[b].copy_(Fd[b], non_blocking=True)
                AB_p[b].copy_(ABd[b], non_blocking=True)
            down_done[b].record(s_down)
        for i in range(nb):
            e2e_step(i)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        s_up.wait_stream(stream)
        for i in range(e_steps):
            e2e_step(i)
        for b in range(nb):
            stream.wait_event(down_done[b])
        a1.record(stream)
        torch.cuda.synchronize()
        ems = a0.elapsed_time(a1) / e_steps
        e2e = {"value": nnz * k / (ems * 1e-3) / 1e9, "unit": "GNNZ*k/s",
               "h2d_bytes_per_step": 2 * n * k * 8, "d2h_bytes_per_step": 2 * n * k * 8 + 8 + 16 * k,
               "ms_per_step": ems,
               "note": "pinned host U, eta in and F, AB, G, Hv out every step; uploads / kernel / downloads "
                       "on three streams, double-buffered (upload of step i+1 overlaps download of step i)"}

    if sharded and not args.no_e2e:
        # each rank: its own rows of U, eta from pinned host memory in, its rows of G, Hv and F out
        n_loc = prob.graph.n_rows
        U_p = torch.from_numpy(np.ascontiguousarray(U_h[prob.r0:prob.r1])).pin_memory()
        E_p = torch.from_numpy(np.ascontiguousarray(eta_h[prob.r0:prob.r1])).pin_memory()
        G_p = torch.empty(n_loc, k, dtype=torch.float64).pin_memory()
        H_p = torch.empty(n_loc, k, dtype=torch.float64).pin_memory()
        F_p = torch.empty(1, dtype=torch.float64).pin_memory()
        e_steps = max(3, min(args.steps, 10))

        def e2e_step():
            prob.U_ext[:n_loc].copy_(U_p, non_blocking=True)
            prob.eta_ext[:n_loc].copy_(E_p, non_blocking=True)
            step()
            G_p.copy_(prob.G, non_blocking=True)
            H_p.copy_(prob.Hv, non_blocking=True)
            F_p.copy_(prob.F, non_blocking=True)
        e2e_step()
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(e_steps):
            e2e_step()
        a1.record(stream)
        barrier()
        ems = a0.elapsed_time(a1) / e_steps
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": nnz * k / (ems * 1e-3) / 1e9, "unit": "GNNZ*k/s",
               "h2d_bytes_per_step": 2 * n * k * 8, "d2h_bytes_per_step": 2 * n * k * 8 + 8 * world,
               "ms_per_step": ems, "note": "bytes summed over ranks; time = max over ranks"}

    # ---- consistency: AB recomputed by the fused pass vs AB_in ----
    variants = None
    if not sharded:
        d = (AB_out - AB_in).abs().max().item() / AB_in.abs().max().item()
        log(f"[bench] AB_out vs AB_in max rel diff {d:.2e}")
        if not args.no_variants:
            variants = measure_variants(args, ctx, stream, plp, G, U, eta, Fb, AB_out, Gr, Hv, n, nnz, k, p,
                                        mode, eps, U_h, eta_h)

    if rank != 0:
        return
    cpu = None
    if not sharded and not args.no_cpu:
        v, dt, desc, cores = cpu_oracle_sample(g, k, p, eps, rows_frac=args.cpu_frac)
        v1, dt1 = cpu_oracle_single_thread(g, k, p, eps)
        cpu = {"value": v, "unit": "GNNZ*k/s", "cores": cores, "kind": "oracle", "sample": desc,
               "seconds": dt, "single_thread_value": v1, "single_thread_seconds": dt1,
               "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    out = {"metric": "fused grad+Hv GNNZ*k/s", "value": value, "unit": "GNNZ*k/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": args.config, "desc": CONFIG_DESC.get(args.config, args.config),
                      "n": n, "nnz": nnz, "k": k, "p": p, "eps": eps, "order": args.order,
                      "hessian": args.mode, "ab_in": "supplied (from plp_fgrad at the same U)",
                      "l2": "inputs (1.8 GB) larger than the 126 MB L2; no flush",
                      "parallelism": f"row-blocks x{world}", "nnz_local_rank0": nnz_local},
           "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
           "variants": variants,
           # per step: edge pass + finalize; collective: + F from the reduced A, B (+ 2 halo packs
           # when a peer needs rows; NCCL's own kernels are not counted)
           "gpu_launches": args.steps * (2 if not sharded else 3 + (2 if world > 1 else 0))}
    print(json.dumps(out), flush=True)


def measure_variants(args, ctx, stream, plp, G, U, eta, Fb, AB_out, Gr, Hv, n, nnz, k, p, mode, eps, U_h, eta_h):
    """the same call with AB_in == NULL (objective pass first: two edge passes),
    and the fused call on the generator-order numbering of the same graph (no locality ordering)."""
    import torch

    def timed(fn, reps):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    reps = max(3, min(args.steps, 10))
    out = {}
    ms = timed(lambda: plp.fgrad_hessvec_raw(ctx, G, k, U, eta, p, None, mode, eps, Fb, AB_out, Gr, Hv), reps)
    out["ab_in_null"] = {"ms_per_step": ms, "value": nnz * k / (ms * 1e-3) / 1e9, "unit": "GNNZ*k/s",
                         "note": "plp_fgrad_hessvec with AB_in == NULL: objective pass + fused pass"}
    try:
        g0 = get_graph_generator_order(args.config)
        G0 = plp.Graph(ctx, g0.row_ptr, g0.col, g0.w, flags=0)
        # the same random draws on the generator numbering (U, eta are iid: any labelling)
        ms = timed(lambda: plp.fgrad_hessvec_raw(ctx, G0, k, U, eta, p, AB_out, mode, eps, Fb, AB_out, Gr, Hv), reps)
        out["generator_order"] = {"ms_per_step": ms, "value": nnz * k / (ms * 1e-3) / 1e9, "unit": "GNNZ*k/s",
                                  "kernel": plp.last_edge_kernel(),
                                  "note": "the fused call on the graph in generator order (no RCM / tile ordering)"}
        del G0
    except Exception as e:  # pragma: no cover - informational only
        out["generator_order"] = {"error": repr(e)[:200]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="plp", choices=["plp", "reference"])
    ap.add_argument("--config", default="C5", choices=sorted(CONFIG_KP))
    ap.add_argument("--order", default="tile", choices=["tile", "rcm", "none"])
    ap.add_argument("--mode", default="sparse", choices=["sparse", "full"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="use the collective path (plp_create_graph_dist, in-library NCCL halo exchange and "
                         "all-reduce) even at one rank: exercises it on a single GPU")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the AB_in == NULL and generator-order timings")
    ap.add_argument("--cpu-frac", type=float, default=0.25)
    ap.add_argument("--ref-frac", type=float, default=1.0,
                    help="reference arm: fraction of the workload's rows per step (1.0: the whole workload)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # launched without torchrun: start the N ranks ourselves (one process per GPU), rank 0 prints
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    args.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: reporting n_gpus={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    dist_on = world > 1 or args.sharded
    if dist_on:
        import torch
        torch.cuda.set_device(args.local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{args.local_rank}"))
    try:
        run_plp(args, rank, world)
    finally:
        if dist_on:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
