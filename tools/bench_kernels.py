"""Per-row timing table (SURVEY.md §8(d) "also reported"): every kernel of the hot path on one
config, with its algorithmic bytes, achieved GB/s and fraction of the measured HBM peak; plus the
fused pass under the three node orderings (generator, RCM, tile).  CUDA events on the context's
stream, median of `reps` launches after warm-up.  Prints one JSON object per row.

  python tools/bench_kernels.py [--config C5] [--reps 20]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import get_graph, CONFIG_KP, load_peaks, algorithmic_bytes  # noqa: E402
from paper_2605_26975_b200 import plp  # noqa: E402
from plp_inputs import draw_U, draw_eta, draw_uniforms  # noqa: E402


def timed(fn, reps, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(stream)
    for i in range(reps):
        fn()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--orders", default="tile,rcm,natural")
    ap.add_argument("--oracle", action="store_true",
                    help="also time the CPU oracle for each row (bounded samples, scaled to the full size)")
    args = ap.parse_args()
    k, p = CONFIG_KP[args.config]
    peak, kind = load_peaks()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = plp.Context(0, stream)

    orc = {}

    def row(name, ms, byts, extra=None):
        gbs = byts / (ms * 1e-3) / 1e9
        d = {"config": args.config, "row": name, "ms": ms, "algorithmic_bytes": int(byts), "GBps": gbs,
             "frac_hbm": gbs / peak, "peak": peak, "peak_kind": kind}
        tag = name.split()[0] + (" full" if "full mode" in name else "") + (" seed" if "seeding" in name else "")
        if tag in orc and not any(x in name for x in ("(rcm order)", "(natural order)", "axpby")):
            o_ms, desc = orc[tag]
            d.update({"oracle_ms_full_size": o_ms, "oracle_sample": desc, "gpu_speedup_vs_oracle": o_ms / ms})
        if extra:
            d.update(extra)
        print(json.dumps(d), flush=True)

    if args.oracle:
        orc.update(oracle_rows(get_graph(args.config, "tile"), k, p))
    for order in args.orders.split(","):
        g = get_graph(args.config, order)
        n, nnz = g.n, g.nnz
        G = plp.Graph(ctx, g.row_ptr, g.col, g.w)
        U = torch.from_numpy(draw_U(n, k, 0)).cuda()
        E = torch.from_numpy(draw_eta(n, k, 0)).cuda()
        F, AB, _ = plp.fgrad(ctx, G, U, p, want_grad=False)
        Gr = torch.empty(n, k, dtype=torch.float64, device="cuda")
        Hv = torch.empty_like(Gr)
        csr = 12 * nnz + 4 * (n + 1)
        ms = timed(lambda: plp.edge_pass(ctx, G, U, E, p, 1e-9, AB_in=AB, G=Gr, Hv=Hv), args.reps, stream)
        row(f"a7 fused F/G/Hv edge pass ({order} order)", ms, algorithmic_bytes(n, nnz, k),
            {"kernel": plp.last_edge_kernel(), "GNNZk": nnz * k / (ms * 1e-3) / 1e9})
        if order != "tile":
            continue
        ms = timed(lambda: plp.fgrad(ctx, G, U, p, want_grad=False), args.reps, stream)
        row("a3 objective pass F, A, B (plp_fgrad, G = NULL)", ms, csr + 8 * n * k,
            {"kernel": plp.last_edge_kernel()})
        ms = timed(lambda: plp.edge_pass(ctx, G, U, None, p, 1e-9, AB_in=AB, G=Gr), args.reps, stream)
        row("a4 gradient pass with A, B supplied", ms, csr + 16 * n * k, {"kernel": plp.last_edge_kernel()})
        ms = timed(lambda: plp.hessvec(ctx, G, U, E, p, AB, Hv=Hv), args.reps, stream)
        row("a5 Hessian-vector product (sparse, Alg. 1)", ms, csr + 24 * n * k, {"kernel": plp.last_edge_kernel()})
        ms = timed(lambda: plp.hessvec(ctx, G, U, E, p, AB, mode=plp.HESS_FULL, G_in=Gr, Hv=Hv), args.reps, stream)
        row("a5+a6 Hessian-vector product (full mode: edge pass + rank-two epilogue)", ms,
            csr + 24 * n * k + 32 * n * k)
        Q = torch.empty_like(U)
        ms = timed(lambda: plp.project(ctx, U, Gr, out=Q), args.reps, stream)
        row("a8 Grassmann projection G - U (U^T G)", ms, 40 * n * k)
        ms = timed(lambda: plp.retract(ctx, U, Gr, Q=Q), args.reps, stream)
        row("a9 Cholesky-QR2 retraction", ms, 2 * 24 * n * k)
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        ms = timed(lambda: plp.dot(ctx, U, E, out=out), args.reps, stream)
        row("a10 dot <x, y>", ms, 16 * n * k)
        ms = timed(lambda: plp.axpby(ctx, 0.5, U, 0.5, Q), args.reps, stream)
        row("a10 axpby y = a x + b y", ms, 24 * n * k)
        u = draw_uniforms(1, k)
        labels, cent, sse, iters = plp.kmeans(ctx, U, k, u, restarts=1, max_iters=20, rel_tol=0.0)
        ms = timed(lambda: plp.kmeans(ctx, U, k, u, restarts=1, max_iters=20, rel_tol=0.0),
                   max(3, args.reps // 4), stream)
        ms0 = timed(lambda: plp.kmeans(ctx, U, k, u, restarts=1, max_iters=0), max(3, args.reps // 4), stream)
        lloyd = (ms - ms0) / max(iters, 1)
        row("a11 k-means Lloyd iteration (assign + centroid partials + update, host convergence check)",
            lloyd, 8 * n * k + 4 * n, {"lloyd_iters": iters})
        row(f"a11 k-means++ seeding + first assignment ({k - 1} D^2 rounds)", ms0, k * (8 * n * k + 8 * n))
        ms = timed(lambda: plp.rcut(ctx, G, k, labels), args.reps, stream)
        row("a12 RCut", ms, csr + 4 * n)
        tcg_rows(ctx, G, U, k, p, stream, row, csr)


def oracle_rows(g, k, p, frac=0.125):
    """The CPU oracle (as it stands, all host cores) per row: edge rows on the shard of the first
    frac of the rows (scaled by its share of nnz), dense rows on the full arrays, k-means on the
    first frac of the points (scaled by n), RCut on the full graph.  Returns {tag: (ms, desc)}."""
    import time
    import oracle
    from oracle import dense as odense
    from paper_2605_26975_b200 import plp as _plp
    oracle.set_threads(os.cpu_count() or 1)
    cores = oracle.get_threads()
    S = max(1, int(g.n * frac))
    halo, rp_loc, col_loc = _plp.halo_plan(g.row_ptr, g.col, 0, S)
    ext = np.concatenate([np.arange(S), halo])

    class Loc:
        row_ptr, col, w = rp_loc, col_loc, g.w[:g.row_ptr[S]]

    U = draw_U(g.n, k, 0)
    E = draw_eta(g.n, k, 0)
    Ul, El = U[ext], E[ext]
    scale = g.nnz / float(rp_loc[-1])
    out = {}

    def t(fn, reps=1):
        t0 = time.time()
        for _ in range(reps):
            r = fn()
        return (time.time() - t0) / reps * 1e3, r
    desc = f"rows [0,{S}) shard ({int(rp_loc[-1])} nnz), x{scale:.2f}, {cores} threads"
    ms, (F, A, B) = t(lambda: oracle.objective(Loc, Ul, p))
    out["a3"] = (ms * scale, desc)
    ms, _ = t(lambda: oracle.euc_grad(Loc, Ul, p, A, B))
    out["a4"] = (ms * scale, desc)
    ms, _ = t(lambda: oracle.hessvec(Loc, Ul, El, p, 1e-9, "sparse", (A, B)))
    out["a5"] = (ms * scale, desc)
    ms, _ = t(lambda: oracle.hessvec(Loc, Ul, El, p, 1e-9, "full", (A, B)))
    out["a5+a6 full"] = (ms * scale, desc)
    ms, _ = t(lambda: (oracle.objective(Loc, Ul, p), oracle.euc_grad(Loc, Ul, p, A, B),
                       oracle.hessvec(Loc, Ul, El, p, 1e-9, "sparse", (A, B))))
    out["a7"] = (ms * scale, desc)
    dd = f"full {g.n} x {k} arrays (numpy)"
    out["a8"] = (t(lambda: odense.project(U, E))[0], dd)
    out["a9"] = (t(lambda: odense.retract(U, E))[0], dd)
    out["a10"] = (t(lambda: odense.dot(U, E))[0], dd)
    Xs = U[:S]
    u = draw_uniforms(1, k)
    m0, _ = t(lambda: oracle.kmeans(Xs, k, u, restarts=1, max_iters=0))
    m3, _ = t(lambda: oracle.kmeans(Xs, k, u, restarts=1, max_iters=3, rel_tol=0.0))
    kd = f"first {S} points, x{g.n / S:.1f}"
    out["a11"] = ((m3 - m0) / 3 * g.n / S, kd)
    out["a11 seed"] = (m0 * g.n / S, kd)
    lab = (np.arange(g.n) * k // g.n).astype(np.int32)
    out["a12"] = (t(lambda: oracle.rcut(g, lab, k))[0], f"full graph, {cores} threads")
    return out


def tcg_rows(ctx, G, U, k, p, stream, row, csr):
    """One truncated-CG iteration (NEXT-1): Hessian-vector product, projection, curvature term,
    two dots, four axpbys -- device-resident (plp_tcg_run, no host read) and host-driven (two
    scalar reads per iteration).  kappa = 0 keeps tCG from converging so every iteration runs."""
    from paper_2605_26975_b200 import solver
    n = G.n_rows
    cfg = solver.SolverConfig(tcg_kappa=0.0, tcg_max_iters=10)
    Uq = plp.retract(ctx, U, torch.zeros_like(U))
    tr = solver.GrassmannTR(ctx, G, k, cfg)
    st = solver._State(tr, Uq, p)
    tr.tcg_device(st, p, 1e6)
    eta, Heta, r, dlt, Hd, scal, status = tr._tcg_buf
    iters = 10

    def dev(fused):
        Hacc = None if fused else Heta  # the solver's fused path accumulates no H step
        plp.tcg_init(ctx, st.grad, 1e6, 0.0, 1.0, eta, Hacc, r, dlt, scal, status)
        plp.tcg_run(ctx, G, st.U, st.AB, None, st.S, p, cfg.eps, plp.HESS_SPARSE, eta, Hacc, r, dlt, Hd,
                    scal, status, 1 << 30, iters, fused=fused)
    ms = timed(lambda: dev(False), 5, stream) / iters
    # per iteration: edge pass (csr + U, eta, Hd), project (40 n k), apply_sub (24 n k),
    # dots (2 x 16 n k), axpbys (4 x 24 n k), projection of r (40 n k)
    byts = csr + 24 * n * k + 40 * n * k + 24 * n * k + 32 * n * k + 96 * n * k + 40 * n * k
    row("NEXT-1 tCG iteration, device-resident (plp_tcg_run)", ms, byts)
    if k in (8, 16):
        # fused: edge pass + pass A (U, EH, d: 24 n k) + pass B (U, EH, d, eta, r read, two written:
        # 56 n k; no H step) + pass C (U, r, d read, r, d written: 40 n k)
        ms = timed(lambda: dev(True), 5, stream) / iters
        row("NEXT-2 tCG iteration, fused passes (plp_tcg_run fused=1, no H step)", ms, csr + 24 * n * k + 120 * n * k)
    res = {}

    def host():
        res["r"] = tr.tcg(st, p, 1e6)
    ms = timed(host, 5, stream)
    nit = res["r"][2]
    row(f"NEXT-1 tCG iteration, host-driven loop ({res['r'][3]} after {nit})", ms / max(nit, 1), byts)


if __name__ == "__main__":
    main()
