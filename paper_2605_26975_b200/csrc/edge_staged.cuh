// Staged row kernel: the default fused F / EucGrad / EucHessianEta edge pass (SURVEY.md §8(a)
// a2-a7).  Same per-row arithmetic and summation order as edge_kernel.cuh (CSR
// order per row, one power per stored edge-column), with the latency chain of the row kernel
// taken apart:
//   * the CSR is cut into chunks of kChunkRows = 32 consecutive rows (the host's degree-sorting
//     window, plp_graph::sched); each warp owns a sequence of chunks (chunk = warp id + t * total
//     warps, a fixed assignment, so the CTA partial sums are deterministic);
//   * lane 0 of the warp stages a chunk's row_ptr slice, its schedule slice and its col / w
//     ranges into the warp's shared-memory ring with TMA bulk copies (cp.async.bulk + mbarrier,
//     kStages chunks in flight), so col/w never sit on the critical path of a row;
//   * the warp processes a chunk in passes of 32/LPR rows (degree-sorted, so the row groups of a
//     pass have near-equal degrees); a group of LPR lanes owns a row, lane li owns columns
//     [li*CPL, li*CPL + CPL);
//   * a row's edges go in batches of UNR: all UNR neighbour rows U_j, eta_j are gathered (one
//     IMAD.WIDE address per gather: 32-bit j times the compile-time row stride) before the batch
//     is computed; tail edges of a batch are skipped, not padded.
// Chunks whose col/w range exceeds the ring slot read col/w from global memory instead (same code,
// other source); rows leaving the fast power domain are recomputed exactly (edge_row_exact).
#pragma once
#include "async_copy.cuh"
#include "edge_kernel.cuh"

namespace plp {

constexpr int kChunkRows = kStagedChunk;  // rows per staged chunk (whole degree-sorting windows)
#ifndef PLP_STAGES
#define PLP_STAGES 2
#endif
constexpr int kStages = PLP_STAGES;
#ifndef PLP_STAGED_CPL8
#define PLP_STAGED_CPL8 4  // columns per lane at k = 8 (1, 2 or 4; tools/tune_edge.py)
#endif
#ifndef PLP_STAGED_PF
#define PLP_STAGED_PF 0  // 1: edge loop software-pipelined by one edge (UNR unused)
#endif
#ifndef PLP_STAGED_CONTIG
#define PLP_STAGED_CONTIG 0  // 1: each CTA sweeps a contiguous chunk range (measured slower)
#endif
#ifndef PLP_STAGED_L2PF
#define PLP_STAGED_L2PF 1  // L2 prefetch of each staged chunk's U / eta rows
#endif
#ifndef PLP_STAGED_UNR
#define PLP_STAGED_UNR 2
#endif

// Per-warp ring slot: row_ptr slice (kChunkRows + 8 ints), schedule slice (kChunkRows ints),
// col (cap + 16 ints), w (cap + 16 doubles).  cap % 4 == 0 keeps every piece 16-byte aligned.
constexpr unsigned kSlotRp = 0, kSlotSched = (kChunkRows + 8) * 4, kSlotCol = kSlotSched + kChunkRows * 4;
__host__ __device__ inline unsigned slot_w_off(int cap) { return kSlotCol + (unsigned)(cap + 16) * 4u; }
__host__ __device__ inline unsigned slot_bytes(int cap) { return slot_w_off(cap) + (unsigned)(cap + 16) * 8u; }
constexpr unsigned kBarBytes = 128;  // kEdgeThreads/32 warps x kStages mbarriers
static_assert((kEdgeThreads / 32) * kStages * 8 <= (int)kBarBytes, "mbarrier area");
__host__ __device__ inline unsigned staged_tab_off() { return kBarBytes; }
__host__ __device__ inline unsigned staged_coef_off(bool tables) {
  return kBarBytes + (tables ? (unsigned)((sizeof(PowTables) + 15) & ~(size_t)15) : 0u);
}
// coefficients (4 PLP_MAX_K doubles) + per-thread partial-sum slots (4 CPL doubles per thread)
__host__ __device__ inline unsigned staged_ring_off(bool tables, int cpl) {
  return staged_coef_off(tables) + (4u * PLP_MAX_K + 4u * cpl * kEdgeThreads) * 8u;
}
__host__ __device__ inline unsigned staged_smem_bytes(int cap, bool tables, int cpl) {
  return staged_ring_off(tables, cpl) + (unsigned)(kEdgeThreads / 32) * kStages * slot_bytes(cap);
}

// base + j * stride: one IMAD.WIDE.U32 per gather (32-bit j times the row stride, 64-bit base)
__device__ __forceinline__ const double* row_at(const double* base, int j, unsigned stride_bytes) {
  return reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) +
                                         (uint64_t)(uint32_t)j * stride_bytes);
}

// Capped form of one stored edge for rows with |d| < eps (the degenerate regime of the method:
// p-Laplacian minimisers are nearly constant on clusters, so neighbour differences fall below the
// curvature cap).  s_raw = |d|^{p-2} from the clamped fast power (valid for every |d| >= 2^-120 and
// for d = 0, where it is finite and multiplies d = 0), s_cap = min(s_raw, eps^{p-2}) (x^{p-2} is
// decreasing for p < 2, so the min is exactly the cap).  The CapRange flags 0 < |d| < 2^-120 and
// |d| >= 2^120 (exact path) and tells whether the fast form would have failed (next row's choice).
// Range tracker of the capped form: min |hi word|, min (|hi word| - 1) (zeros wrap to the top, so it
// is the minimum over nonzero differences) and max |hi word| over the row's differences.
struct CapRange {
  unsigned mn = ~0u, mnz = ~0u, mx = 0u;
  __device__ __forceinline__ bool bad() const { return (mnz < kHiMin - 1u) | (mx >= kHiMax); }
  // would the fast form (edge_update_mx) have failed on these differences?
  template <class POW>
  __device__ __forceinline__ bool fast_fails(const POW& pw) const {
    return (mn * 2u < pw.fast_lo2) | (mx * 2u - pw.fast_lo2 >= pw.fast_span2);
  }
};
template <int CPL, class POW, bool HAS_ETA, bool WANT_L = true>
__device__ __forceinline__ void edge_update_capsel(const POW& pw, double wv, const double (&ui)[CPL],
                                                   const double (&uj)[CPL], const double (&ei)[CPL],
                                                   const double (&ej)[CPL], double (&L)[CPL],
                                                   double (&HA)[CPL], CapRange& rg) {
  const double wcap = wv * pw.s_eps;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const double d = ui[c] - uj[c];
    const unsigned ahi = abs_hi(d);
    rg.mn = min(rg.mn, ahi);
    rg.mnz = min(rg.mnz, ahi - 1u);
    rg.mx = max(rg.mx, ahi);
    const double wsr = wv * pw.pow_fast(fmax(fabs(d), 0x1p-120));  // w |d|^{p-2}
    if constexpr (WANT_L) L[c] = fma(wsr, d, L[c]);                 // w phi_p(d)
    if constexpr (HAS_ETA) HA[c] = fma(fmin(wsr, wcap), ei[c] - ej[c], HA[c]);  // w cap(|d|)^{p-2}
  }
}

// One stored edge for the lane's CPL columns (branch-free); `mx` collects the fast-domain test
// (hi word of |d| relative to the lower bound, unsigned max: >= fast_span2 means some |d| left
// the domain and the row is recomputed exactly).
// WANT_L = false: the Hessian-vector-only passes skip the gradient sum L.
template <int CPL, class POW, bool HAS_ETA, bool WANT_L = true>
__device__ __forceinline__ void edge_update_mx(const POW& pw, double wv, const double (&ui)[CPL],
                                               const double (&uj)[CPL], const double (&ei)[CPL],
                                               const double (&ej)[CPL], double (&L)[CPL],
                                               double (&HA)[CPL], unsigned& mx) {
  unsigned h2[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const double d = ui[c] - uj[c];
    if constexpr (POW::kIsP2) {
      if constexpr (WANT_L) L[c] = fma(wv, d, L[c]);
      if constexpr (HAS_ETA) HA[c] = fma(wv, ei[c] - ej[c], HA[c]);
    } else {
      h2[c] = (unsigned)__double2hiint(d) * 2u - pw.fast_lo2;
      const double wsr = wv * pw.pow_fast(d);  // w |d|^{p-2}
      if constexpr (WANT_L) L[c] = fma(wsr, d, L[c]);  // w phi_p(d)
      if constexpr (HAS_ETA) HA[c] = fma(wsr, ei[c] - ej[c], HA[c]);
    }
  }
  if constexpr (!POW::kIsP2) {
    // three-input max (VIMNMX3) over the columns' domain tests
#pragma unroll
    for (int c = 0; c + 1 < CPL; c += 2) mx = max(mx, max(h2[c], h2[c + 1]));
    if constexpr (CPL % 2 == 1) mx = max(mx, h2[CPL - 1]);
  }
}

template <int KC, int CPL, int LPR, int UNR, class POW, bool HAS_ETA>
__global__ void __launch_bounds__(kEdgeThreads, PLP_EDGE_MINB) edge_staged_kernel(EdgeArgs a, POW pw) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NW = kEdgeThreads / 32;
  constexpr int RPW = 32 / LPR;               // rows per pass
  constexpr int NPASS = kChunkRows / RPW;     // passes per chunk
  static_assert(kChunkRows % RPW == 0, "chunk rows");
  if constexpr (POW::kNeedsTables) pw.init_smem(smem + staged_tab_off());
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane / LPR, li = lane % LPR;
  const int cap = a.chunk_cap;
  const unsigned sbytes = slot_bytes(cap);
  unsigned char* ring = smem + staged_ring_off(POW::kNeedsTables, CPL) + (size_t)warp * kStages * sbytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * kStages;
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();  // power tables and barriers visible

  const int k = KC > 0 ? KC : a.k;
  const unsigned kb = (unsigned)k * 8u;    // row stride of G, Hv (bytes)
  const unsigned xb = (unsigned)a.ldx * 8u; // row stride of U, eta (bytes)
  const int c0 = li * CPL;
  const bool active = c0 < k;
  const int n_rows = (int)a.n_rows;
  const int64_t n_chunks = (a.n_rows + kChunkRows - 1) / kChunkRows;
  // chunk sequence of this warp: cbeg, cbeg + cstep, ... < cend (a fixed assignment)
#if PLP_STAGED_CONTIG
  // each CTA sweeps its own contiguous range of chunks (warps interleaved within it), so the
  // neighbour rows of a tile-ordered graph are re-read from this SM's L1 while the sweep passes
  const int64_t cbeg = (int64_t)blockIdx.x * n_chunks / gridDim.x + warp, cstep = NW;
  const int64_t cend = ((int64_t)blockIdx.x + 1) * n_chunks / gridDim.x;
#else
  const int64_t cbeg = (int64_t)blockIdx.x * NW + warp, cstep = (int64_t)gridDim.x * NW;
  const int64_t cend = n_chunks;
#endif
  const int32_t* __restrict__ rp = a.rp;
  const double p = a.p;
  const double pp1 = p * (p - 1.0);

  // Row-epilogue coefficients in shared memory (registers go to the gathers): per column
  // (p/B, A/B, p(p-1)/B, p(p-1)A/B^2); the per-thread partial sums A', B', alpha, gamma live in
  // per-thread shared slots (updated once per row).
  double* coef = reinterpret_cast<double*>(smem + staged_coef_off(POW::kNeedsTables));
  // slot (q, c) of this thread at dslot[(q * CPL + c) * kEdgeThreads]: consecutive lanes hit
  // consecutive words (no bank conflicts), and the layout is the final reduction's
  double* dslot = coef + 4 * PLP_MAX_K + threadIdx.x;  // q = A', B', alpha, gamma
  for (int l = threadIdx.x; l < k; l += blockDim.x) {
    double cg = 0.0, cab = 0.0, cha = 0.0, chb = 0.0;
    if (a.AB != nullptr) {
      const double A = a.AB[l], B = a.AB[k + l];
      cg = p / B;
      cab = A / B;
      cha = pp1 / B;
      chb = pp1 * A / (B * B);
    }
    coef[4 * l + 0] = cg;
    coef[4 * l + 1] = cab;
    coef[4 * l + 2] = cha;
    coef[4 * l + 3] = chb;
  }
#pragma unroll
  for (int c = 0; c < 4 * CPL; ++c) dslot[c * kEdgeThreads] = 0.0;
  __syncthreads();

  // lane 0: stage chunk c (row_ptr bounds eb, ee) into ring slot s
  auto issue = [&](int s, int64_t c, int eb, int ee) {
    unsigned char* st = ring + (size_t)s * sbytes;
    const int r0 = (int)(c * kChunkRows);
    const int r1 = min(r0 + kChunkRows, n_rows);
    const unsigned rp_b = (unsigned)(((r1 + 1 + 3) & ~3) - r0) * 4u;  // r0 % 4 == 0
    const unsigned sc_b = (unsigned)(((r1 + 3) & ~3) - r0) * 4u;
    const int cb = eb & ~3, ce = (ee + 3) & ~3, wb = eb & ~1, we = (ee + 1) & ~1;
    const bool body = (ee - eb <= cap) && ce > cb;
    const unsigned col_b = body ? (unsigned)(ce - cb) * 4u : 0u;
    const unsigned w_b = body ? (unsigned)(we - wb) * 8u : 0u;
    mbar_expect_tx(&bars[s], rp_b + sc_b + col_b + w_b);
    tma_bulk_g2s(st + kSlotRp, rp + r0, rp_b, &bars[s]);
    tma_bulk_g2s(st + kSlotSched, a.sched + r0, sc_b, &bars[s]);
    if (body) {
      tma_bulk_g2s(st + kSlotCol, a.col + cb, col_b, &bars[s]);
      tma_bulk_g2s(st + slot_w_off(cap), a.w + wb, w_b, &bars[s]);
    }
#if PLP_STAGED_L2PF
    // warm L2 with the chunk's own U / eta rows: neighbour gathers of the rows processed before
    // this chunk then find them in L2 instead of HBM
    l2_prefetch_range(a.U + (int64_t)r0 * a.ldx, (size_t)(r1 - r0) * xb);
    if (a.eta != nullptr && a.eta != a.U + k)
      l2_prefetch_range(a.eta + (int64_t)r0 * a.ldx, (size_t)(r1 - r0) * xb);
#endif
  };
  if (lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      const int64_t c = cbeg + s * cstep;
      if (c < cend) {
        const int r0 = (int)(c * kChunkRows);
        issue(s, c, __ldg(rp + r0), __ldg(rp + min(r0 + kChunkRows, n_rows)));
      }
    }
  }

  const double* Ub = a.U + c0;    // the lane's columns of row 0
  const double* Eb = a.eta + c0;  // (unused without eta)
  for (int t = 0;; ++t) {
    const int64_t c = cbeg + (int64_t)t * cstep;
    if (c >= cend) break;
    const int s = t % kStages;
    // bounds of the chunk that will reuse this slot, loaded now and consumed after the passes
    const int64_t cn = c + (int64_t)kStages * cstep;
    int pb = 0, pe = 0;
    if (lane == 0 && cn < cend) {
      const int rn0 = (int)(cn * kChunkRows);
      pb = __ldg(rp + rn0);
      pe = __ldg(rp + min(rn0 + kChunkRows, n_rows));
    }
    mbar_wait(&bars[s], (unsigned)(t / kStages) & 1u);
    const unsigned char* st = ring + (size_t)s * sbytes;
    const int* rp_s = reinterpret_cast<const int*>(st + kSlotRp);
    const int* sc_s = reinterpret_cast<const int*>(st + kSlotSched);
    const int r0 = (int)(c * kChunkRows);
    const int nr = min(kChunkRows, n_rows - r0);
    const int eb = rp_s[0], ee = rp_s[nr];
    const bool staged = ee - eb <= cap;
    // smem views indexed by global CSR position
    const int* col_s = reinterpret_cast<const int*>(st + kSlotCol) - (eb & ~3);
    const double* w_s = reinterpret_cast<const double*>(st + slot_w_off(cap)) - (eb & ~1);

#pragma unroll 1
    for (int q = 0; q < NPASS; ++q) {
      const int lr = q * RPW + grp;
      if (!active || lr >= nr) continue;
      const int row = sc_s[lr];
      const int e0 = rp_s[row - r0], e1 = rp_s[row - r0 + 1];
      double ui[CPL], ei[CPL];
      ld_vec<CPL>(row_at(Ub, row, xb), ui);
      if constexpr (HAS_ETA) ld_vec<CPL>(row_at(Eb, row, xb), ei);
      double L[CPL], HA[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) L[cc] = HA[cc] = 0.0;
      unsigned mx = 0;
      // node terms sn = cap(|u|)^{p-2}, tn = |u|^{p-1} on the fast path (same domain test as
      // the edges: a row with |u| or some |d| outside it is recomputed exactly below)
      double sn[CPL], tn[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const double au = fabs(ui[cc]);
        if constexpr (POW::kIsP2) {
          sn[cc] = 1.0;
          tn[cc] = au;
        } else {
          mx = max(mx, (unsigned)__double2hiint(au) * 2u - pw.fast_lo2);
          sn[cc] = pw.pow_fast(au);
          tn[cc] = sn[cc] * au;
        }
      }
      auto edges = [&](const int* colp, const double* wp) {
        if constexpr (PLP_STAGED_PF) {
          // software-pipelined by one edge with ping-pong register buffers: the gathers of edge
          // e + 1 are in flight while edge e is computed (no register moves between iterations)
          if (e0 >= e1) return;
          double wa = wp[e0], wb = 0.0;
          double ua[CPL], ea[CPL], ub[CPL], eb_[CPL];
          ld_vec<CPL>(row_at(Ub, colp[e0], xb), ua);
          if constexpr (HAS_ETA) ld_vec<CPL>(row_at(Eb, colp[e0], xb), ea);
#pragma unroll 1
          for (int e = e0;;) {
            if (e + 1 < e1) {
              const int jn = colp[e + 1];
              wb = wp[e + 1];
              ld_vec<CPL>(row_at(Ub, jn, xb), ub);
              if constexpr (HAS_ETA) ld_vec<CPL>(row_at(Eb, jn, xb), eb_);
            }
            edge_update_mx<CPL, POW, HAS_ETA>(pw, wa, ui, ua, ei, ea, L, HA, mx);
            if (++e >= e1) break;
            if (e + 1 < e1) {
              const int jn = colp[e + 1];
              wa = wp[e + 1];
              ld_vec<CPL>(row_at(Ub, jn, xb), ua);
              if constexpr (HAS_ETA) ld_vec<CPL>(row_at(Eb, jn, xb), ea);
            }
            edge_update_mx<CPL, POW, HAS_ETA>(pw, wb, ui, ub, ei, eb_, L, HA, mx);
            if (++e >= e1) break;
          }
        } else {
#pragma unroll 1
        for (int e = e0; e < e1; e += UNR) {
          const int nrem = e1 - e;
          int j[UNR];
          double wv[UNR];
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            j[u] = colp[e + u];  // past e1: padding / the next row (unused)
            wv[u] = wp[e + u];
          }
          double uj[UNR][CPL], ej[UNR][CPL];
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            if (u < nrem) {
              ld_vec<CPL>(row_at(Ub, j[u], xb), uj[u]);
              if constexpr (HAS_ETA) ld_vec<CPL>(row_at(Eb, j[u], xb), ej[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < UNR; ++u) {
            if (u < nrem) edge_update_mx<CPL, POW, HAS_ETA>(pw, wv[u], ui, uj[u], ei, ej[u], L, HA, mx);
          }
        }
        }
      };
      if (staged) edges(col_s, w_s);
      else edges(a.col, a.w);
      if constexpr (!POW::kIsP2) {
        if (mx >= pw.fast_span2) {  // rare: exact libdevice recomputation of the row
          edge_row_exact<CPL, POW, HAS_ETA>(pw, e0, e1, a.col, a.w, a.U, a.eta, k, c0, ui, ei, L, HA);
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) pw.eval(fabs(ui[cc]), sn[cc], tn[cc]);
        }
      }

      // ---- row epilogue: node terms, outputs, partial sums ----
      double g[CPL], h[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        const double2 cf0 = reinterpret_cast<const double2*>(coef)[2 * (c0 + cc)];      // (p/B, A/B)
        const double2 cf1 = reinterpret_cast<const double2*>(coef)[2 * (c0 + cc) + 1];  // p(p-1)(1, A/B)/B
        const double au = fabs(ui[cc]);
        constexpr int T = kEdgeThreads;
        dslot[cc * T] = fma(ui[cc], L[cc], dslot[cc * T]);                  // A'
        dslot[(CPL + cc) * T] = fma(tn[cc], au, dslot[(CPL + cc) * T]);     // B'
        const double phi = copysign(tn[cc], ui[cc]);
        g[cc] = cf0.x * (L[cc] - cf0.y * phi);
        if constexpr (HAS_ETA) {
          h[cc] = cf1.x * HA[cc] - cf1.y * sn[cc] * ei[cc];
          if (a.want_dots) {
            dslot[(2 * CPL + cc) * T] = fma(p * phi, ei[cc], dslot[(2 * CPL + cc) * T]);  // alpha
            dslot[(3 * CPL + cc) * T] = fma(g[cc], ei[cc], dslot[(3 * CPL + cc) * T]);    // gamma
          }
        } else {
          h[cc] = 0.0;
        }
      }
      if (a.G != nullptr) st_vec<CPL>(const_cast<double*>(row_at(a.G + c0, row, kb)), g);
      if constexpr (HAS_ETA) {
        if (a.Hv != nullptr) st_vec<CPL>(const_cast<double*>(row_at(a.Hv + c0, row, kb)), h);
      }
    }
    __syncwarp();
    if (lane == 0 && cn < cend) {
      fence_proxy_async();  // the slot's generic reads are done before the async refill
      issue(s, cn, pb, pe);
    }
  }

  // ---- fixed-order CTA reduction of the per-thread partial-sum slots ----
  __syncthreads();
  const double* red = coef + 4 * PLP_MAX_K;
  const int nt = blockDim.x;
  for (int tt = threadIdx.x; tt < 4 * k; tt += nt) {
    const int q = tt / k, cl = tt % k;
    const int l = cl / CPL, cc = cl % CPL;
    const double* base = red + (q * CPL + cc) * nt;
    double sum = 0.0;
    for (int th = l; th < nt; th += LPR) sum += base[th];
    a.partials[((int64_t)blockIdx.x * 4 + q) * k + cl] = sum;
  }
}

// smem budget per CTA (PLP_EDGE_MINB CTAs per SM share ~220 KB)
constexpr unsigned kStagedSmemBudget = 220u * 1024u / PLP_EDGE_MINB;

// The ring slot capacity (edges per chunk) for a graph: its largest chunk, bounded by the budget.
inline int staged_cap(int max_chunk_nnz, bool tables, int cpl) {
  const unsigned avail = kStagedSmemBudget - staged_ring_off(tables, cpl);
  const unsigned per_slot = avail / ((kEdgeThreads / 32) * kStages);
  int cap_budget = (int)((per_slot - kSlotCol) / 12u) - 16;
  cap_budget &= ~3;
  int cap = (max_chunk_nnz + 3) & ~3;
  return cap < cap_budget ? cap : cap_budget;
}

template <int KC, int CPL, int LPR, class POW, bool HAS_ETA>
plp_status launch_staged_shape(plp_ctx* ctx, const EdgeArgs& a0, const POW& pw, int* grid_out) {
  constexpr int UNR = (CPL == 1) ? 2 * PLP_STAGED_UNR : (CPL == 2) ? PLP_STAGED_UNR : (PLP_STAGED_UNR + 1) / 2;
  auto kern = edge_staged_kernel<KC, CPL, LPR, UNR, POW, HAS_ETA>;
  EdgeArgs a = a0;
  if (a.ldx == 0) a.ldx = a.k;
  a.chunk_cap = staged_cap(a.max_chunk_nnz, POW::kNeedsTables, CPL);
  const unsigned smem = staged_smem_bytes(a.chunk_cap, POW::kNeedsTables, CPL);
  static unsigned attr_set_d[64] = {};  // per instantiation and device (the opt-in is per device)
  static int occ_d[64] = {};
  unsigned& attr_set = attr_set_d[ctx->device & 63];
  int& occ = occ_d[ctx->device & 63];
  if (attr_set < smem) {
    PLP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = smem;
    int o = 0;
    PLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kEdgeThreads, smem));
    occ = o < 1 ? 1 : o;
  }
  const int64_t n_chunks = (a.n_rows + kChunkRows - 1) / kChunkRows;
  const int64_t need = (n_chunks + kEdgeThreads / 32 - 1) / (kEdgeThreads / 32);
  int64_t grid = (int64_t)occ * ctx->num_sms;
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  if (need < grid) grid = need > 0 ? need : 1;
  kern<<<(int)grid, kEdgeThreads, smem, ctx->stream>>>(a, pw);
  PLP_LAUNCH_CHECK("edge_staged_kernel");
  note_edge_kernel("edge_staged_kernel", KC, CPL, LPR, UNR, POW::kName, HAS_ETA);
  *grid_out = (int)grid;
  return PLP_OK;
}

// Dispatch on k (and alignment) to a (KC, CPL, LPR) shape; compile-time k for k = 2, 4, 8, 16.
template <class POW>
plp_status launch_staged_pow(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid) {
  const int k = a.k;
  auto al = [](const void* ptr, unsigned b) { return ((uintptr_t)ptr & (b - 1)) == 0; };
  auto all_al = [&](unsigned b) {
    return al(a.U, b) && (a.eta == nullptr || al(a.eta, b)) && (a.G == nullptr || al(a.G, b)) &&
           (a.Hv == nullptr || al(a.Hv, b));
  };
  const bool vec_ok = (k % 2 == 0) && all_al(16);
  const bool vec4_ok = (k % 4 == 0) && all_al(32);  // 256-bit loads
  const bool he = a.eta != nullptr;
#define PLP_SSHAPE(KC, C, L)                                                              \
  return he ? launch_staged_shape<KC, C, L, POW, true>(ctx, a, pw, grid)                  \
            : launch_staged_shape<KC, C, L, POW, false>(ctx, a, pw, grid)
  if (vec_ok && k == 8) {
    if constexpr (PLP_STAGED_CPL8 == 4) {
      if (vec4_ok) PLP_SSHAPE(8, 4, 2);
    }
    if constexpr (PLP_STAGED_CPL8 == 1) PLP_SSHAPE(8, 1, 8);
    PLP_SSHAPE(8, 2, 4);
  }
#ifdef PLP_TUNE_ONLY
  return set_error(PLP_ERR_ARG, "tuning build: k = 8 only");
#else
  // all lanes busy for the configs' odd shapes: k = 20 as 4 lanes x 5 columns (C4), k = 3 as one
  // lane x 3 columns (C1)
  if (k == 20) PLP_SSHAPE(20, 5, 4);
  if (k == 3) PLP_SSHAPE(3, 3, 1);
  if (vec_ok) {
    if (k == 2) PLP_SSHAPE(2, 2, 1);
    if (k == 4) PLP_SSHAPE(4, 2, 2);
    if (k == 16) PLP_SSHAPE(16, 2, 8);
    const int half = k / 2;
    if (half <= 4) PLP_SSHAPE(0, 2, 4);
    if (half <= 8) PLP_SSHAPE(0, 2, 8);
    PLP_SSHAPE(0, 2, 16);
  }
  if (k <= 1) PLP_SSHAPE(0, 1, 1);
  if (k <= 2) PLP_SSHAPE(0, 1, 2);
  if (k <= 4) PLP_SSHAPE(0, 1, 4);
  if (k <= 8) PLP_SSHAPE(0, 1, 8);
  if (k <= 16) PLP_SSHAPE(0, 1, 16);
  PLP_SSHAPE(0, 1, 32);
#endif
#undef PLP_SSHAPE
}

}  // namespace plp
