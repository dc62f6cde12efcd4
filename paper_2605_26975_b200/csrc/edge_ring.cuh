// Ring-gather edge kernel: the fused F / EucGrad / EucHessianEta pass for
// wide rows without locality (C4: k = 20, a 10-D kNN graph whose 224-row tiles touch ~2,100 outside
// rows, so halo tiles do not apply and every neighbour row is an L2 gather).
//
// The row kernel (edge_kernel.cuh) gathers a batch of neighbour rows into registers right before
// using them: ~2.5 KB in flight per warp, far from the ~130 KB per SM that hides the L2 latency at
// this gather rate, and deeper register batches spill.  Here each warp streams its neighbour rows
// through a private shared-memory ring instead: while it computes batch b, the copies of batches
// b+1 .. b+S-1 are in flight (cp.async, 16 B per lane, SASS LDGSTS), so the bytes in flight are
// bounded by shared memory, not registers.
//   * a pass = RPW rows of the degree-sorted schedule (one row per group of LPR lanes, CPL columns
//     per lane); a batch = E consecutive edges of each of the pass's rows; the batch's RPW*E
//     neighbour rows of U and eta (and, in a pass's first batch, the pass's own rows) land in one
//     ring stage;
//   * fetch and compute run the same sequence of (pass, batch) items, the fetch S - 1 items ahead
//     (across pass boundaries), one cp.async group per item;
//   * per-row arithmetic, summation order (CSR order within the row) and the exact libdevice
//     recomputation of rows leaving the fast power domain are those of the row kernel.
#pragma once
#include "async_copy.cuh"
#include "edge_kernel.cuh"
#include "edge_staged.cuh"

namespace plp {

constexpr int kRingThreads = 256;  // 8 warps; two CTAs per SM
#ifndef PLP_RING_E
#define PLP_RING_E 4  // edges per row per batch
#endif
#ifndef PLP_RING_S
#define PLP_RING_S 3  // ring stages (items in flight: S - 1 ahead of the one computed)
#endif

template <int K>
struct RingShape {
  static constexpr int CPL = 2, LPR = K / CPL, RPW = 32 / LPR, E = PLP_RING_E, S = PLP_RING_S;
  static constexpr int SLOTS = RPW * E;                    // neighbour rows per stage
  static constexpr int ROWB = K * 8;                       // bytes per U (or eta) row
  static constexpr int PIECES = ROWB / 16;                 // 16-byte pieces per row
  // stage: [SLOTS + RPW own rows][U | eta][K] doubles, then SLOTS weights
  static constexpr int STAGE_ROWS = SLOTS + RPW;
  static constexpr int W_OFF = STAGE_ROWS * 2 * ROWB;
  static constexpr int STAGE_BYTES = W_OFF + SLOTS * 8;
  static constexpr int WARP_BYTES = S * STAGE_BYTES;
  static_assert(K % 4 == 0 && RPW >= 1, "ring shape");
};

template <int K, class POW, bool HAS_ETA>
__global__ void __launch_bounds__(kRingThreads, 2) edge_ring_kernel(EdgeArgs a, POW pw) {
  using R = RingShape<K>;
  constexpr int CPL = R::CPL, LPR = R::LPR, RPW = R::RPW, E = R::E, S = R::S;
  extern __shared__ __align__(16) unsigned char smem[];
  if constexpr (POW::kNeedsTables) {
    pw.init_smem(smem);
    __syncthreads();
  }
  const unsigned tab = POW::kNeedsTables ? (unsigned)((sizeof(PowTables) + 127) & ~(size_t)127) : 0u;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = smem + tab + (size_t)warp * R::WARP_BYTES;
  const int grp = lane / LPR, li = lane % LPR, c0 = li * CPL;
  const bool active = grp < RPW;
  const double p = a.p, pp1 = p * (p - 1.0);
  double cG[CPL], cAB[CPL], cHA[CPL], cHB[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    cG[c] = cAB[c] = cHA[c] = cHB[c] = 0.0;
    if (a.AB != nullptr) {
      const double A = a.AB[c0 + c], B = a.AB[K + c0 + c];
      cG[c] = p / B;
      cAB[c] = A / B;
      cHA[c] = pp1 / B;
      cHB[c] = pp1 * A / (B * B);
    }
  }
  double accA[CPL], accB[CPL], accAl[CPL], accGa[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) accA[c] = accB[c] = accAl[c] = accGa[c] = 0.0;

  const int64_t n = a.n_rows;
  const int64_t stride = (int64_t)gridDim.x * (kRingThreads / 32) * RPW;
  const int64_t first = ((int64_t)blockIdx.x * (kRingThreads / 32) + warp) * RPW;
  // pass metadata held by lanes 0..RPW-1 (lane g: row g of the pass): row, e0, e1
  struct Pass {
    int64_t base;  // schedule index of row 0
    int row, e0, e1, nb;  // (lane g's row) ; nb = batches of the pass (warp-uniform)
  };
  auto load_pass = [&](int64_t base) {
    Pass P;
    P.base = base;
    P.row = 0;
    P.e0 = P.e1 = 0;
    if (lane < RPW && base + lane < n) {
      P.row = __ldg(a.sched + base + lane);
      P.e0 = __ldg(a.rp + P.row);
      P.e1 = __ldg(a.rp + P.row + 1);
    }
    int deg = P.e1 - P.e0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) deg = max(deg, __shfl_xor_sync(0xffffffffu, deg, o));
    P.nb = base < n ? max(1, (deg + E - 1) / E) : 0;
    return P;
  };

  // ---- fetch cursor: issue the copies of item (fp, fb) into stage fs ----
  Pass fp = load_pass(first);
  int fb = 0, fs = 0;
  auto fetch = [&]() {
    unsigned char* st = ring + (size_t)fs * R::STAGE_BYTES;
    if (fp.base < n) {
      // lane l < SLOTS: slot l = (row g = l / E, edge q = l % E) of the batch
      const int g = min(lane / E, RPW - 1), q = lane % E;
      const int e0 = __shfl_sync(0xffffffffu, fp.e0, g), e1 = __shfl_sync(0xffffffffu, fp.e1, g);
      const int rowg = __shfl_sync(0xffffffffu, fp.row, g);
      int j = rowg;
      if (lane < R::SLOTS) {
        const int e = e0 + fb * E + q;
        const bool v = e < e1 && fp.base + g < n;
        // padding: a copy of the row's last edge with weight 0 (exact zero contributions, and the
        // same |d| as a real edge for the fast-domain test); an edgeless row pads with itself
        j = v ? __ldg(a.col + e) : (e1 > e0 ? __ldg(a.col + e1 - 1) : rowg);
        reinterpret_cast<double*>(st + R::W_OFF)[lane] = v ? __ldg(a.w + e) : 0.0;
      }
      // own rows of the pass in its first batch (slots SLOTS .. SLOTS + RPW - 1)
      const int nslot = R::SLOTS + (fb == 0 ? RPW : 0);
      const int npieces = nslot * 2 * R::PIECES;
      for (int pc = lane; pc < ((R::STAGE_ROWS * 2 * R::PIECES + 31) & ~31); pc += 32) {
        const int slot = min(pc / (2 * R::PIECES), R::STAGE_ROWS - 1), rem = pc % (2 * R::PIECES);
        const int arr = rem / R::PIECES, part = rem % R::PIECES;
        const int vj = __shfl_sync(0xffffffffu, j, min(slot, 31));
        const int vr = __shfl_sync(0xffffffffu, fp.row, slot >= R::SLOTS ? slot - R::SLOTS : 0);
        const int jj = slot < R::SLOTS ? vj : vr;
        if (pc < npieces && (arr == 0 || HAS_ETA)) {
          const double* src = (arr == 0 ? a.U : a.eta) + (int64_t)jj * K + part * 2;
          cp_async16(st + ((size_t)slot * 2 + arr) * R::ROWB + part * 16, src);
        }
      }
    }
    cp_async_commit();  // one group per item (empty past the end: keeps the group count uniform)
    fs = (fs + 1) % S;
    if (++fb >= fp.nb && fp.base < n) {
      fp = load_pass(fp.base + stride);
      fb = 0;
    }
  };
  for (int s = 0; s < S - 1; ++s) fetch();

  // ---- compute cursor ----
  int64_t cbase = first;
  int cs = 0;
  while (cbase < n) {
    const Pass cp = load_pass(cbase);  // same metadata the fetch cursor saw (L1 hits)
    const int e0 = __shfl_sync(0xffffffffu, cp.e0, active ? grp : 0);
    const int e1 = __shfl_sync(0xffffffffu, cp.e1, active ? grp : 0);
    const int row = __shfl_sync(0xffffffffu, cp.row, active ? grp : 0);
    const bool has_row = active && cbase + grp < n;
    double ui[CPL], ei[CPL], L[CPL], HA[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) ui[c] = ei[c] = L[c] = HA[c] = 0.0;
    unsigned mx = 0;
    for (int b = 0; b < cp.nb; ++b) {
      fetch();                       // item S - 1 ahead
      cp_async_wait_group<S - 1>();  // this item's copies have landed (ours; __syncwarp: everyone's)
      __syncwarp();
      const unsigned char* st = ring + (size_t)cs * R::STAGE_BYTES;
      if (b == 0) {
        lds_vec<CPL>(reinterpret_cast<const double*>(st + ((size_t)(R::SLOTS + grp) * 2 + 0) * R::ROWB) + c0, ui);
        if constexpr (HAS_ETA)
          lds_vec<CPL>(reinterpret_cast<const double*>(st + ((size_t)(R::SLOTS + grp) * 2 + 1) * R::ROWB) + c0, ei);
      }
      if (has_row) {
        const double* wst = reinterpret_cast<const double*>(st + R::W_OFF);
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const int slot = grp * E + q;
          double uj[CPL], ej[CPL];
          lds_vec<CPL>(reinterpret_cast<const double*>(st + ((size_t)slot * 2 + 0) * R::ROWB) + c0, uj);
          if constexpr (HAS_ETA)
            lds_vec<CPL>(reinterpret_cast<const double*>(st + ((size_t)slot * 2 + 1) * R::ROWB) + c0, ej);
          edge_update_mx<CPL, POW, HAS_ETA>(pw, wst[slot], ui, uj, ei, ej, L, HA, mx);
        }
      }
      __syncwarp();  // stage cs free for the fetch S - 1 items later
      cs = (cs + 1) % S;
    }
    if (has_row) {
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
      if constexpr (!POW::kIsP2) {
        if (mx >= pw.fast_span2) {  // rare: exact recomputation of the row
          edge_row_exact<CPL, POW, HAS_ETA>(pw, e0, e1, a.col, a.w, a.U, a.eta, K, c0, ui, ei, L, HA);
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) pw.eval(fabs(ui[cc]), sn[cc], tn[cc]);
        }
      }
      double g[CPL], hv[CPL];
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        accA[cc] = fma(ui[cc], L[cc], accA[cc]);
        accB[cc] = fma(tn[cc], fabs(ui[cc]), accB[cc]);
        const double phi = copysign(tn[cc], ui[cc]);
        g[cc] = cG[cc] * (L[cc] - cAB[cc] * phi);
        if constexpr (HAS_ETA) {
          hv[cc] = cHA[cc] * HA[cc] - cHB[cc] * sn[cc] * ei[cc];
          if (a.want_dots) {
            accAl[cc] = fma(p * phi, ei[cc], accAl[cc]);
            accGa[cc] = fma(g[cc], ei[cc], accGa[cc]);
          }
        } else {
          hv[cc] = 0.0;
        }
      }
      if (a.G != nullptr) st_vec<CPL>(a.G + (int64_t)row * K + c0, g);
      if constexpr (HAS_ETA) {
        if (a.Hv != nullptr) st_vec<CPL>(a.Hv + (int64_t)row * K + c0, hv);
      }
    }
    cbase += stride;
  }
  cp_async_wait_all();

  // ---- fixed-order CTA reduction (reuses the rings) ----
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem + tab);  // [4][CPL][threads]
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) {
    red[(0 * CPL + cc) * kRingThreads + threadIdx.x] = active ? accA[cc] : 0.0;
    red[(1 * CPL + cc) * kRingThreads + threadIdx.x] = active ? accB[cc] : 0.0;
    red[(2 * CPL + cc) * kRingThreads + threadIdx.x] = active ? accAl[cc] : 0.0;
    red[(3 * CPL + cc) * kRingThreads + threadIdx.x] = active ? accGa[cc] : 0.0;
  }
  __syncthreads();
  for (int tt = threadIdx.x; tt < 4 * K; tt += kRingThreads) {
    const int q = tt / K, cl = tt % K;
    const int l = cl / CPL, cc = cl % CPL;
    const double* base = red + (q * CPL + cc) * kRingThreads;
    double sum = 0.0;
    for (int w = 0; w < kRingThreads / 32; ++w)
      for (int gg = 0; gg < RPW; ++gg) sum += base[w * 32 + gg * LPR + l];
    a.partials[((int64_t)blockIdx.x * 4 + q) * K + cl] = sum;
  }
}

template <int K, class POW, bool HAS_ETA>
plp_status launch_ring_shape(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid_out) {
  using R = RingShape<K>;
  auto kern = edge_ring_kernel<K, POW, HAS_ETA>;
  const size_t tab = POW::kNeedsTables ? ((sizeof(PowTables) + 127) & ~(size_t)127) : 0;
  const size_t red = (size_t)4 * R::CPL * kRingThreads * 8;
  const size_t ring = (size_t)(kRingThreads / 32) * R::WARP_BYTES;
  const size_t smem = tab + (ring > red ? ring : red);
  static unsigned attr_set[64] = {};
  static int occ_d[64] = {};
  unsigned& set_to = attr_set[ctx->device & 63];
  int& occ = occ_d[ctx->device & 63];
  if (set_to < smem) {
    PLP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set_to = (unsigned)smem;
    int o = 0;
    PLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kRingThreads, smem));
    occ = o < 1 ? 1 : o;
  }
  const int64_t rows_per_cta = (kRingThreads / 32) * R::RPW;
  const int64_t need = (a.n_rows + rows_per_cta - 1) / rows_per_cta;
  int64_t grid = (int64_t)occ * ctx->num_sms;
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  if (need < grid) grid = need > 0 ? need : 1;
  kern<<<(int)grid, kRingThreads, smem, ctx->stream>>>(a, pw);
  PLP_LAUNCH_CHECK("edge_ring_kernel");
  note_edge_kernel("edge_ring_kernel", K, R::CPL, R::LPR, R::E, POW::kName, HAS_ETA);
  *grid_out = (int)grid;
  return PLP_OK;
}

// k = 20 rows without halo tiles (C4); contiguous, 16-byte aligned arrays.
template <class POW>
plp_status try_launch_ring(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid, bool* used) {
  *used = false;
  auto al16 = [](const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; };
  if (a.k != 20 || (a.ldx != 0 && a.ldx != a.k) || !al16(a.U) || (a.eta && !al16(a.eta)) ||
      (a.G && !al16(a.G)) || (a.Hv && !al16(a.Hv)))
    return PLP_OK;
  *used = true;
  return a.eta ? launch_ring_shape<20, POW, true>(ctx, a, pw, grid)
               : launch_ring_shape<20, POW, false>(ctx, a, pw, grid);
}

}  // namespace plp
