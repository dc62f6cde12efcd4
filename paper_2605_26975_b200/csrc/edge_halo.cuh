// Halo-tile edge kernel: the fused F / EucGrad / EucHessianEta pass (
// DESIGN.md §5) with every neighbour row served from shared memory.
//
// The rows are cut into tiles of kHaloT = PLP_HALO_TILE (240) consecutive rows.  plp_create_graph
// lists, per tile, the distinct columns outside it (the tile's halo, ordered by decreasing number
// of references) and re-encodes every stored edge as a tile-local index: j - r0 for an internal
// neighbour, kHaloT + x for the x-th halo row.  One persistent CTA of 16 warps per SM walks the
// tiles (interleaved across CTAs, so neighbouring tiles are in flight together and the halo rows
// hit L2), double-buffered:
//   * a producer warp (warp specialisation: 15 consumer warps + 1) stages each tile: lane 0 issues
//     TMA bulk copies (cp.async.bulk + mbarrier) of the tile's own U / eta rows, row_ptr and
//     schedule slices, (enc, w) ranges, and two tiles ahead the tile's halo list; the 32 lanes
//     gather the halo rows U_j, eta_j with cp.async (16-byte pieces, 8 rows per instruction at
//     k = 8) whose cp.async.mbarrier.arrive joins the TMA bytes on the buffer's "full" mbarrier;
//     a tile whose halo exceeds the staged rows (overflow mode) leaves its least referenced halo
//     rows in L2, where the consumers read them;
//   * consumers release a buffer with one arrival per warp on its "empty" mbarrier; there is no
//     CTA-wide barrier per tile, so a warp that finishes early goes on with the next (resident)
//     tile; while tile i is computed, tile i + 1 is resident and tile i + 2 is in flight.
// Rows are processed as in the row kernels (one group of LPR lanes per row, CPL = 2 columns per
// lane at k = 4, 8, 4 at k = 16; CSR order per row, one power per stored edge-column, edges in
// pairs), reading U_j / eta_j with 32-bit shared-window loads, so the only global traffic is the
// streaming of the tile data and the G / Hv stores.  The tile's degree-sorted rows form slices of
// 32 / LPR rows dealt to the warps in snake order (a heavy and a light slice per warp).
#pragma once
#include "async_copy.cuh"
#include "dense_mma.cuh"
#include "edge_kernel.cuh"
#include "edge_staged.cuh"

namespace plp {

constexpr int kHaloT = PLP_HALO_TILE;  // rows per tile (plp.h)
constexpr int kHaloProd = 1;  // producer warps (2, splitting the halo gathers, measured slower)
constexpr int kHaloCWarps = kHaloT / 16;  // consumers: two slices of 8 rows each per tile
constexpr int kHaloThreads = (kHaloCWarps + kHaloProd) * 32;  // + the producer warp(s)
static_assert(kHaloT % kSchedWindow == 0 && kHaloThreads <= 1024, "tile map");

// CPL doubles at shared-window address addr + OFF (16-byte aligned for even CPL)
template <unsigned OFF>
__device__ __forceinline__ void lds_pair(unsigned addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(a), "=d"(b) : "r"(addr), "n"(OFF));
}
template <int CPL, unsigned OFF>
__device__ __forceinline__ void lds_row(unsigned addr, double (&v)[CPL]) {
  static_assert(CPL == 2 || CPL == 4, "halo kernel: 2 or 4 columns per lane");
  lds_pair<OFF>(addr, v[0], v[1]);
  if constexpr (CPL == 4) lds_pair<OFF + 16u>(addr, v[2], v[3]);
}

// Per-buffer shared-memory layout (bytes), identical on host and device.
struct HaloLayout {
  unsigned rp, sched, nl, enc, w, U, E, bytes;
};
// Staged halo rows per tile at most (the U / eta row blocks have a fixed size, so the eta rows sit
// at a compile-time offset from the U rows and the consumers address both with one register);
// tiles with more halo rows run in overflow mode.
#ifndef PLP_HALO_CAP8
#define PLP_HALO_CAP8 380
#endif
#ifndef PLP_HALO_CAP16
#define PLP_HALO_CAP16 64
#endif
__host__ __device__ constexpr int halo_rows_cap(int k) { return k <= 4 ? 800 : k == 8 ? PLP_HALO_CAP8 : PLP_HALO_CAP16; }

__host__ __device__ inline HaloLayout halo_layout(int k, int ext_cap, int nnz_cap, bool obj = false,
                                                  bool eta = true) {
  HaloLayout L;
  (void)ext_cap;
  unsigned o = 0;
  L.U = o; o += (unsigned)(kHaloT + halo_rows_cap(k)) * (unsigned)k * 8u;
  L.E = o; o += eta ? (unsigned)(kHaloT + halo_rows_cap(k)) * (unsigned)k * 8u : 0u;
  L.rp = o; o += (kHaloT + 8) * 4;
  L.sched = o; o += kHaloT * 4;
  L.nl = o; o += obj ? (kHaloT + 8) * 4 : 0u;  // lower-edge counts (objective mode only)
  L.enc = o; o += (unsigned)(nnz_cap + 16) * 4;
  o = (o + 15u) & ~15u;
  L.w = o; o += (unsigned)(nnz_cap + 16) * 8;
  L.bytes = (o + 127u) & ~127u;
  return L;
}
#ifndef PLP_HALO_NBUF
#define PLP_HALO_NBUF 2  // tile buffers in flight (2 or 3)
#endif
#ifndef PLP_HALO_NBUF_NOETA
#define PLP_HALO_NBUF_NOETA 3  // passes without eta (objective, gradient) stage half the rows: 3 buffers
#endif
constexpr int kHaloNBuf = PLP_HALO_NBUF;
#ifndef PLP_HALO_COEF_SMEM
#define PLP_HALO_COEF_SMEM 0  // 1: the row epilogue's A, B coefficients in shared memory (16 registers)
#endif
// mbarriers (full[NBUF], list[3], empty[NBUF]) in the first 256 bytes, the epilogue coefficients
// (PLP_HALO_COEF_SMEM: [4][k <= 16] doubles) after them; tables follow
constexpr unsigned kHaloHead = PLP_HALO_COEF_SMEM ? 256 + 4 * 16 * 8 : 256;
__host__ __device__ inline unsigned halo_tab_bytes(bool tables) {
  return tables ? (unsigned)((sizeof(PowTables) + 127) & ~(size_t)127) : 0u;
}
__host__ __device__ inline unsigned halo_lists_off(bool tables) { return kHaloHead + halo_tab_bytes(tables); }
__host__ __device__ inline unsigned halo_bufs_off(int ext_cap, bool tables) {
  return (halo_lists_off(tables) + 3u * (unsigned)(ext_cap + 4) * 4u + 127u) & ~127u;
}
__host__ __device__ inline unsigned halo_smem_bytes(int k, int ext_cap, int nnz_cap, bool tables,
                                                    bool obj = false, bool eta = true, int nbuf = kHaloNBuf) {
  return halo_bufs_off(ext_cap, tables) + (unsigned)nbuf * halo_layout(k, ext_cap, nnz_cap, obj, eta).bytes;
}
#ifndef PLP_HALO_CTAS
#define PLP_HALO_CTAS 1  // resident CTAs per SM (each with its own double buffer)
#endif
constexpr unsigned kHaloSmemMax = 225u * 1024u / PLP_HALO_CTAS;

#ifndef PLP_HALO_SLEEP_NS
#define PLP_HALO_SLEEP_NS 64  // producer back-off between polls of the "empty" barrier
#endif
#ifndef PLP_HALO_CPL8
#define PLP_HALO_CPL8 2  // k = 8 columns per lane outside the Hessian-vector-only passes (2 or 4)
#endif
// columns per lane: 4 at k = 16, 2 at k = 4, 8.  PLP_HALO_CPL8=4 (k = 8 passes with a gradient or
// objective: 2 lanes per row, one edge per iteration, four independent power chains per lane,
// 7 % fewer instructions) measured slower on C5: 0.928 against 0.823 ms (16 rows per warp pass
// and one slice per warp per tile); the Hessian-vector-only passes (and their pass-A fold, which
// needs the 2-column accumulator layout) always take 2 (k = 8: 1 column per lane measured slower)
template <int K, bool HVO = false>
constexpr int halo_cpl() { return K == 16 ? 4 : (K == 8 && !HVO) ? PLP_HALO_CPL8 : 2; }

// OBJ: objective-only pass (no eta, no G) on a symmetric graph: A_l = sum over the upper-triangle
// edges (j > i) of w_ij |u_il - u_jl|^p, i.e. Eq. (1)'s numerator with each undirected edge once
// (half the powers of the row form); B_l from the node terms as usual.
// ADAPT: rows that leave the fast domain (mostly |d| < eps: the solver's degenerate regime, where
// p-Laplacian iterates flatten on clusters) are recomputed from shared memory in the capped form,
// and a warp whose previous pass needed it goes there directly; libdevice only for |d| < 2^-120 or
// >= 2^120.  Off for the fused F/G/Hv pass (the benchmark unit; its random inputs rarely leave the
// domain, and the plain loop keeps its code), which recomputes such rows with libdevice.
#ifdef PLP_HALO_TRACE
// Pipeline trace (tools/trace_halo.py; a build flag, never in the product build): clock64 per tile
// iteration: [0] producer past the "empty" wait, [1] producer done issuing, [2 + w] consumer warp w
// past the "full" wait, [16 + w] consumer warp w released the buffer, [32..34] producer past the
// list wait / done with the TMA copies / done with the halo gathers.
constexpr int kTraceTiles = 320, kTraceSlots = 36;
static __device__ long long g_halo_trace[160 * kTraceTiles * kTraceSlots];
#define PLP_TRACE(it, slot)                                                                         \
  do {                                                                                              \
    if ((it) < kTraceTiles && blockIdx.x < 160)                                                     \
      g_halo_trace[((int64_t)blockIdx.x * kTraceTiles + (it)) * kTraceSlots + (slot)] = clock64();  \
  } while (0)
#else
#define PLP_TRACE(it, slot) do {} while (0)
#endif

// DOTS: also accumulate the full-mode dots alpha, gamma (a.want_dots; a template flag so that the
// sparse passes carry no code for them).
// OVF: some tile's halo exceeds what fits in shared memory (a.halo_stage rows are staged, the rest
// -- the tile's least referenced halo rows, the list being ordered by reference count -- are read
// from global memory / L2 by the consumers; C3's random long-range edges).
// HVO: Hessian-vector product only (plp_hessvec, sparse mode: no gradient sum L, no A, B partials).
// GRAM (HVO at k = 4, 8; the fused tCG, tcg.cu): pass A of the tCG iteration folded into the row
// epilogue.  A warp's row pass holds an 8 x 8 block X[g][2q + h] (lane 4g + q, column pair h) of
// U, d = eta and EH = Hv -- k = 8: row g is the pass's g-th row; k = 4: the rows of groups 2g and
// 2g + 1 side by side (the folded view of tcg.cu) -- which is the accumulator layout of
// mma.m8n8k4: EH - d S on the fp64 tensor cores, tr += d (EH - d S) element by element, and
// M1 += X_U^T X_EH, M2 += X_U^T X_D over the block's rows (U, d rows from shared memory, EH
// transposed by shuffles).  The CTA writes [M1 | M2 | tr | 0] entry-major (partials[e * grid + cta]),
// what tcg_reduce_kernel<8, 0> reads after pass A.
template <int K, class POW, bool HAS_ETA, bool OBJ, int NB, bool ADAPT, bool DOTS, bool OVF, bool HVO = false,
          bool GRAM = false>
__global__ void __launch_bounds__(kHaloThreads, PLP_HALO_CTAS) edge_halo_kernel(POW pw, EdgeArgs a) {
  constexpr bool WL = !HVO;
  static_assert(!(OBJ && HAS_ETA), "objective mode has no eta");
  static_assert(!GRAM || (HVO && !OVF && !DOTS && (K == 4 || K == 8)), "pass-A fold: Hv-only pass, k = 4 / 8");
  constexpr int CPL = halo_cpl<K, HVO>(), LPR = K / CPL, RPW = 32 / LPR;  // rows per pass
  constexpr int EB = (CPL == 4 && K == 8) ? 1 : 2;  // edges per loop iteration (independent chains: EB x CPL)
  static_assert(!GRAM || CPL == 2, "pass-A fold: the 2-column accumulator layout");
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // [2] tile data landed
  uint64_t* lbar = full + NB;                   // [3] halo list landed
  uint64_t* empty = lbar + 3;                          // [NBUF] consumers done with the buffer
  if constexpr (POW::kNeedsTables) pw.init_smem(smem + kHaloHead);
  const int ext_cap = OVF ? a.halo_stage : a.halo_ext_cap;  // halo rows staged per tile
  const int LS = ext_cap + 4;                  // shared list slot: n_ext, eb, ee, pad, columns
  const int LSG = a.halo_ext_cap + 4;          // global list stride
  int* lists = reinterpret_cast<int*>(smem + halo_lists_off(POW::kNeedsTables));
  const HaloLayout Ly = halo_layout(K, ext_cap, a.halo_nnz_cap, OBJ, HAS_ETA);
  unsigned char* buf0 = smem + halo_bufs_off(ext_cap, POW::kNeedsTables);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grp = lane / LPR, li = lane % LPR, c0 = li * CPL;
  const int pw_id = warp - kHaloCWarps;  // producer index (>= 0): 0 stages the streamed parts and lists
  if (tid == 0) {
    // full: the producer's arrive.expect_tx (TMA bytes) + one cp.async arrival per producer lane
    for (int q = 0; q < NB; ++q) {
      mbar_init(&full[q], 1 + 32 * kHaloProd);
      mbar_init(&empty[q], kHaloCWarps);
    }
    for (int q = 0; q < 3; ++q) mbar_init(&lbar[q], 1);
    fence_mbar_init();
  }
  const int n_rows = (int)a.n_rows;
  // work items: the tiles, or (a.tile_list) the listed tiles [tile_begin, + tile_count) -- the
  // interior / boundary launches of the multi-rank overlap (edge.cu)
  const int64_t n_tiles = a.tile_list ? a.tile_count : (a.n_rows + kHaloT - 1) / kHaloT;
  auto tile_of = [&](int64_t li) -> int64_t { return a.tile_list ? (int64_t)a.tile_list[a.tile_begin + li] : li; };
  const double p = a.p, pp1 = p * (p - 1.0);
  double* coef = reinterpret_cast<double*>(smem + 256);  // PLP_HALO_COEF_SMEM: [cG | cAB | cHA | cHB][K]
  double cG[CPL], cAB[CPL], cHA[CPL], cHB[CPL];
  if constexpr (PLP_HALO_COEF_SMEM) {
    if (tid < K) {
      double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
      if (a.AB != nullptr) {
        const double A = a.AB[tid], B = a.AB[K + tid];
        g0 = p / B;
        g1 = A / B;
        g2 = pp1 / B;
        g3 = pp1 * A / (B * B);
      }
      coef[tid] = g0;
      coef[K + tid] = g1;
      coef[2 * K + tid] = g2;
      coef[3 * K + tid] = g3;
    }
  } else {
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
  }
  double accA[CPL], accB[CPL], accAl[CPL], accGa[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) accA[c] = accB[c] = accAl[c] = accGa[c] = 0.0;
  double gm1[2] = {0.0, 0.0}, gm2[2] = {0.0, 0.0}, gtr = 0.0;  // GRAM accumulators (consumers)
  __syncthreads();

  // (thread 0) stage the halo list of tile t into list slot q
  auto issue_list = [&](int64_t t, int q) {
    if (t >= n_tiles) return;
    mbar_expect_tx(&lbar[q], (unsigned)LS * 4u);
    tma_bulk_g2s(lists + q * LS, a.halo_ext + tile_of(t) * LSG, (unsigned)LS * 4u, &lbar[q]);
  };
  int trace_it = 0;  // the producer's iteration (pipeline trace build only)
  (void)trace_it;
  // (producer warp) stage tile t into buffer b; its halo list is in slot q (use parity lph)
  auto issue_tile = [&](int64_t t, int b, int q, unsigned lph) {
    if (t >= n_tiles) return;
    unsigned char* B = buf0 + (size_t)b * Ly.bytes;
    const int r0 = (int)(tile_of(t) * kHaloT), r1 = min(r0 + kHaloT, n_rows);
    constexpr unsigned RB = K * 8u;  // bytes per row
    mbar_wait(&lbar[q], lph);
    if (lane == 0 && pw_id == 0) PLP_TRACE(trace_it, 32);
    const int* Lq = lists + q * LS;
    const int nx = OVF ? min(Lq[0], ext_cap) : Lq[0];  // rows staged (OVF: the first ext_cap)
    PLP_DCHECK(nx >= 0 && nx <= ext_cap, "halo count within the tile's list slot");
    if (lane == 0 && pw_id == 0) {
      const int eb = Lq[1], ee = Lq[2];
      PLP_DCHECK(ee - eb >= 0 && ee - eb <= a.halo_nnz_cap, "tile nnz within the buffer");
      PLP_DCHECK(eb == (int)a.rp[r0] && ee == (int)a.rp[r1], "tile CSR bounds match row_ptr");
      const unsigned rp_b = (unsigned)(((r1 + 1 + 3) & ~3) - r0) * 4u;
      const unsigned sc_b = (unsigned)(((r1 + 3) & ~3) - r0) * 4u;
      const int cb = eb & ~3, ce = (ee + 3) & ~3, wb = eb & ~1, we = (ee + 1) & ~1;
      const unsigned enc_b = (unsigned)(ce - cb) * 4u, w_b = (unsigned)(we - wb) * 8u;
      const unsigned own_b = (unsigned)(r1 - r0) * RB;
      mbar_expect_tx(&full[b], rp_b + (OBJ ? 2u : 1u) * sc_b + enc_b + w_b + (HAS_ETA ? 2u : 1u) * own_b);
      tma_bulk_g2s(B + Ly.rp, a.rp + r0, rp_b, &full[b]);
      tma_bulk_g2s(B + Ly.sched, (OBJ ? a.sched_up : a.sched) + r0, sc_b, &full[b]);
      if constexpr (OBJ) tma_bulk_g2s(B + Ly.nl, a.nlow + r0, sc_b, &full[b]);
      if (enc_b) {
        tma_bulk_g2s(B + Ly.enc, a.halo_enc + cb, enc_b, &full[b]);
        tma_bulk_g2s(B + Ly.w, a.w + wb, w_b, &full[b]);
      }
      tma_bulk_g2s(B + Ly.U, a.U + (int64_t)r0 * K, own_b, &full[b]);
      if constexpr (HAS_ETA) tma_bulk_g2s(B + Ly.E, a.eta + (int64_t)r0 * K, own_b, &full[b]);
      PLP_TRACE(trace_it, 33);
    }
    // halo rows: PPR lanes per row, 32 / PPR rows per warp instruction
    constexpr int PPR = K / 2, RPI = 32 / PPR;
    const int rl = lane / PPR + pw_id * RPI, pc = lane % PPR;
#pragma unroll 4
    for (int x = rl; x < nx; x += RPI * kHaloProd) {
      const int j = Lq[4 + x];
      PLP_DCHECK(j >= 0 && (int64_t)j < a.n_cols && (j < r0 || j >= r1), "halo column outside the tile, inside U");
      const unsigned off = ((unsigned)(kHaloT + x) * K + 2 * pc) * 8u;
      cp_async16(B + Ly.U + off, a.U + (int64_t)j * K + 2 * pc);
      if constexpr (HAS_ETA) cp_async16(B + Ly.E + off, a.eta + (int64_t)j * K + 2 * pc);
    }
    if (lane == 0 && pw_id == 0) PLP_TRACE(trace_it, 34);
    cp_async_mbar_arrive(&full[b]);
  };

  const int64_t t0 = blockIdx.x, ts = gridDim.x;
  if (warp >= kHaloCWarps) {
    // ---- producer warp: stages tile it into buffer it & 1 once the consumers released it, and
    // the halo list of tile it + 2 into list slot (it + 2) % 3 (freed by tile it - 1) ----
    if (lane == 0 && pw_id == 0) {
      issue_list(t0, 0);
      issue_list(t0 + ts, 1);
    }
    __syncwarp();
    for (int it = 0;; ++it) {
      const int64_t t = t0 + (int64_t)it * ts;
      if (t >= n_tiles) break;
      const int b = it % NB;
      if (it >= NB)
        mbar_wait_sleep(&empty[b], (unsigned)((it - NB) / NB) & 1u, PLP_HALO_SLEEP_NS);
      if (lane == 0 && pw_id == 0) PLP_TRACE(it, 0);
      if (lane == 0) fence_proxy_async();  // consumers' generic reads before the async refill
      __syncwarp();
      trace_it = it;
      issue_tile(t, b, it % 3, (unsigned)(it / 3) & 1u);
      if (lane == 0 && pw_id == 0) PLP_TRACE(it, 1);
      if (lane == 0 && pw_id == 0) issue_list(t + 2 * ts, (it + 2) % 3);
      // warm L2 with the next tile's streamed parts (own rows, enc, w), so that its TMA copies,
      // issued only once the consumers release a buffer, are L2 hits (per-row bulk prefetches of
      // the halo rows too measured 1.6x slower: tiny bulk operations)
      if (lane == 0 && pw_id == 0) {
        const int64_t tn = t + ts;
        if (tn < n_tiles) {
          const int qn = (it + 1) % 3;
          mbar_wait(&lbar[qn], (unsigned)((it + 1) / 3) & 1u);
          const int* Ln = lists + qn * LS;
          const int r0 = (int)(tile_of(tn) * kHaloT), r1 = min(r0 + kHaloT, n_rows);
          const size_t rows_b = (size_t)(r1 - r0) * K * 8u;
          l2_prefetch_range(a.U + (int64_t)r0 * K, rows_b);
          if constexpr (HAS_ETA) l2_prefetch_range(a.eta + (int64_t)r0 * K, rows_b);
          l2_prefetch_range(a.halo_enc + Ln[1], (size_t)(Ln[2] - Ln[1]) * 4u);
          l2_prefetch_range(a.w + Ln[1], (size_t)(Ln[2] - Ln[1]) * 8u);
        }
      }
      __syncwarp();
    }
  } else {
  // The tile's rows are split into NSL slices of RPW schedule-consecutive rows (rows of similar
  // degree: the schedule sorts by degree); slices go to the consumer warps in snake order (warp w
  // takes slices w, 2C - 1 - w, 2C + w, ...), so every warp gets a heavy and a light slice.
  constexpr int NSL = kHaloT / RPW, C = kHaloCWarps;
  bool capmode = false;  // this warp's previous row needed the capped form
  // GRAM: B fragments of -S (rows 4s + q, column g), the warp's M1 / M2 accumulators and its share
  // of sum d (EH - d S)
  const int g8 = lane >> 2, q4 = lane & 3;
  double gS[2] = {0.0, 0.0};
  if constexpr (GRAM) {
    gS[0] = -a.gram_S[q4 * 8 + g8];
    gS[1] = -a.gram_S[(4 + q4) * 8 + g8];
  }
  (void)gS;
  (void)g8;
  (void)q4;
  for (int it = 0;; ++it) {
    const int64_t t = t0 + (int64_t)it * ts;
    if (t >= n_tiles) break;
    const int b = it % NB;
    mbar_wait(&full[b], (unsigned)(it / NB) & 1u);  // tile t resident
    if (lane == 0) PLP_TRACE(it, 2 + warp);

    const unsigned char* B = buf0 + (size_t)b * Ly.bytes;
    const int* rp_s = reinterpret_cast<const int*>(B + Ly.rp);
    const int* sc_s = reinterpret_cast<const int*>(B + Ly.sched);
    const int64_t tt = tile_of(t);
    const int r0 = (int)(tt * kHaloT);
    const int nr = min(kHaloT, n_rows - r0);
    const int eb = rp_s[0];
    const int* enc_s = reinterpret_cast<const int*>(B + Ly.enc) - (eb & ~3);
    const double* w_s = reinterpret_cast<const double*>(B + Ly.w) - (eb & ~1);
    const double* tU = reinterpret_cast<const double*>(B) + c0;  // Ly.U == 0
    const double* tE = tU + (kHaloT + halo_rows_cap(K)) * K;   // Ly.E: a compile-time offset
    // neighbour rows: tile-local index x; OVF: x >= kHaloT + ext_cap is an unstaged halo row, read
    // through its global id in the tile's (global) halo list
    const int* glist = a.halo_ext + tt * LSG + 4 - kHaloT;
    // staged rows by 32-bit shared-window address: one IMAD per neighbour row serves U and eta
    // (eta at a compile-time offset)
    const unsigned sU = smem_u32(tU);
    constexpr unsigned kEOff = (unsigned)(kHaloT + halo_rows_cap(K)) * K * 8u;
    auto ldU = [&](int x, double (&v)[CPL]) {
      if constexpr (OVF) {
        if (x >= kHaloT + ext_cap) {
          lds_vec<CPL>(a.U + (int64_t)__ldg(glist + x) * K + c0, v);
          return;
        }
      }
      lds_row<CPL, 0>(sU + (unsigned)x * (K * 8u), v);
    };
    auto ldE = [&](int x, double (&v)[CPL]) {
      if constexpr (OVF) {
        if (x >= kHaloT + ext_cap) {
          lds_vec<CPL>(a.eta + (int64_t)__ldg(glist + x) * K + c0, v);
          return;
        }
      }
      lds_row<CPL, kEOff>(sU + (unsigned)x * (K * 8u), v);
    };

#pragma unroll 1
    for (int rd = 0; rd * C < NSL; ++rd) {
      // snake order alternating with the tile parity: over any two consecutive tiles (one is
      // resident while the other is computed) every warp takes a heavy and a light slice
      const int sl = rd * C + (((rd + it) & 1) ? C - 1 - warp : warp);
      if (sl >= NSL) continue;
      const int lr = sl * RPW + grp;  // position in the tile's schedule
      double gH[CPL];                 // GRAM: the group's EH values
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) gH[cc] = 0.0;
      // GRAM, before the rows (their latency hides behind the edge loop): the block's U and d
      // operands from the tile buffer, M2 += X_U^T X_D and P = X_D S on the tensor cores; the
      // EH-dependent part (M1, d (EH - P)) follows the rows.  X[r][c] lives in group (k = 8) r,
      // (k = 4) 2r + c / 4, column c % k, i.e. at lane group * LPR.
      const int glrow = GRAM ? (lr < nr ? sc_s[lr] - r0 : -1) : -1;  // the group's tile row
      double gAU[2] = {0.0, 0.0}, gP0 = 0.0, gP1 = 0.0;
      if constexpr (GRAM) {
        const double* tUr = tU - c0;
        const double* tEr = tE - c0;
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          const int grpA = K == 8 ? g8 : 2 * g8 + s, colA = K == 8 ? 4 * s + q4 : q4;
          const int lrA = __shfl_sync(0xffffffffu, glrow, grpA * LPR);
          const int r = 4 * s + q4;
          const int grpB = K == 8 ? r : 2 * r + (g8 >> 2), colB = K == 8 ? g8 : (g8 & 3);
          const int lrB = __shfl_sync(0xffffffffu, glrow, grpB * LPR);
          const double dA = lrA >= 0 ? tEr[lrA * K + colA] : 0.0;   // X_D[g][4s + q]
          gAU[s] = lrB >= 0 ? tUr[lrB * K + colB] : 0.0;          // X_U[4s + q][g]
          const double bd = lrB >= 0 ? tEr[lrB * K + colB] : 0.0;  // X_D[4s + q][g]
          dmma884(gP0, gP1, dA, gS[s]);
          dmma884(gm2[0], gm2[1], gAU[s], bd);
        }
      }
      (void)gAU;
      do {  // the row (a `continue` below ends it; GRAM then joins the warp's block update)
      if (lr >= nr) break;
      const int row = sc_s[lr];
      const int lrow = row - r0;
      const int e0 = rp_s[lrow], e1 = rp_s[lrow + 1];
      double ui[CPL], ei[CPL];
      lds_vec<CPL>(tU + lrow * K, ui);
      if constexpr (HAS_ETA) lds_vec<CPL>(tE + lrow * K, ei);
      if constexpr (OBJ) {
        // ---- objective mode: the row's upper-triangle edges [e0 + nlow, e1) only ----
        const int* nl_s = reinterpret_cast<const int*>(B + Ly.nl);
        const int eu = e0 + nl_s[lrow];
        double Ar[CPL];
        unsigned mx = 0;
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) Ar[cc] = 0.0;
        auto obj_edge = [&](double wv, const double (&uj)[CPL]) {
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) {
            const double d = ui[cc] - uj[cc];
            if constexpr (POW::kIsP2) {
              Ar[cc] = fma(wv * d, d, Ar[cc]);
            } else {
              mx = max(mx, (unsigned)__double2hiint(d) * 2u - pw.fast_lo2);
              const double ws = wv * pw.pow_fast(d);  // w |d|^{p-2}
              Ar[cc] = fma(ws, d * d, Ar[cc]);        // w |d|^p
            }
          }
        };
        int e = eu;
        if constexpr (EB == 2) {
#pragma unroll 1
          for (; e + 1 < e1; e += 2) {
            const int x0 = enc_s[e], x1 = enc_s[e + 1];
            const double w0 = w_s[e], w1 = w_s[e + 1];
            double uj0[CPL], uj1[CPL];
            ldU(x0, uj0);
            ldU(x1, uj1);
            obj_edge(w0, uj0);
            obj_edge(w1, uj1);
          }
        }
#pragma unroll 1
        for (; e < e1; ++e) {  // EB = 1: every edge; EB = 2: the odd last one
          double uj0[CPL];
          ldU(enc_s[e], uj0);
          obj_edge(w_s[e], uj0);
        }
        double tn[CPL];
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          const double au = fabs(ui[cc]);
          if constexpr (POW::kIsP2) {
            tn[cc] = au;
          } else {
            mx = max(mx, (unsigned)__double2hiint(au) * 2u - pw.fast_lo2);
            tn[cc] = pw.pow_fast(au) * au;
          }
        }
        if constexpr (!POW::kIsP2) {
          if (mx >= pw.fast_span2) {  // some |d| outside the fast domain (usually |d| < eps)
            unsigned bad = 0;
#pragma unroll
            for (int cc = 0; cc < CPL; ++cc) {
              Ar[cc] = 0.0;
              double sn;
              pw.eval(fabs(ui[cc]), sn, tn[cc]);
            }
            if constexpr (ADAPT) {
              // A needs the uncapped |d|^p: the clamped fast power from shared memory covers d = 0
              // and every |d| >= 2^-120; libdevice below only for what it flags
#pragma unroll 1
              for (int ee = eu; ee < e1; ++ee) {
                double uj0[CPL];
                ldU(enc_s[ee], uj0);
                const double wv = w_s[ee];
#pragma unroll
                for (int cc = 0; cc < CPL; ++cc) {
                  const double d = ui[cc] - uj0[cc];
                  bad |= out_of_domain(abs_hi(d));
                  Ar[cc] = fma(wv * pw.pow_fast(fmax(fabs(d), 0x1p-120)), d * d, Ar[cc]);
                }
              }
            } else {
              bad = 1;
            }
            if (bad) {
#pragma unroll
              for (int cc = 0; cc < CPL; ++cc) Ar[cc] = 0.0;
            }
            for (int ee = eu; ee < e1 && bad; ++ee) {
              const int64_t j = a.col[ee];
              const double wv = a.w[ee];
#pragma unroll
              for (int cc = 0; cc < CPL; ++cc) {
                const double ad = fabs(ui[cc] - a.U[j * K + c0 + cc]);
                Ar[cc] += wv * ((ad != 0.0) ? pow(ad, a.p) : 0.0);
              }
            }
          }
        }
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          accA[cc] += Ar[cc];
          accB[cc] = fma(tn[cc], fabs(ui[cc]), accB[cc]);
        }
        continue;
      }
      double L[CPL], HA[CPL];
      unsigned mx = 0;
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) L[cc] = HA[cc] = 0.0;

      // edge pairs as straight-line code (their dependency chains interleave), then the
      // remaining edge; summation order stays the CSR order
      int e = (ADAPT && capmode) ? e1 : e0;  // capmode: the capped form below recomputes the row
      const int* ep = enc_s + e;  // running pointers: immediate-offset loads, no per-pair index math
      const double* wp = w_s + e;
      const int* const ep_last = enc_s + (e1 - 1);
      if constexpr (EB == 1) {
#pragma unroll 1
        for (; ep <= ep_last; ++ep, ++wp) {
          const int x0 = *ep;
          const double w0 = *wp;
          double uj0[CPL], ej0[CPL];
          ldU(x0, uj0);
          if constexpr (HAS_ETA) ldE(x0, ej0);
          edge_update_mx<CPL, POW, HAS_ETA, WL>(pw, w0, ui, uj0, ei, ej0, L, HA, mx);
        }
      }
#pragma unroll 1
      for (; EB == 2 && ep < ep_last; ep += 2, wp += 2) {
        const int x0 = ep[0], x1 = ep[1];
        PLP_DCHECK(x0 >= 0 && x1 >= 0 && x0 < kHaloT + a.halo_ext_cap && x1 < kHaloT + a.halo_ext_cap && (x0 < nr || x0 >= kHaloT) &&
                       (x1 < nr || x1 >= kHaloT), "edge's tile-local neighbour index");
        const double w0 = wp[0], w1 = wp[1];
        double uj0[CPL], ej0[CPL], uj1[CPL], ej1[CPL];
        ldU(x0, uj0);
        ldU(x1, uj1);
        if constexpr (HAS_ETA) {
          ldE(x0, ej0);
          ldE(x1, ej1);
        }
        edge_update_mx<CPL, POW, HAS_ETA, WL>(pw, w0, ui, uj0, ei, ej0, L, HA, mx);
        edge_update_mx<CPL, POW, HAS_ETA, WL>(pw, w1, ui, uj1, ei, ej1, L, HA, mx);
      }
      if (EB == 2 && ep == ep_last) {  // the odd last edge
        const int x0 = *ep;
        const double w0 = *wp;
        double uj0[CPL], ej0[CPL];
        ldU(x0, uj0);
        if constexpr (HAS_ETA) ldE(x0, ej0);
        edge_update_mx<CPL, POW, HAS_ETA, WL>(pw, w0, ui, uj0, ei, ej0, L, HA, mx);
      }
      // node terms sn = cap(|u|)^{p-2}, tn = |u|^{p-1}, after the edges (fewer live registers in
      // the edge loop); same fast-domain test, exact recomputation of the row when it fails
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
      if constexpr (!POW::kIsP2 && !ADAPT) {
        if (mx >= pw.fast_span2) {  // rare: exact libdevice recomputation of the row
          edge_row_exact<CPL, POW, HAS_ETA>(pw, e0, e1, a.col, a.w, a.U, a.eta, K, c0, ui, ei, L, HA);
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) pw.eval(fabs(ui[cc]), sn[cc], tn[cc]);
        }
      }
      if constexpr (!POW::kIsP2 && ADAPT) {
        // capmode skipped the fast loop (mx then holds the node tests only)
        const bool need = capmode || mx >= pw.fast_span2;
        bool fast_fails = mx >= pw.fast_span2;
        if (need) {
          // some |d| left the fast domain (usually |d| < eps: the degenerate regime): the row
          // again from shared memory in the capped form; libdevice only for what that cannot take
          CapRange rg;
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) L[cc] = HA[cc] = 0.0;
          int ee = e0;
#pragma unroll 1
          for (; EB == 2 && ee + 1 < e1; ee += 2) {  // edge pairs: two dependency chains interleave
            const int x0 = enc_s[ee], x1 = enc_s[ee + 1];
            double uj0[CPL], ej0[CPL], uj1[CPL], ej1[CPL];
            ldU(x0, uj0);
            ldU(x1, uj1);
            if constexpr (HAS_ETA) {
              ldE(x0, ej0);
              ldE(x1, ej1);
            }
            edge_update_capsel<CPL, POW, HAS_ETA, WL>(pw, w_s[ee], ui, uj0, ei, ej0, L, HA, rg);
            edge_update_capsel<CPL, POW, HAS_ETA, WL>(pw, w_s[ee + 1], ui, uj1, ei, ej1, L, HA, rg);
          }
#pragma unroll 1
          for (; ee < e1; ++ee) {  // EB = 1: every edge; EB = 2: the odd last one
            const int x0 = enc_s[ee];
            double uj0[CPL], ej0[CPL];
            ldU(x0, uj0);
            if constexpr (HAS_ETA) ldE(x0, ej0);
            edge_update_capsel<CPL, POW, HAS_ETA, WL>(pw, w_s[ee], ui, uj0, ei, ej0, L, HA, rg);
          }
          if (rg.bad()) edge_row_exact<CPL, POW, HAS_ETA>(pw, e0, e1, a.col, a.w, a.U, a.eta, K, c0, ui, ei, L, HA);
#pragma unroll
          for (int cc = 0; cc < CPL; ++cc) pw.eval(fabs(ui[cc]), sn[cc], tn[cc]);
          fast_fails = fast_fails || rg.fast_fails(pw);
        }
        // the warp's next pass goes straight to the capped form iff the fast form failed here
        capmode = __any_sync(__activemask(), fast_fails);
      }
      double g[CPL], hv[CPL];
      if constexpr (PLP_HALO_COEF_SMEM) {
        lds_vec<CPL>(coef + c0, cG);
        lds_vec<CPL>(coef + K + c0, cAB);
        lds_vec<CPL>(coef + 2 * K + c0, cHA);
        lds_vec<CPL>(coef + 3 * K + c0, cHB);
      }
#pragma unroll
      for (int cc = 0; cc < CPL; ++cc) {
        if constexpr (!HVO) {
          accA[cc] = fma(ui[cc], L[cc], accA[cc]);
          accB[cc] = fma(tn[cc], fabs(ui[cc]), accB[cc]);
        }
        const double phi = copysign(tn[cc], ui[cc]);
        g[cc] = HVO ? 0.0 : cG[cc] * (L[cc] - cAB[cc] * phi);
        if constexpr (HAS_ETA) {
          hv[cc] = cHA[cc] * HA[cc] - cHB[cc] * sn[cc] * ei[cc];
          if constexpr (DOTS) {
            accAl[cc] = fma(p * phi, ei[cc], accAl[cc]);
            accGa[cc] = fma(g[cc], ei[cc], accGa[cc]);
          }
        } else {
          hv[cc] = 0.0;
        }
      }
      if (!HVO && a.G != nullptr) st_vec<CPL>(a.G + (int64_t)row * K + c0, g);
      if constexpr (HAS_ETA) {
        if (a.Hv != nullptr) st_vec<CPL>(a.Hv + (int64_t)row * K + c0, hv);
      }
      if constexpr (GRAM) {
#pragma unroll
        for (int cc = 0; cc < CPL; ++cc) {
          gH[cc] = hv[cc];
          gtr = fma(ei[cc], hv[cc] + (cc == 0 ? gP0 : gP1), gtr);  // d (EH - d S): gP = X_D (-S)
        }
      }
      } while (0);
      if constexpr (GRAM) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {  // M1 += X_U^T X_EH over rows 4s .. 4s + 3 of the block
          const int src = 4 * (4 * s + q4) + (g8 >> 1);  // C-layout lane of X[4s + q][g]
          const double h0 = __shfl_sync(0xffffffffu, gH[0], src), h1 = __shfl_sync(0xffffffffu, gH[1], src);
          dmma884(gm1[0], gm1[1], gAU[s], (g8 & 1) ? h1 : h0);
        }
      }
    }
    __syncwarp();
    if (lane == 0) PLP_TRACE(it, 16 + warp);
    if (lane == 0) mbar_arrive(&empty[b]);  // this warp is done with buffer b
  }
  }

  // ---- fixed-order CTA reduction (reuses buffer 0: every issued copy has been consumed) ----
  __syncthreads();
  double* red = reinterpret_cast<double*>(buf0);  // [4][CPL][threads]
  if constexpr (GRAM) {
    // [M1 | M2 | tr | 0]: fragment element (g, 2q + h) of consumer warp w at red[j][w * 32 + 4g + q]
    // (j = h for M1, 2 + h for M2, 4 for tr), summed over the warps in order
    red[0 * kHaloThreads + tid] = gm1[0];
    red[1 * kHaloThreads + tid] = gm1[1];
    red[2 * kHaloThreads + tid] = gm2[0];
    red[3 * kHaloThreads + tid] = gm2[1];
    red[4 * kHaloThreads + tid] = gtr;
    __syncthreads();
    constexpr int E = 2 * 64 + 2;
    for (int e = tid; e < E; e += kHaloThreads) {
      double sum = 0.0;
      if (e < 128) {
        const int m = e & 63, gg = m >> 3, cc = m & 7;
        const int j = (e >> 6) * 2 + (cc & 1), ln = 4 * gg + (cc >> 1);
        for (int w = 0; w < kHaloCWarps; ++w) sum += red[j * kHaloThreads + w * 32 + ln];
      } else if (e == 128) {
        for (int th = 0; th < kHaloCWarps * 32; ++th) sum += red[4 * kHaloThreads + th];
      }
      a.partials[(int64_t)e * gridDim.x + blockIdx.x] = sum;
    }
    return;
  }
#pragma unroll
  for (int cc = 0; cc < CPL; ++cc) {
    red[(0 * CPL + cc) * kHaloThreads + tid] = accA[cc];
    red[(1 * CPL + cc) * kHaloThreads + tid] = accB[cc];
    red[(2 * CPL + cc) * kHaloThreads + tid] = accAl[cc];
    red[(3 * CPL + cc) * kHaloThreads + tid] = accGa[cc];
  }
  __syncthreads();
  for (int tt = tid; tt < 4 * K; tt += kHaloThreads) {
    const int q = tt / K, cl = tt % K;
    const int l = cl / CPL, cc = cl % CPL;
    const double* base = red + (q * CPL + cc) * kHaloThreads;
    double sum = 0.0;
    for (int th = l; th < kHaloThreads; th += LPR) sum += base[th];
    a.partials[((int64_t)blockIdx.x * 4 + q) * K + cl] = sum;
  }
}

// Halo rows staged per tile: the whole halo (ext_cap) if the buffers fit, else the largest multiple
// of 4 that fits (overflow mode); 0 if not even 64 rows fit.
inline int halo_stage_rows(int k, int ext_cap, int nnz_cap, bool tables, bool obj, bool eta, int nb) {
  ext_cap = ext_cap < halo_rows_cap(k) ? ext_cap : halo_rows_cap(k);
  if (halo_smem_bytes(k, ext_cap, nnz_cap, tables, obj, eta, nb) <= kHaloSmemMax) return ext_cap;
  int lo = 0, hi = ext_cap;
  while (hi - lo > 4) {
    const int mid = ((lo + hi) / 2) & ~3;
    if (halo_smem_bytes(k, mid, nnz_cap, tables, obj, eta, nb) <= kHaloSmemMax) lo = mid; else hi = mid;
  }
  return lo >= 64 ? lo : 0;
}

template <int K, class POW, bool HAS_ETA, bool OBJ>
plp_status launch_halo_shape(plp_ctx* ctx, const EdgeArgs& a0, const POW& pw, int* grid_out) {
  EdgeArgs a = a0;
  const bool T = POW::kNeedsTables;
  // passes without eta stage U rows only: a third buffer fits where the eta pass has two
  constexpr int NB3 = HAS_ETA ? kHaloNBuf : PLP_HALO_NBUF_NOETA;
  const bool deep = NB3 != kHaloNBuf && a.halo_ext_cap <= halo_rows_cap(K) &&
                    halo_smem_bytes(K, a.halo_ext_cap, a.halo_nnz_cap, T, OBJ, HAS_ETA, NB3) <= kHaloSmemMax;
  const int nb = deep ? NB3 : kHaloNBuf;
  a.halo_stage = halo_stage_rows(K, a.halo_ext_cap, a.halo_nnz_cap, T, OBJ, HAS_ETA, nb);
  const bool ovf = a.halo_stage < a.halo_ext_cap;
  // the fused F/G/Hv pass (G and eta) keeps the plain loop; every other pass adapts
  const bool adapt = !(HAS_ETA && a.G != nullptr);
  const bool dots = HAS_ETA && a.want_dots;
  const bool hvo = HAS_ETA && !OBJ && adapt && !dots && a.G == nullptr && !a.need_ab;
  // the fused tCG's pass A in the Hessian-vector-only pass (k = 4, 8; single launch, no tile list)
  constexpr bool kGramShape = HAS_ETA && !OBJ && (K == 4 || K == 8);
  const bool gram = kGramShape && hvo && !ovf && a.gram_S != nullptr && a.tile_list == nullptr;
  if (a.gram_used) *a.gram_used = gram ? 1 : 0;
  auto kern = deep ? edge_halo_kernel<K, POW, HAS_ETA, OBJ, NB3, true, false, false>
            : gram ? edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, true, false, false, kGramShape, kGramShape>
            : (hvo && !ovf) ? edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, true, false, false, HAS_ETA && !OBJ>
            : ovf  ? (adapt ? edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, true, false, true>
                            : edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, false, false, true>)
                   : (adapt ? (dots ? edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, true, HAS_ETA, false>
                                    : edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, true, false, false>)
                            : (dots ? edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, false, HAS_ETA, false>
                                    : edge_halo_kernel<K, POW, HAS_ETA, OBJ, kHaloNBuf, false, false, false>));
  const unsigned smem = halo_smem_bytes(K, ovf ? a.halo_stage : a.halo_ext_cap, a.halo_nnz_cap, T, OBJ, HAS_ETA, nb);
  // the dynamic shared-memory opt-in is a per-device function attribute: set it on this ctx's
  // device whenever a launch needs more than the value set so far (per template instance)
  static unsigned attr_set[64][9] = {};
  const int vi = deep ? 4 : gram ? 8 : (hvo && !ovf) ? 7 : ovf ? 5 + (adapt ? 1 : 0) : (adapt ? 1 : 0) + (dots ? 2 : 0);
  unsigned& set_to = attr_set[ctx->device & 63][vi];
  if (set_to < smem) {
    PLP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set_to = smem;
  }
  const int64_t n_tiles = a.tile_list ? a.tile_count : (a.n_rows + kHaloT - 1) / kHaloT;
  int64_t grid = (int64_t)ctx->num_sms * PLP_HALO_CTAS;
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  if (grid > n_tiles) grid = n_tiles > 0 ? n_tiles : 1;
  kern<<<(int)grid, kHaloThreads, smem, ctx->stream>>>(pw, a);
  PLP_LAUNCH_CHECK("edge_halo_kernel");
  // [adapt]: the capped-form row recompute (every pass but the fused F/G/Hv benchmark pass);
  // [ovf]: halo rows beyond what fits in shared memory read from L2
  char name[96];
  snprintf(name, sizeof(name), "edge_halo_kernel%s", OBJ ? (deep ? "[objective,3buf,adapt]" : ovf ? "[objective,ovf,adapt]" : "[objective,adapt]")
                                                         : deep ? "[3buf,adapt]" : ovf ? (adapt ? "[ovf,adapt]" : "[ovf]")
                                                         : gram ? "[adapt,hv,gram]"
                                                         : (hvo && !ovf) ? "[adapt,hv]"
                                                         : adapt ? "[adapt]" : "");
  constexpr int kCplN = halo_cpl<K>();  // the name reports the non-Hessian-vector shape
  note_edge_kernel(name, K, (hvo && !ovf) ? halo_cpl<K, true>() : kCplN, K / ((hvo && !ovf) ? halo_cpl<K, true>() : kCplN),
                   (hvo && !ovf) || kCplN == 2 ? 2 : 1, POW::kName, HAS_ETA);
  *grid_out = (int)grid;
  return PLP_OK;
}

// The halo kernel applies when the graph has halo tiles, k is 4, 8 or 16, the dense arrays are
// 16-byte aligned, U / eta are contiguous (ldx == k) and the buffers fit in shared memory.
template <class POW>
plp_status try_launch_halo(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid, bool* used) {
  *used = false;
  const int k = a.k;
  auto al16 = [](const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; };
  if (a.halo_enc == nullptr || (k != 4 && k != 8 && k != 16) || (a.ldx != 0 && a.ldx != k) ||
      !al16(a.U) || (a.eta && !al16(a.eta)) || (a.G && !al16(a.G)) || (a.Hv && !al16(a.Hv)))
    return PLP_OK;
  const bool he = a.eta != nullptr;
  if (halo_stage_rows(k, a.halo_ext_cap, a.halo_nnz_cap, POW::kNeedsTables, false, true, kHaloNBuf) == 0)
    return PLP_OK;  // not even 64 halo rows per tile fit: the staged kernel
  if (he && a.want_dots &&
      halo_stage_rows(k, a.halo_ext_cap, a.halo_nnz_cap, POW::kNeedsTables, false, true, kHaloNBuf) <
          a.halo_ext_cap)
    return PLP_OK;  // full-mode dots with an overflowing halo: the staged kernel
  *used = true;
  const bool obj = !he && a.G == nullptr && a.upper_ok && a.nlow != nullptr && a.sched_up != nullptr;
#define PLP_HSHAPE(K)                                                                      \
  return he ? launch_halo_shape<K, POW, true, false>(ctx, a, pw, grid)                     \
            : (obj ? launch_halo_shape<K, POW, false, true>(ctx, a, pw, grid)               \
                   : launch_halo_shape<K, POW, false, false>(ctx, a, pw, grid))
#ifdef PLP_TUNE_ONLY
  PLP_HSHAPE(8);
#else
  if (k == 4) PLP_HSHAPE(4);
  if (k == 8) PLP_HSHAPE(8);
  PLP_HSHAPE(16);
#endif
#undef PLP_HSHAPE
}

}  // namespace plp
