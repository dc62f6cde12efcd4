// Tiled fused F / EucGrad / EucHessianEta edge kernel.
//
// The graph is cut into tiles of <= PLP_TILE_ROWS consecutive rows (compact graph regions after
// plp_tile_order; host-side caps keep a tile within the shared-memory budget).  A persistent CTA
// loops over tiles:
//   stage    one thread issues TMA bulk copies (cp.async.bulk, mbarrier completion) of the tile's
//            contiguous U rows, eta rows, row_ptr, encoded columns, weights and external-column
//            list into shared memory, and warms L2 with the CTA's next tile;
//   gather   all threads start cp.async copies of the external rows U_j, eta_j into the value
//            slots of the external edges (they land while phases 0 and 1a run);
//   phase 0  every edge that owns a value slot adds itself to the tile's work list: each INTERNAL
//            undirected edge (both ends in the tile) once, at its upper row, and each EXTERNAL edge;
//   phase 1  flat, balanced sweeps over the work list compute the one power per edge-column and
//            the slot value, from the upper row i's side (d = u_i - u_j):
//              (cL, cH) = (w |d|^{p-2} d,  w cap(|d|)^{p-2} (eta_i - eta_j))
//                       = (w phi_p(d),     the w~_ij (eta_i - eta_j) term of Alg. 1);
//   phase 2  each row walks its CSR row in order (the oracle's order) and sums
//              L_i += s cL,  HA_i += s cH,  s = -1 at the lower row of an internal edge (both
//              terms are antisymmetric in (i, j)), +1 otherwise;
//            then the row epilogue (node terms, G, Hv, partial sums of A, B, alpha, gamma).
// Each internal undirected edge costs one power instead of two and its U_j / eta_j come from
// shared memory, which takes most of the gather traffic off L2.  Every reduction is in a fixed
// order: results are deterministic.
#pragma once
#include <cstdlib>

#include "async_copy.cuh"
#include "edge_kernel.cuh"
#include "edge_staged.cuh"
#include "edge_halo.cuh"

namespace plp {

constexpr int kTileRows = PLP_TILE_ROWS;

struct TiledLayout {
  unsigned coef, ut, et, w, enc, rp, xc, list, val, tab, total;
};
__host__ __device__ inline unsigned align16u(unsigned x) { return (x + 15u) & ~15u; }
// Shared-memory layout (byte offsets), identical on host and device.
__host__ __device__ inline TiledLayout tiled_layout(int k, int max_nnz, int max_slots, int max_ext,
                                                     int cpl, bool eta, bool tables) {
  TiledLayout L;
  unsigned o = 16;  // mbarrier
  L.coef = o; o += align16u(4 * k * 8);
  // rows of U and eta are padded to k + 2 doubles and value slots to k + 1 double2: consecutive
  // rows / slots then start on different banks (no shared-memory bank conflicts between groups)
  L.ut = o; o += align16u(kTileRows * (k + 2) * 8);
  L.et = o; o += eta ? align16u(kTileRows * (k + 2) * 8) : 0u;
  L.w = o; o += align16u((max_nnz + 4) * 8);
  L.enc = o; o += align16u((max_nnz + 8) * 4);
  L.rp = o; o += align16u((kTileRows + 1 + 8) * 4);
  L.xc = o; o += align16u((max_ext + 8) * 4);
  L.list = o; o += align16u(max_slots * 4 + 4);
  L.val = o;
  const unsigned vb = (unsigned)max_slots * (k + 1) * 16;
  const unsigned red = 4u * cpl * kEdgeThreads * 8;  // final CTA reduction reuses the value area
  o += align16u(vb > red ? vb : red);
  L.tab = o;
  if (tables) o += align16u(sizeof(PowTables));
  L.total = o;
  return L;
}


// Exact slot value with libdevice powers (rare: |d| below the cap, a tie, or outside the fast
// power domain): (w phi_p(d), w cap(|d|)^{p-2} de).
static __device__ __noinline__ double2 slot_exact(double d, double wv, double q, double pm1,
                                                  double eps, double s_eps, double de) {
  const double ad = fabs(d);
  const double cl = (ad != 0.0) ? wv * copysign(pow(ad, pm1), d) : 0.0;
  const double wc = (ad < eps) ? wv * s_eps : wv * pow(ad, q);
  return make_double2(cl, wc * de);
}

// Slot values (cL, cH) of the lane's CPL columns for one edge (weight wv, d = ui - uj,
// de = ei - ej); branch-free except for the rare exact path.
template <int CPL, class POW, bool HAS_ETA>
__device__ __forceinline__ void slot_values(const POW& pw, double wv, const double (&ui)[CPL],
                                            const double (&uj)[CPL], const double (&ei)[CPL],
                                            const double (&ej)[CPL], double2 (&out)[CPL]) {
  bool rare = false;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const double d = ui[c] - uj[c];
    const double de = HAS_ETA ? ei[c] - ej[c] : 0.0;
    if constexpr (POW::kIsP2) {
      out[c] = make_double2(wv * d, wv * de);
    } else {
      rare |= !pw.fast_hi(d);
      const double ws = wv * pw.pow_fast(d);
      out[c] = make_double2(ws * d, ws * de);
    }
  }
  if (rare) {
#pragma unroll
    for (int c = 0; c < CPL; ++c)
      out[c] = slot_exact(ui[c] - uj[c], wv, pw.q, pw.pm1, pw.eps, pw.s_eps,
                          HAS_ETA ? ei[c] - ej[c] : 0.0);
  }
}

template <int CPL, int LPR, int KT, class POW, bool HAS_ETA>
__global__ void __launch_bounds__(kEdgeThreads, 2) edge_tiled_kernel(EdgeArgs a, POW pw) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int k = KT ? KT : a.k;
  const int us = k + 2;   // padded smem row stride of U and eta (doubles)
  const int vs1 = k + 1;  // padded value-slot stride (double2)
  const TiledLayout Ly =
      tiled_layout(k, a.max_nnz, a.max_slots, a.max_ext, CPL, HAS_ETA, POW::kNeedsTables);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
  double* coef = reinterpret_cast<double*>(sm + Ly.coef);  // [4][k]: p/B, A/B, p(p-1)/B, p(p-1)A/B^2
  double* Ut = reinterpret_cast<double*>(sm + Ly.ut);
  double* Et = reinterpret_cast<double*>(sm + Ly.et);
  double* Wt = reinterpret_cast<double*>(sm + Ly.w);
  int32_t* Ct = reinterpret_cast<int32_t*>(sm + Ly.enc);
  int32_t* Rt = reinterpret_cast<int32_t*>(sm + Ly.rp);
  int32_t* Xt = reinterpret_cast<int32_t*>(sm + Ly.xc);
  int32_t* list = reinterpret_cast<int32_t*>(sm + Ly.list);
  double2* val = reinterpret_cast<double2*>(sm + Ly.val);
  if constexpr (POW::kNeedsTables) pw.init_smem(sm + Ly.tab);
  const double p = a.p;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (a.AB != nullptr) {
    const double pp1 = p * (p - 1.0);
    for (int l = threadIdx.x; l < k; l += blockDim.x) {
      const double A = a.AB[l], B = a.AB[k + l];
      coef[l] = p / B;
      coef[k + l] = A / B;
      coef[2 * k + l] = pp1 / B;
      coef[3 * k + l] = pp1 * A / (B * B);
    }
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int li = lane % LPR;
  const int grp = threadIdx.x / LPR;  // group id within the CTA
  const int G = blockDim.x / LPR;     // groups per CTA
  const int c0 = li * CPL;
  const bool active = c0 < k;
  // active lanes of this lane's group (lanes li with li * CPL < k)
  const int nact = (k + CPL - 1) / CPL < LPR ? (k + CPL - 1) / CPL : LPR;
  const unsigned gmask = (nact >= 32 ? 0xFFFFFFFFu : ((1u << nact) - 1u)) << (lane - li);

  double accA[CPL], accB[CPL], accAl[CPL], accGa[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) accA[c] = accB[c] = accAl[c] = accGa[c] = 0.0;

  unsigned parity = 0;
  for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x, parity ^= 1u) {
    const int4 tm = __ldg(a.tile_meta + t);  // (e0, ext_off, n_int, n_ext)
    const int e0 = tm.x, e1 = __ldg(&a.tile_meta[t + 1].x);
    const int n_int = tm.z, n_ext = tm.w, n_slots = tm.z + tm.w;
    const int64_t r0 = __ldg(a.tile_row + t);
    const int nrows = __ldg(a.tile_row + t + 1) - (int)r0;
    // staging offsets: bulk copies need 16-byte aligned global sources
    const int w_off = e0 & 1, c_off = e0 & 3, r_off = (int)(r0 & 3), x_off = tm.y & 3;
    // ---- stage the tile: TMA bulk copies of the CSR pieces (one elected thread) ----
    if (threadIdx.x == 0) {
      fence_proxy_async();  // order earlier generic smem accesses before the async writes
      const unsigned bw = align16u((unsigned)(e1 - e0 + w_off) * 8);
      const unsigned bc = align16u((unsigned)(e1 - e0 + c_off) * 4);
      const unsigned br = align16u((unsigned)(nrows + 1 + r_off) * 4);
      const unsigned bx = align16u((unsigned)(n_ext + x_off) * 4);
      mbar_expect_tx(bar, bw + bc + br + bx);
      tma_bulk_g2s(Wt, a.w + (e0 - w_off), bw, bar);
      tma_bulk_g2s(Ct, a.enc + (e0 - c_off), bc, bar);
      tma_bulk_g2s(Rt, a.rp + (r0 - r_off), br, bar);
      tma_bulk_g2s(Xt, a.ext_col + (tm.y - x_off), bx, bar);
    }
    // warm L2 with the CTA's next tile (its bulk copies then hit L2)
    if (threadIdx.x == 32 && t + gridDim.x < a.n_tiles) {
      const int64_t tn = t + gridDim.x;
      const int ne0 = __ldg(&a.tile_meta[tn].x), ne1 = __ldg(&a.tile_meta[tn + 1].x);
      const int64_t nr0 = __ldg(a.tile_row + tn);
      const unsigned nb = (unsigned)((__ldg(a.tile_row + tn + 1) - (int)nr0) * k * 8);
      l2_prefetch(a.U + nr0 * k, nb);
      if constexpr (HAS_ETA) l2_prefetch(a.eta + nr0 * k, nb);
      l2_prefetch(a.w + (ne0 & ~1), align16u((unsigned)(ne1 - (ne0 & ~1)) * 8));
      l2_prefetch(a.enc + (ne0 & ~3), align16u((unsigned)(ne1 - (ne0 & ~3)) * 4));
    }
    // ---- stage U and eta rows into padded rows (cp.async, 16-byte chunks, all threads) ----
    const int half = k >> 1;  // 16-byte chunks per row
    {
      const int per = HAS_ETA ? k : half;
      for (int ch = threadIdx.x; ch < nrows * per; ch += blockDim.x) {
        const int r = ch / per, part = ch - r * per;
        if (part < half) cp_async16(Ut + r * us + 2 * part, a.U + (r0 + r) * k + 2 * part);
        else cp_async16(Et + r * us + 2 * (part - half), a.eta + (r0 + r) * k + 2 * (part - half));
      }
      cp_async_commit();
    }
    mbar_wait(bar, parity);
    const double* W = Wt + w_off;
    const int32_t* C = Ct + c_off;
    const int32_t* R = Rt + r_off;
    const int32_t* X = Xt + x_off;
    // ---- gather: external rows U_j, eta_j into the two halves of slot n_int + x's value area ----
    {
      const int per = HAS_ETA ? k : half;
      for (int ch = threadIdx.x; ch < n_ext * per; ch += blockDim.x) {
        const int x = ch / per, part = ch - x * per;
        const int64_t j = X[x];
        double* dst = reinterpret_cast<double*>(val + (n_int + x) * vs1);
        if (part < half) cp_async16(dst + 2 * part, a.U + j * k + 2 * part);
        else cp_async16(dst + k + 2 * (part - half), a.eta + j * k + 2 * (part - half));
      }
      cp_async_commit();
    }

    // ---- phase 0: work list (slot -> row << 16 | edge) ----
    for (int rl = grp; rl < nrows; rl += G) {
      const int b = R[rl] - e0, e = R[rl + 1] - e0;
      for (int q = b + li; q < e; q += LPR) {
        const int c = C[q];
        if (c >= 0) list[c & 0xFFFF] = (rl << 16) | q;  // slot owner: internal upper or external
      }
    }
    cp_async_wait_staged();  // U, eta rows of the tile (the external gathers may still fly)
    __syncthreads();

    // ---- phase 1a: internal undirected edges (U, eta of both ends in shared memory) ----
    if (active) {
      for (int s = grp; s < n_int; s += G) {
        const int ent = list[s];
        const int rl = ent >> 16, q = ent & 0xFFFF;
        const int jl = (C[q] >> 16) & 0x7FFF;
        double ui[CPL], uj[CPL], ei[CPL] = {}, ej[CPL] = {};
        lds_vec<CPL>(Ut + rl * us + c0, ui);
        lds_vec<CPL>(Ut + jl * us + c0, uj);
        if constexpr (HAS_ETA) {
          lds_vec<CPL>(Et + rl * us + c0, ei);
          lds_vec<CPL>(Et + jl * us + c0, ej);
        }
        double2 out[CPL];
        slot_values<CPL, POW, HAS_ETA>(pw, W[q], ui, uj, ei, ej, out);
        double2* vs = val + s * vs1 + c0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) vs[c] = out[c];
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- phase 1b: external edges (U_j, eta_j arrived asynchronously) ----
    if (active) {
      for (int s = n_int + grp; s < n_slots; s += G) {
        const int ent = list[s];
        const int rl = ent >> 16, q = ent & 0xFFFF;
        const double* xr = reinterpret_cast<const double*>(val + s * vs1);  // [U_j | eta_j]
        double ui[CPL], uj[CPL], ei[CPL] = {}, ej[CPL] = {};
        lds_vec<CPL>(Ut + rl * us + c0, ui);
        lds_vec<CPL>(xr + c0, uj);
        if constexpr (HAS_ETA) {
          lds_vec<CPL>(Et + rl * us + c0, ei);
          lds_vec<CPL>(xr + k + c0, ej);
        }
        __syncwarp(gmask);  // the whole group has read U_j, eta_j before the value overwrites them
        double2 out[CPL];
        slot_values<CPL, POW, HAS_ETA>(pw, W[q], ui, uj, ei, ej, out);
        double2* vs = val + s * vs1 + c0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) vs[c] = out[c];
      }
    }
    __syncthreads();

    // ---- phase 2: per-row sums in CSR order + row epilogue ----
    if (active) {
      for (int rl = grp; rl < nrows; rl += G) {
        const int b = R[rl] - e0, e = R[rl + 1] - e0;
        double ui[CPL], ei[CPL], L[CPL], HA[CPL];
        lds_vec<CPL>(Ut + rl * us + c0, ui);
        if constexpr (HAS_ETA) lds_vec<CPL>(Et + rl * us + c0, ei);
#pragma unroll
        for (int c = 0; c < CPL; ++c) L[c] = HA[c] = 0.0;
        for (int q = b; q < e; ++q) {
          const int c = C[q];
          const double2* vs = val + (c & 0xFFFF) * vs1 + c0;
          const double sg = c < 0 ? -1.0 : 1.0;  // lower row of an internal edge
#pragma unroll
          for (int c2 = 0; c2 < CPL; ++c2) {
            const double2 v = vs[c2];
            L[c2] = fma(sg, v.x, L[c2]);
            if constexpr (HAS_ETA) HA[c2] = fma(sg, v.y, HA[c2]);
          }
        }
        const int64_t row = r0 + rl;
        double g[CPL], h[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const double au = fabs(ui[c]);
          double sn, tn;
          pw.eval(au, sn, tn);
          accA[c] = fma(ui[c], L[c], accA[c]);
          accB[c] = fma(tn, au, accB[c]);
          const double phi = copysign(tn, ui[c]);
          g[c] = coef[c0 + c] * (L[c] - coef[k + c0 + c] * phi);
          if constexpr (HAS_ETA) {
            h[c] = coef[2 * k + c0 + c] * HA[c] - coef[3 * k + c0 + c] * sn * ei[c];
            if (a.want_dots) accAl[c] = fma(p * phi, ei[c], accAl[c]);
          } else {
            h[c] = 0.0;
          }
        }
        if (a.G != nullptr) st_vec<CPL>(a.G + row * k + c0, g);
        if constexpr (HAS_ETA) {
          if (a.Hv != nullptr) st_vec<CPL>(a.Hv + row * k + c0, h);
          if (a.want_dots) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) accGa[c] = fma(g[c], ei[c], accGa[c]);
          }
        }
      }
    }
    __syncthreads();  // the next tile's bulk copies overwrite the staging buffers
  }

  // ---- fixed-order CTA reduction of the partial sums (reuses the value area) ----
  double* red = reinterpret_cast<double*>(sm + Ly.val);  // [4][CPL][blockDim]
  const int nt = blockDim.x;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    red[(0 * CPL + c) * nt + threadIdx.x] = accA[c];
    red[(1 * CPL + c) * nt + threadIdx.x] = accB[c];
    red[(2 * CPL + c) * nt + threadIdx.x] = accAl[c];
    red[(3 * CPL + c) * nt + threadIdx.x] = accGa[c];
  }
  __syncthreads();
  for (int tt = threadIdx.x; tt < 4 * k; tt += nt) {
    const int q = tt / k, cl = tt % k;
    const int l = cl / CPL, c = cl % CPL;
    const double* base = red + (q * CPL + c) * nt;
    double s = 0.0;
    for (int th = l; th < nt; th += LPR) s += base[th];
    a.partials[((int64_t)blockIdx.x * 4 + q) * k + cl] = s;
  }
}

template <int CPL, int LPR, int KT, class POW, bool HAS_ETA>
plp_status launch_tiled_shape(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid_out) {
  auto kern = edge_tiled_kernel<CPL, LPR, KT, POW, HAS_ETA>;
  const TiledLayout Ly =
      tiled_layout(a.k, a.max_nnz, a.max_slots, a.max_ext, CPL, HAS_ETA, POW::kNeedsTables);
  static int attr_set = 0;
  static int occ = 1;
  if (attr_set < (int)Ly.total) {
    PLP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ly.total));
    attr_set = (int)Ly.total;
    int o = 0;
    PLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kEdgeThreads, Ly.total));
    occ = o < 1 ? 1 : o;
  }
  int64_t grid = (int64_t)occ * ctx->num_sms;
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  if (grid > a.n_tiles) grid = a.n_tiles > 0 ? a.n_tiles : 1;
  kern<<<(int)grid, kEdgeThreads, Ly.total, ctx->stream>>>(a, pw);
  PLP_LAUNCH_CHECK("edge_tiled_kernel");
  note_edge_kernel("edge_tiled_kernel", KT, CPL, LPR, 1, POW::kName, HAS_ETA);
  *grid_out = (int)grid;
  return PLP_OK;
}

#ifndef PLP_TILED_CPL
#define PLP_TILED_CPL 2  // columns per lane at k = 8 (2 or 4; tools/tune_edge.py)
#endif

// Launches the tiled kernel when the graph is tiled, k is even (16-byte column pairs), the dense
// arrays are 16-byte aligned and the tile fits in shared memory; *used = false otherwise.
template <class POW>
plp_status try_launch_tiled(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid, bool* used) {
  *used = false;
  const int k = a.k;
  auto al16 = [](const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; };
  // Kernel choice: the row kernel is the default until the tiled kernel measures
  // faster; PLP_EDGE_TILED=1 selects the tiled kernel, PLP_EDGE_ROWS=1 forces the row kernel.
  static const bool use_tiled = getenv("PLP_EDGE_TILED") != nullptr && getenv("PLP_EDGE_ROWS") == nullptr;
  if (!use_tiled || a.enc == nullptr || k % 2 != 0 || !al16(a.U) || (a.eta && !al16(a.eta)) ||
      (a.G && !al16(a.G)) || (a.Hv && !al16(a.Hv)))
    return PLP_OK;
  const TiledLayout Ly =
      tiled_layout(k, a.max_nnz, a.max_slots, a.max_ext, 4, a.eta != nullptr, POW::kNeedsTables);
  (void)Ly;
  if (Ly.total > 220u * 1024u) return PLP_OK;
  *used = true;
  const bool he = a.eta != nullptr;
  const int half = k / 2;
#define PLP_TSHAPE(C, L, KT)                                                          \
  return he ? launch_tiled_shape<C, L, KT, POW, true>(ctx, a, pw, grid)               \
            : launch_tiled_shape<C, L, KT, POW, false>(ctx, a, pw, grid)
  if (k == 8) {
    if constexpr (PLP_TILED_CPL == 4) PLP_TSHAPE(4, 2, 8);
    else PLP_TSHAPE(2, 4, 8);
  }
  if (k == 2) PLP_TSHAPE(2, 1, 2);
  if (k == 4) PLP_TSHAPE(2, 2, 4);
  if (k == 16) PLP_TSHAPE(4, 4, 16);
  if (half <= 4) PLP_TSHAPE(2, 4, 0);
  if (half <= 8) PLP_TSHAPE(2, 8, 0);
  PLP_TSHAPE(2, 16, 0);
#undef PLP_TSHAPE
}

// Edge-pass entry for one power policy: the halo-tile kernel where it applies, else
// the staged row kernel; PLP_EDGE_STAGED=1 forces the staged kernel, PLP_EDGE_TILED=1 selects the
// tiled kernel (where it applies), PLP_EDGE_ROWS=1 the unstaged row kernel (kept for comparison
// measurements and parity tests).
template <class POW>
plp_status launch_edge_any(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid) {
#ifdef PLP_TUNE_ONLY  // tuning builds (tools/tune_edge.py): k = 8 halo or staged shapes only
  if (a.k != 8) return set_error(PLP_ERR_ARG, "tuning build: k = 8 only");
  bool used_h = false;
  if (getenv("PLP_EDGE_STAGED") == nullptr) {
    plp_status sh = try_launch_halo(ctx, a, pw, grid, &used_h);
    if (sh || used_h) return sh;
  }
  return launch_staged_pow(ctx, a, pw, grid);
#else
  bool used = false;
  plp_status st = try_launch_tiled(ctx, a, pw, grid, &used);
  if (st || used) return st;
  static const bool rows = getenv("PLP_EDGE_ROWS") != nullptr;
  if (rows) return launch_edge_pow(ctx, a, pw, grid);
  static const bool staged = getenv("PLP_EDGE_STAGED") != nullptr;
  if (!staged) {
    st = try_launch_halo(ctx, a, pw, grid, &used);
    if (st || used) return st;
    // wide rows without a halo tiling (C4: k = 20 on a random block graph): the gathers are
    // latency-bound and the row kernel, without the staged kernel's shared-memory ring, keeps more
    // warps resident (C4: 2.04 against 2.41 ms)
    if (a.k > 16) return launch_edge_pow(ctx, a, pw, grid);
  }
  return launch_staged_pow(ctx, a, pw, grid);
#endif
}

}  // namespace plp
