// The fused F / EucGrad / EucHessianEta edge kernel.
//
// One pass over the CSR computes, per row i and column l:
//   per stored edge (i, j):  d = U_il - U_jl, a = |d|,  s = cap(a)^{p-2} (the one power), and
//                            dL with s dL = phi_p(d)  (dL = d unless a < eps)
//       L_il   += (w_ij s) dL                   ((Delta_p u)_i)
//       HA_il  += (w_ij s) (eta_il - eta_jl)    (Laplacian of w~ applied to eta; Alg. 1 lines 7-9)
//   per node:  sn = cap(|U_il|)^{p-2}, tn = |U_il|^{p-1}:
//       A'_l  += U_il L_il                      (= A_l summed over all rows: <u, Delta_p u> = A)
//       B'_l  += tn |U_il|                      (Eq. (1) denominator)
//       G_il  = (p/B_l) (L_il - (A_l/B_l) copysign(tn, U_il))                  (reading #4)
//       Hv_il = p(p-1)/B_l HA_il - p(p-1) A_l/B_l^2 sn eta_il                  (Alg. 1, #5)
// Thread mapping ("one warp or sub-warp per row with the k columns vectorised", north star):
//   a group of LPR lanes owns a row; lane li owns columns [li*CPL, li*CPL + CPL); a gathered
//   neighbour row U_j (8k bytes) is read by the group as LPR contiguous CPL-vectors (coalesced);
//   col_idx/w are broadcast within the group.  Rows are taken in the graph's schedule order
//   (degree-sorted within windows, plp_create_graph) so the groups of a warp have near-equal
//   degrees.  Persistent grid-stride loop; each CTA reduces its A', B', alpha, gamma partials in a
//   fixed order (no atomics).
#pragma once
#include "plp_internal.h"
#include "pow64.cuh"

#ifndef PLP_LD256
#define PLP_LD256 1  // 256-bit gathers for 4-column lanes
#endif

namespace plp {

template <int CPL>
__device__ __forceinline__ void ld_vec(const double* __restrict__ p, double (&v)[CPL]) {
  if constexpr (CPL % 4 == 0 && PLP_LD256) {
    // 256-bit loads (LDG.E.ENL2.256 on sm_100a): a 4-column lane segment in one request (the
    // launchers select CPL = 4 only for 32-byte aligned arrays)
#pragma unroll
    for (int c = 0; c < CPL; c += 4)
      asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(v[c]), "=d"(v[c + 1]), "=d"(v[c + 2]), "=d"(v[c + 3])
                   : "l"(p + c));
  } else if constexpr (CPL % 2 == 0) {
#pragma unroll
    for (int c = 0; c < CPL; c += 2) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p + c));
      v[c] = t.x;
      v[c + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = __ldg(p + c);
  }
}

template <int CPL>
__device__ __forceinline__ void lds_vec(const double* p, double (&v)[CPL]) {
  if constexpr (CPL % 2 == 0) {
#pragma unroll
    for (int c = 0; c < CPL; c += 2) {
      const double2 t = *reinterpret_cast<const double2*>(p + c);
      v[c] = t.x;
      v[c + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = p[c];
  }
}

template <int CPL>
__device__ __forceinline__ void st_vec(double* __restrict__ p, const double (&v)[CPL]) {
  if constexpr (CPL % 4 == 0) {
#pragma unroll
    for (int c = 0; c < CPL; c += 4)
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + c), "d"(v[c]), "d"(v[c + 1]),
                   "d"(v[c + 2]), "d"(v[c + 3])
                   : "memory");
  } else if constexpr (CPL % 2 == 0) {
#pragma unroll
    for (int c = 0; c < CPL; c += 2) *reinterpret_cast<double2*>(p + c) = make_double2(v[c], v[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < CPL; ++c) p[c] = v[c];
  }
}

constexpr int kEdgeThreads = 256;
// Tuning knobs (tools/tune_edge.py builds variants): edges unrolled per step, min CTAs per SM
// (register cap), and 4-column lanes for k % 4 == 0.
#ifndef PLP_EDGE_UNR
#define PLP_EDGE_UNR 4
#endif
#ifndef PLP_EDGE_MINB
#define PLP_EDGE_MINB 2
#endif
#ifndef PLP_EDGE_CPL4
#define PLP_EDGE_CPL4 0
#endif

// One stored edge (weight wv) for the lane's CPL columns; branch-free.
template <int CPL, class POW, bool HAS_ETA>
__device__ __forceinline__ void edge_update(const POW& pw, double wv,
                                            const double (&ui)[CPL], const double (&uj)[CPL],
                                            const double (&ei)[CPL], const double (&ej)[CPL],
                                            double (&L)[CPL], double (&HA)[CPL], unsigned& bad) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    const double d = ui[c] - uj[c];
    if constexpr (POW::kIsP2) {
      L[c] = fma(wv, d, L[c]);
      if constexpr (HAS_ETA) HA[c] = fma(wv, ei[c] - ej[c], HA[c]);
    } else {
      // fast domain: |d| >= eps (no cap) and the branch-free power is valid; anything else
      // (ties, |d| < eps, extreme magnitudes) flags the row for the exact recomputation
      bad |= (unsigned)!pw.fast_hi(d);
      const double wsr = wv * pw.pow_fast(d);  // w |d|^{p-2}
      L[c] = fma(wsr, d, L[c]);                // w phi_p(d)
      if constexpr (HAS_ETA) HA[c] = fma(wsr, ei[c] - ej[c], HA[c]);
    }
  }
}

// Exact (libdevice) recomputation of a row's sums when some |d| left the fast domain (rare).
template <int CPL, class POW, bool HAS_ETA>
__device__ __forceinline__ void edge_row_exact(const POW& pw, int e0, int e1, const int32_t* col,
                                            const double* wt, const double* U, const double* eta,
                                            int k, int c0, const double (&ui)[CPL],
                                            const double (&ei)[CPL], double (&L)[CPL],
                                            double (&HA)[CPL]) {
#pragma unroll
  for (int c = 0; c < CPL; ++c) L[c] = HA[c] = 0.0;
  for (int e = e0; e < e1; ++e) {
    const int64_t j = col[e];
    const double wv = wt[e];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const double d = ui[c] - U[j * k + c0 + c];
      const double a = fabs(d);
      L[c] += wv * ((a != 0.0) ? copysign(pow(a, pw.pm1), d) : 0.0);
      if constexpr (HAS_ETA) {
        const double s = (a < pw.eps) ? pw.s_eps : pow(a, pw.q);
        HA[c] += wv * s * (ei[c] - eta[j * k + c0 + c]);
      }
    }
  }
}

// UNR_T: edges per gather batch (0: the PLP_EDGE_UNR default).  LPR need not divide 32 (k = 20:
// 10 lanes x 2 columns, 3 rows per warp, 2 idle lanes): lanes past the last row group are idle.
template <int CPL, int LPR, class POW, bool HAS_ETA, int UNR_T = 0>
__global__ void __launch_bounds__(kEdgeThreads, PLP_EDGE_MINB) edge_kernel(EdgeArgs a, POW pw) {
  extern __shared__ double4 smem_raw[];
  if constexpr (POW::kNeedsTables) {
    pw.init_smem(smem_raw);
    __syncthreads();
  }
  constexpr int RPW = 32 / LPR;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int grp = lane / LPR;
  const int li = lane % LPR;
  const int rows_per_iter = (blockDim.x >> 5) * RPW;
  const int k = a.k;
  const int c0 = li * CPL;
  // k even when CPL is even, so a lane owns all or none of its columns
  const bool active = c0 < k && grp < RPW;
  const double p = a.p;
  const double pp1 = p * (p - 1.0);

  double cG[CPL], cAB[CPL], cHA[CPL], cHB[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) cG[c] = cAB[c] = cHA[c] = cHB[c] = 0.0;
  if (a.AB != nullptr && active) {
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const double A = a.AB[c0 + c], B = a.AB[k + c0 + c];
      cG[c] = p / B;               // p / B
      cAB[c] = A / B;              // A / B
      cHA[c] = pp1 / B;            // p(p-1) / B
      cHB[c] = pp1 * A / (B * B);  // p(p-1) A / B^2
    }
  }
  double accA[CPL], accB[CPL], accAl[CPL], accGa[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) accA[c] = accB[c] = accAl[c] = accGa[c] = 0.0;

  const int32_t* __restrict__ rp = a.rp;
  const int32_t* __restrict__ col = a.col;
  const int32_t* __restrict__ sched = a.sched;
  const double* __restrict__ wt = a.w;
  const double* __restrict__ U = a.U;
  const double* __restrict__ eta = a.eta;

  if (active) {
    const int64_t stride = (int64_t)gridDim.x * rows_per_iter;
    int64_t idx = (int64_t)blockIdx.x * rows_per_iter + warp * RPW + grp;
    // software pipeline: the next row's schedule entry and row bounds are loaded one iteration
    // ahead, so each row starts with its edge metadata already in flight
    int row = idx < a.n_rows ? __ldg(sched + idx) : 0;
    int e0 = idx < a.n_rows ? __ldg(rp + row) : 0, e1 = idx < a.n_rows ? __ldg(rp + row + 1) : 0;
    for (; idx < a.n_rows; idx += stride) {
      const int64_t idxn = idx + stride;
      const int rown = idxn < a.n_rows ? __ldg(sched + idxn) : row;
      double ui[CPL], ei[CPL];
      ld_vec<CPL>(U + (int64_t)row * k + c0, ui);
      if constexpr (HAS_ETA) ld_vec<CPL>(eta + (int64_t)row * k + c0, ei);
      double L[CPL], HA[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) L[c] = HA[c] = 0.0;

      // edges in batches of UNR; the last batch is padded with weight-0 copies of the first edge
      constexpr int UNR = UNR_T > 0 ? UNR_T : (CPL <= 2) ? PLP_EDGE_UNR : (PLP_EDGE_UNR + 1) / 2;
      unsigned bad = 0;
      const int jpad = e0 < e1 ? __ldg(col + e0) : row;
      for (int e = e0; e < e1; e += UNR) {
        int j[UNR];
        double wv[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const bool v = e + u < e1;
          j[u] = v ? __ldg(col + e + u) : jpad;
          wv[u] = v ? __ldg(wt + e + u) : 0.0;
        }
        double uj[UNR][CPL], ej[UNR][CPL];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          ld_vec<CPL>(U + (int64_t)j[u] * k + c0, uj[u]);
          if constexpr (HAS_ETA) ld_vec<CPL>(eta + (int64_t)j[u] * k + c0, ej[u]);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          edge_update<CPL, POW, HAS_ETA>(pw, wv[u], ui, uj[u], ei, ej[u], L, HA, bad);
        }
      }
      const int e0n = __ldg(rp + rown), e1n = __ldg(rp + rown + 1);
      if (bad) edge_row_exact<CPL, POW, HAS_ETA>(pw, e0, e1, col, wt, U, eta, k, c0, ui, ei, L, HA);

      // ---- row epilogue: node terms, outputs, partial sums ----
      double g[CPL], h[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const double au = fabs(ui[c]);
        double sn, tn;
        pw.eval(au, sn, tn);
        accA[c] = fma(ui[c], L[c], accA[c]);
        accB[c] = fma(tn, au, accB[c]);
        const double phi = copysign(tn, ui[c]);
        g[c] = cG[c] * (L[c] - cAB[c] * phi);
        if constexpr (HAS_ETA) {
          h[c] = cHA[c] * HA[c] - cHB[c] * sn * ei[c];
          if (a.want_dots) accAl[c] = fma(p * phi, ei[c], accAl[c]);
        } else {
          h[c] = 0.0;
        }
      }
      if (a.G != nullptr) st_vec<CPL>(a.G + (int64_t)row * k + c0, g);
      if constexpr (HAS_ETA) {
        if (a.Hv != nullptr) st_vec<CPL>(a.Hv + (int64_t)row * k + c0, h);
        if (a.want_dots) {
#pragma unroll
          for (int c = 0; c < CPL; ++c) accGa[c] = fma(g[c], ei[c], accGa[c]);
        }
      }
      row = rown;
      e0 = e0n;
      e1 = e1n;
    }
  }

  // ---- fixed-order CTA reduction of the partial sums ----
  __syncthreads();
  double* red = reinterpret_cast<double*>(smem_raw);  // [4][CPL][blockDim]
  const int nt = blockDim.x;
#pragma unroll
  for (int c = 0; c < CPL; ++c) {
    red[(0 * CPL + c) * nt + threadIdx.x] = accA[c];
    red[(1 * CPL + c) * nt + threadIdx.x] = accB[c];
    red[(2 * CPL + c) * nt + threadIdx.x] = accAl[c];
    red[(3 * CPL + c) * nt + threadIdx.x] = accGa[c];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 4 * k; t += nt) {
    const int q = t / k, cl = t % k;
    const int l = cl / CPL, c = cl % CPL;
    const double* base = red + (q * CPL + c) * nt;
    double s = 0.0;
    for (int w = 0; w < (nt >> 5); ++w)
      for (int gg = 0; gg < RPW; ++gg) s += base[w * 32 + gg * LPR + l];  // idle lanes hold zeros
    a.partials[((int64_t)blockIdx.x * 4 + q) * k + cl] = s;
  }
}

template <int CPL, int LPR, class POW, bool HAS_ETA, int UNR_T = 0>
plp_status launch_edge_shape(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid_out) {
  auto kern = edge_kernel<CPL, LPR, POW, HAS_ETA, UNR_T>;
  const size_t red_bytes = (size_t)4 * CPL * kEdgeThreads * sizeof(double);
  const size_t tab_bytes = POW::kNeedsTables ? sizeof(PowTables) : 0;
  const size_t smem = red_bytes > tab_bytes ? red_bytes : tab_bytes;
  static int occ = -1;  // per instantiation
  if (occ < 0) {
    if (smem > 48 * 1024)
      PLP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int o = 0;
    PLP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kEdgeThreads, smem));
    occ = o < 1 ? 1 : o;
  }
  const int rows_per_iter = (kEdgeThreads / 32) * (32 / LPR);
  int64_t need = (a.n_rows + rows_per_iter - 1) / rows_per_iter;
  int grid = occ * ctx->num_sms;
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  if (need < grid) grid = (int)(need > 0 ? need : 1);
  kern<<<grid, kEdgeThreads, smem, ctx->stream>>>(a, pw);
  PLP_LAUNCH_CHECK("edge_kernel");
  note_edge_kernel("edge_kernel", 0, CPL, LPR, UNR_T > 0 ? UNR_T : (CPL <= 2) ? PLP_EDGE_UNR : (PLP_EDGE_UNR + 1) / 2,
                   POW::kName, HAS_ETA);
  *grid_out = grid;
  return PLP_OK;
}

// Dispatch on k (and alignment) to a (CPL, LPR) shape.
template <class POW>
plp_status launch_edge_pow(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid) {
  const int k = a.k;
  auto al16 = [](const void* ptr) { return ((uintptr_t)ptr & 15u) == 0; };
  const bool vec_ok = (k % 2 == 0) && al16(a.U) && (a.eta == nullptr || al16(a.eta)) &&
                      (a.G == nullptr || al16(a.G)) && (a.Hv == nullptr || al16(a.Hv));
  const bool he = a.eta != nullptr;
#define PLP_SHAPE(C, L)                                                                 \
  return he ? launch_edge_shape<C, L, POW, true>(ctx, a, pw, grid)                      \
            : launch_edge_shape<C, L, POW, false>(ctx, a, pw, grid)
  if constexpr (PLP_EDGE_CPL4 != 0) {
    if (vec_ok && k % 4 == 0) {
      const int quarter = k / 4;
      if (quarter <= 1) PLP_SHAPE(4, 1);
      if (quarter <= 2) PLP_SHAPE(4, 2);
      if (quarter <= 4) PLP_SHAPE(4, 4);
      PLP_SHAPE(4, 8);
    }
  }
#ifndef PLP_EDGE_K20_UNR
#define PLP_EDGE_K20_UNR 4  // k = 20 (C4): edges per gather batch (8 and 12 measured slower: registers)
#endif
  if (vec_ok && k == 20) {
    return he ? launch_edge_shape<2, 10, POW, true, PLP_EDGE_K20_UNR>(ctx, a, pw, grid)
              : launch_edge_shape<2, 10, POW, false, PLP_EDGE_K20_UNR>(ctx, a, pw, grid);
  }
  if (vec_ok) {
    const int half = k / 2;
    if (half <= 1) PLP_SHAPE(2, 1);
    if (half <= 2) PLP_SHAPE(2, 2);
    if (half <= 4) PLP_SHAPE(2, 4);
    if (half <= 8) PLP_SHAPE(2, 8);
    PLP_SHAPE(2, 16);
  }
  if (k <= 1) PLP_SHAPE(1, 1);
  if (k <= 2) PLP_SHAPE(1, 2);
  if (k <= 4) PLP_SHAPE(1, 4);
  if (k <= 8) PLP_SHAPE(1, 8);
  if (k <= 16) PLP_SHAPE(1, 16);
  PLP_SHAPE(1, 32);
#undef PLP_SHAPE
}

}  // namespace plp
