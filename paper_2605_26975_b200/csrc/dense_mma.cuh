// Tall-skinny Gram and apply kernels on the fp64 tensor cores (DMMA, mma.sync m8n8k4 f64) for
// k = 8 and k = 16 ("tensor cores only for the k x k Gram products if they
// pay").  They pay in instructions, not flops: one warp instruction does 4 rows x 8 x 8 FMAs of a
// Gram, fed by two coalesced 256-byte loads, so the kernels stream at the HBM rate where the scalar
// versions (dense.cu) were issue/latency bound.
//   gram:   C (k x k) = sum_r (X_r + Xa_r)^T (Y_r + Ya_r), per-CTA partials reduced in a fixed order
//           (sum_partials_kernel) -- A fragment = 4 rows of X transposed, B fragment = 4 rows of Y
//           (SYM: Y = X, Ya = Xa, one set of loads);
//   apply:  out_r = S_r + sgn (X_r + Xa_r) M for 8-row blocks -- A = 8 rows x 4 columns of X,
//           B = 4 x 8 slice of sgn M, C/D = the block of S / out (out may alias S, X or Xa: each
//           warp reads its rows before writing them).
#pragma once
#include "plp_internal.h"

namespace plp {

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int kMmaThreads = 256;

// k = 8 KT.  Each warp owns a contiguous range of 4-row blocks; D[ta][tb] holds
// C[8 ta + g][8 tb + 2 q + {0, 1}] with g = lane / 4, q = lane % 4.
template <int KT, bool SYM>
__global__ void __launch_bounds__(kMmaThreads) gram_mma_kernel(int64_t n, const double* __restrict__ X,
                                                               const double* __restrict__ Xa,
                                                               const double* __restrict__ Y,
                                                               const double* __restrict__ Ya,
                                                               double* __restrict__ part) {
  constexpr int K = 8 * KT, E = K * K, NW = kMmaThreads / 32;
  __shared__ double red[NW][E];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t blocks = (n + 3) / 4;
  const int64_t tw = (int64_t)gridDim.x * NW, wid = (int64_t)blockIdx.x * NW + warp;
  const int64_t b0 = blocks * wid / tw, b1 = blocks * (wid + 1) / tw;
  double d[KT][KT][2];
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < KT; ++j) d[i][j][0] = d[i][j][1] = 0.0;
  // lane's element of a 4-row block: row 4 b + q, column 8 t + g
  constexpr int UNR = 4;
  int64_t b = b0;
  for (; b + UNR <= b1; b += UNR) {
    double a[UNR][KT], c[UNR][KT];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t r = 4 * (b + u) + q;
      const bool ok = r < n;
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        const int64_t o = r * K + 8 * t + g;
        a[u][t] = ok ? __ldg(X + o) + (Xa ? __ldg(Xa + o) : 0.0) : 0.0;
        c[u][t] = SYM ? a[u][t] : ok ? __ldg(Y + o) + (Ya ? __ldg(Ya + o) : 0.0) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u)
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) dmma884(d[i][j][0], d[i][j][1], a[u][i], c[u][j]);
  }
  for (; b < b1; ++b) {
    const int64_t r = 4 * b + q;
    const bool ok = r < n;
    double a[KT], c[KT];
#pragma unroll
    for (int t = 0; t < KT; ++t) {
      const int64_t o = r * K + 8 * t + g;
      a[t] = ok ? __ldg(X + o) + (Xa ? __ldg(Xa + o) : 0.0) : 0.0;
      c[t] = SYM ? a[t] : ok ? __ldg(Y + o) + (Ya ? __ldg(Ya + o) : 0.0) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < KT; ++i)
#pragma unroll
      for (int j = 0; j < KT; ++j) dmma884(d[i][j][0], d[i][j][1], a[i], c[j]);
  }
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < KT; ++j) {
      red[warp][(8 * i + g) * K + 8 * j + 2 * q] = d[i][j][0];
      red[warp][(8 * i + g) * K + 8 * j + 2 * q + 1] = d[i][j][1];
    }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kMmaThreads) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) s += red[w][e];
    part[(int64_t)blockIdx.x * E + e] = s;
  }
}

// out = S + sgn (X + Xa) M, k = 8 KT, 8-row blocks per warp instruction group.
template <int KT>
__global__ void __launch_bounds__(kMmaThreads) apply_mma_kernel(int64_t n, const double* S, double sgn,
                                                                const double* X, const double* Xa,
                                                                const double* __restrict__ M,
                                                                double* out) {
  constexpr int K = 8 * KT, NW = kMmaThreads / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  // B fragments of sgn M: slice (ta, ks) -> rows 8 ta + 4 ks + q, column block tb: column 8 tb + g
  double bm[KT][2][KT];
#pragma unroll
  for (int ta = 0; ta < KT; ++ta)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int tb = 0; tb < KT; ++tb) bm[ta][ks][tb] = sgn * M[(8 * ta + 4 * ks + q) * K + 8 * tb + g];
  const int64_t blocks = (n + 7) / 8;
  const int64_t tw = (int64_t)gridDim.x * NW, wid = (int64_t)blockIdx.x * NW + warp;
  const int64_t b0 = blocks * wid / tw, b1 = blocks * (wid + 1) / tw;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t r = 8 * b + g;
    const bool ok = r < n;
    double a[KT][2];
#pragma unroll
    for (int ta = 0; ta < KT; ++ta)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int64_t o = r * K + 8 * ta + 4 * ks + q;
        a[ta][ks] = ok ? X[o] + (Xa ? Xa[o] : 0.0) : 0.0;
      }
    double d[KT][2];
#pragma unroll
    for (int tb = 0; tb < KT; ++tb) {
      const int64_t o = r * K + 8 * tb + 2 * q;
      if (S != nullptr && ok) {
        const double2 s2 = *reinterpret_cast<const double2*>(S + o);
        d[tb][0] = s2.x;
        d[tb][1] = s2.y;
      } else {
        d[tb][0] = d[tb][1] = 0.0;
      }
    }
#pragma unroll
    for (int tb = 0; tb < KT; ++tb)
#pragma unroll
      for (int ta = 0; ta < KT; ++ta)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) dmma884(d[tb][0], d[tb][1], a[ta][ks], bm[ta][ks][tb]);
    if (ok) {
#pragma unroll
      for (int tb = 0; tb < KT; ++tb)
        *reinterpret_cast<double2*>(out + r * K + 8 * tb + 2 * q) = make_double2(d[tb][0], d[tb][1]);
    }
  }
}

}  // namespace plp
