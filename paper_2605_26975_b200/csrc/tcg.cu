// Device-resident truncated CG (Steihaug-Toint; Absil-Baker-Gallivan 2007, Alg. 2) for the
// trust-region subproblem of the Grassmann Newton solver (SURVEY.md §8(f) NEXT-1,
// "CUDA-Graph the tCG iteration").  The same recurrences as solver.py's host loop, with every
// scalar kept on the device: one iteration is a fixed launch sequence (Hessian-vector product,
// projection, curvature term, dots, scalar updates, axpbys with device coefficients), so the host
// can launch many iterations without reading anything back and the sequence can be captured in a
// CUDA graph.  The scalar kernels use explicitly rounded fp64 operations in the host code's order
// (no FMA contraction), so the device recurrence is bitwise that of solver.py's loop; after the
// exit condition every further iteration is a no-op for eta, Heta, r and delta.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "dense_mma.cuh"
#include "plp_internal.h"

namespace plp {

// scalar slots (double sc[PLP_TCG_SCAL_LEN]) and status (int st[2] = {status, iterations});
// the fused path also keeps its reduction totals in sc (from kMat)
enum {
  kZr = 0, kStopTol = 1, kDelta = 2, kEPe = 3, kEPd = 4, kDPd = 5, kDHd = 6, kAlpha = 7,
  kZnew = 9, kCEta = 10, kCR = 11, kCA = 12, kCB = 13, kTrDE = 14, kZraw = 15, kMat = 64
};
// totals of pass A at kTotA = [M1 | M2 | tr | <Gdd, S>] (M1 first, read by pass B), of pass B at
// kTotB = [MR | ||r||^2] (MR read by pass C)
constexpr int kTotA = kMat, kM1 = kTotA, kTotB = kMat + 2 * PLP_MAX_K * PLP_MAX_K + 64, kMR = kTotB;
constexpr int kSx = kTotB + PLP_MAX_K * PLP_MAX_K + 64;  // S expanded block-diagonally (folded k < 8)
static_assert(kSx + 64 <= PLP_TCG_SCAL_LEN, "scal too short");

__global__ void tcg_init_kernel(double* sc, int* st, double delta, double kappa, double theta) {
  const double zr = sc[kZr];
  const double r0 = sqrt(zr);
  const double rt = pow(r0, theta);
  sc[kStopTol] = __dmul_rn(r0, rt < kappa ? rt : kappa);
  sc[kDelta] = delta;
  sc[kEPe] = 0.0;
  sc[kEPd] = 0.0;
  sc[kDPd] = zr;
  st[0] = r0 == 0.0 ? PLP_TCG_INTERIOR : PLP_TCG_RUNNING;
  st[1] = 0;
}

// after <delta, H delta>: step length, trust-boundary / negative-curvature exit
__device__ void tcg_scalar_a(double* sc, int* st) {
  if (st[0] != PLP_TCG_RUNNING) {
    sc[kCEta] = 0.0;
    sc[kCR] = 0.0;
    return;
  }
  st[1] += 1;
  const double zr = sc[kZr], dHd = sc[kDHd], ePe = sc[kEPe], ePd = sc[kEPd], dPd = sc[kDPd];
  const double delta = sc[kDelta];
  const double alpha = dHd != 0.0 ? zr / dHd : INFINITY;
  // e_Pe + 2 alpha e_Pd + alpha alpha d_Pd, left to right as in solver.py
  const double ePe_new =
      __dadd_rn(__dadd_rn(ePe, __dmul_rn(__dmul_rn(2.0, alpha), ePd)), __dmul_rn(__dmul_rn(alpha, alpha), dPd));
  const double dd = __dmul_rn(delta, delta);
  if (dHd <= 0.0 || ePe_new >= dd) {
    const double disc = __dadd_rn(__dmul_rn(ePd, ePd), __dmul_rn(dPd, __dsub_rn(dd, ePe)));
    const double tau = __ddiv_rn(__dadd_rn(-ePd, sqrt(disc)), dPd);
    sc[kCEta] = tau;
    sc[kCR] = 0.0;
    st[0] = dHd <= 0.0 ? PLP_TCG_NEGATIVE_CURVATURE : PLP_TCG_BOUNDARY;
    return;
  }
  sc[kEPe] = ePe_new;
  sc[kAlpha] = alpha;
  sc[kCEta] = alpha;
  sc[kCR] = alpha;
}

__global__ void tcg_scalar_a_kernel(double* sc, int* st) { tcg_scalar_a(sc, st); }

// after <r, r>: convergence test, conjugation; returns whether the iteration goes on
__device__ bool tcg_scalar_b(double* sc, int* st, int max_iters) {
  if (st[0] != PLP_TCG_RUNNING) {
    sc[kCA] = 0.0;
    sc[kCB] = 1.0;
    return false;
  }
  const double znew = sc[kZnew];
  if (sqrt(znew) <= sc[kStopTol]) {
    st[0] = PLP_TCG_CONVERGED;
    sc[kCA] = 0.0;
    sc[kCB] = 1.0;
    return false;
  }
  const double zr = sc[kZr], alpha = sc[kAlpha], ePd = sc[kEPd], dPd = sc[kDPd];
  const double beta = __ddiv_rn(znew, zr);
  sc[kZr] = znew;
  sc[kCA] = -1.0;
  sc[kCB] = beta;
  sc[kEPd] = __dmul_rn(beta, __dadd_rn(ePd, __dmul_rn(alpha, dPd)));
  sc[kDPd] = __dadd_rn(znew, __dmul_rn(__dmul_rn(beta, beta), dPd));
  if (st[1] >= max_iters) st[0] = PLP_TCG_MAXITER;
  return true;
}

__global__ void tcg_scalar_b_kernel(double* sc, int* st, int max_iters) { tcg_scalar_b(sc, st, max_iters); }

// ---------------------------------------------------------------------------------------------
// Fused iteration for k = 8 KT: after the edge pass writes EH =
// EucHess[d], three streaming passes replace the nine tall-skinny launches of the unfused loop.
// With d horizontal (U^T d = 0 up to rounding) and Hd = EH - U M1 - d S, M1 = U^T EH:
//   <d, Hd> = tr(d^T EH) - <U^T d, M1>_F - <d^T d, S>_F                    (pass A: Grams only)
//   eta += c d, Heta += c Hd, r += c' Hd, MR = U^T r, ||r||^2                (pass B: Hd never stored)
//   r <- r - U MR (the residual's re-projection), ||P r||^2 = ||r||^2 - ||MR||_F^2,
//   d <- -r + beta d                                                          (pass C)
// Pass C writes only d: the stored r keeps the un-projected residual and the next pass B applies
// -U MR (MR still in scal[kMR]) to it before adding cr Hd -- the same operations in the same
// order, so the iterates are bitwise those of writing r in pass C, and each iteration moves 8 n k
// bytes less.  The last iteration of a tcg_run batch writes r (projected) and zeroes scal[kMR], so
// r is the projected residual between calls.
// All Grams and the k x k applies run on the fp64 tensor cores (dmma884, as dense_mma.cuh).
// ---------------------------------------------------------------------------------------------
constexpr int kTcgThreads = 256, kTcgWarps = kTcgThreads / 32;

// Grid reductions: each pass CTA writes its E block totals entry-major (part[e * P + cta]); then
// tcg_reduce_kernel runs one CTA per entry (coalesced fixed-order sum: thread-strided, warp xor
// tree, warps in order) and its last CTA (ticket) applies the scalar step on the totals.
// pass A: [M1 | M2 | tr(d^T EH) | <d^T d, S>_F] over 4-row blocks
#ifndef PLP_TCG_DS_LDG
#define PLP_TCG_DS_LDG 0  // 1: k = 8 reads the row of d for d S from L1 instead of 8 shuffles
#endif
#ifndef PLP_TCG_DHD_ROWWISE
#define PLP_TCG_DHD_ROWWISE 1  // <d, EH - d S> element by element (cancellation before the sum)
#endif
#ifndef PLP_TCG_MINB_A
#define PLP_TCG_MINB_A 3
#endif
template <int KT, int UNR>
__global__ void __launch_bounds__(kTcgThreads, KT == 1 ? PLP_TCG_MINB_A : 1) tcg_gram_a_kernel(int64_t n, const double* __restrict__ U,
                                                                 const double* __restrict__ EH,
                                                                 const double* __restrict__ D,
                                                                 const double* __restrict__ S,
                                                                 double* __restrict__ part) {
  constexpr int K = 8 * KT, KK = K * K, E = 2 * KK + 2;
  __shared__ double red[E];
  __shared__ double sS[KK];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  for (int e = threadIdx.x; e < E; e += kTcgThreads) red[e] = 0.0;
  for (int e = threadIdx.x; e < KK; e += kTcgThreads) sS[e] = S[e];
  __syncthreads();
  double sc1[8];  // k = 8: the lane's column g of S in registers
#pragma unroll
  for (int a = 0; a < 8; ++a) sc1[a] = KT == 1 ? sS[a * K + g] : 0.0;
  double m1[KT][KT][2], m2[KT][KT][2], gd[KT][KT][2], tr = 0.0, ds = 0.0;
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < KT; ++j) m1[i][j][0] = m1[i][j][1] = m2[i][j][0] = m2[i][j][1] = gd[i][j][0] = gd[i][j][1] = 0.0;
  double de[KT][2];
#pragma unroll
  for (int i = 0; i < KT; ++i) de[i][0] = de[i][1] = 0.0;
  const int64_t blocks = (n + 3) / 4;
  const int64_t tw = (int64_t)gridDim.x * kTcgWarps, wid = (int64_t)blockIdx.x * kTcgWarps + warp;
  const int64_t b0 = blocks * wid / tw, b1 = blocks * (wid + 1) / tw;
  for (int64_t b = b0; b < b1; b += UNR) {
    double u[UNR][KT], h[UNR][KT], dd[UNR][KT];
#pragma unroll
    for (int v = 0; v < UNR; ++v) {
      const int64_t r = 4 * (b + v) + q;
      const bool ok = b + v < b1 && r < n;
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        const int64_t o = r * K + 8 * t + g;
        u[v][t] = ok ? __ldg(U + o) : 0.0;
        h[v][t] = ok ? __ldg(EH + o) : 0.0;
        dd[v][t] = ok ? __ldg(D + o) : 0.0;
      }
    }
#pragma unroll
    for (int v = 0; v < UNR; ++v) {
#pragma unroll
      for (int i = 0; i < KT; ++i) {
#pragma unroll
        for (int j = 0; j < KT; ++j) {
          dmma884(m1[i][j][0], m1[i][j][1], u[v][i], h[v][j]);
          dmma884(m2[i][j][0], m2[i][j][1], u[v][i], dd[v][j]);
#if !PLP_TCG_DHD_ROWWISE
          dmma884(gd[i][j][0], gd[i][j][1], dd[v][i], dd[v][j]);
#endif
        }
#if !PLP_TCG_DHD_ROWWISE
        dmma884(de[i][0], de[i][1], dd[v][i], h[v][i]);
#endif
      }
#if PLP_TCG_DHD_ROWWISE
      // d (EH - d S) per element; (d S)[r][c] = sum_a d[r][a] S[a][c], the row's d values from the
      // lanes with the same q (a = 8 t2 + g2 ascending)
#if PLP_TCG_DS_LDG
      if constexpr (KT == 1) {
        // the row's d values straight from L1 (the 8 lanes of a row read the same 64 bytes)
        const int64_t rr = 4 * (b + v) + q;
        double drow[8];
        if (b + v < b1 && rr < n) {
#pragma unroll
          for (int a2 = 0; a2 < 8; a2 += 2) {
            const double2 x = __ldg(reinterpret_cast<const double2*>(D + rr * K + a2));
            drow[a2] = x.x;
            drow[a2 + 1] = x.y;
          }
        } else {
#pragma unroll
          for (int a2 = 0; a2 < 8; ++a2) drow[a2] = 0.0;
        }
        double dS = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < 8; ++g2) dS = fma(drow[g2], sc1[g2], dS);
        tr = fma(dd[v][0], h[v][0] - dS, tr);
      } else
#endif
      {
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        double dS = 0.0;
#pragma unroll
        for (int t2 = 0; t2 < KT; ++t2)
#pragma unroll
          for (int g2 = 0; g2 < 8; ++g2)
            dS = fma(__shfl_sync(0xffffffffu, dd[v][t2], g2 * 4 + q),
                     KT == 1 ? sc1[g2] : sS[(8 * t2 + g2) * K + 8 * t + g], dS);
        tr = fma(dd[v][t], h[v][t] - dS, tr);
      }
      }
#endif
    }
  }
#if !PLP_TCG_DHD_ROWWISE
  // diagonal of the d^T EH tiles: element (8i + g, 8i + 2q + h) is diagonal iff g == 2q + h
#pragma unroll
  for (int i = 0; i < KT; ++i) tr += (g == 2 * q ? de[i][0] : 0.0) + (g == 2 * q + 1 ? de[i][1] : 0.0);
  // <d^T d, S>_F from this lane's fragment of d^T d (S is known before the pass)
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < KT; ++j)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) ds = fma(gd[i][j][hh], sS[(8 * i + g) * K + 8 * j + 2 * q + hh], ds);
#endif
  (void)gd;
  (void)de;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    tr += __shfl_xor_sync(0xffffffffu, tr, o);
    ds += __shfl_xor_sync(0xffffffffu, ds, o);
  }
  __syncthreads();
  for (int w = 0; w < kTcgWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int e = (8 * i + g) * K + 8 * j + 2 * q + hh;
            red[e] += m1[i][j][hh];
            red[KK + e] += m2[i][j][hh];
          }
      if (lane == 0) {
        red[2 * KK] += tr;
        red[2 * KK + 1] += ds;
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < E; e += kTcgThreads) part[(int64_t)e * gridDim.x + blockIdx.x] = red[e];
}

// pass B over 8-row blocks: Hd = EH - U M1 - d S on the tensor cores (accumulator = EH),
// eta += ce d, Heta += ce Hd, r += cr Hd, then partials of MR = U^T r and ||r||^2.
#ifndef PLP_TCG_MINB_B
#define PLP_TCG_MINB_B 4  // k = 8: 4 CTAs (32 warps) per SM at <= 64 registers, no spills
#endif
template <int KT, bool HETA>
__global__ void __launch_bounds__(kTcgThreads, KT == 1 ? PLP_TCG_MINB_B : 1) tcg_update_kernel(int64_t n, const double* __restrict__ U,
                                                                 const double* __restrict__ EH,
                                                                 const double* __restrict__ D,
                                                                 const double* __restrict__ S,
                                                                 const double* sc,
                                                                 double* __restrict__ eta,
                                                                 double* __restrict__ Heta,
                                                                 double* __restrict__ r,
                                                                 double* __restrict__ part) {
  constexpr int K = 8 * KT, KK = K * K, E = KK + 1;
  __shared__ double red[E];
  __shared__ __align__(16) double tile[kTcgWarps][8 * K];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  for (int e = threadIdx.x; e < E; e += kTcgThreads) red[e] = 0.0;
  // B fragments of -M1 and -S: rows 8 ta + 4 ks + q, column 8 tb + g
  double bm[KT][2][KT], bs[KT][2][KT];
#pragma unroll
  for (int ta = 0; ta < KT; ++ta)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int tb = 0; tb < KT; ++tb) {
        const int e = (8 * ta + 4 * ks + q) * K + 8 * tb + g;
        bm[ta][ks][tb] = -sc[kM1 + e];
        bs[ta][ks][tb] = -S[e];
      }
  // B fragments of -MR of the previous iteration (zero after tcg_init and after a batch's last
  // pass C, which left r projected)
  double bp[KT][2][KT];
#pragma unroll
  for (int ta = 0; ta < KT; ++ta)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int tb = 0; tb < KT; ++tb) bp[ta][ks][tb] = -sc[kMR + (8 * ta + 4 * ks + q) * K + 8 * tb + g];
  const double ce = sc[kCEta], cr = sc[kCR];
  double mr[KT][KT][2], zz = 0.0;
#pragma unroll
  for (int i = 0; i < KT; ++i)
#pragma unroll
    for (int j = 0; j < KT; ++j) mr[i][j][0] = mr[i][j][1] = 0.0;
  double* tl = tile[warp];
  const int64_t blocks = (n + 7) / 8;
  const int64_t tw = (int64_t)gridDim.x * kTcgWarps, wid = (int64_t)blockIdx.x * kTcgWarps + warp;
  const int64_t b0 = blocks * wid / tw, b1 = blocks * (wid + 1) / tw;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t row = 8 * b + g;
    const bool ok = row < n;
    double au[KT][2], ad[KT][2];
#pragma unroll
    for (int ta = 0; ta < KT; ++ta)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int64_t o = row * K + 8 * ta + 4 * ks + q;
        au[ta][ks] = ok ? __ldg(U + o) : 0.0;
        ad[ta][ks] = ok ? __ldg(D + o) : 0.0;
      }
    double hd[KT][2];
    double2 d2[KT], e2[KT], h2[KT], r2[KT];
#pragma unroll
    for (int tb = 0; tb < KT; ++tb) {
      const int64_t o = row * K + 8 * tb + 2 * q;
      const double2 z = make_double2(0.0, 0.0);
      const double2 x = ok ? __ldg(reinterpret_cast<const double2*>(EH + o)) : z;
      hd[tb][0] = x.x;
      hd[tb][1] = x.y;
      d2[tb] = ok ? __ldg(reinterpret_cast<const double2*>(D + o)) : z;
      e2[tb] = ok ? *reinterpret_cast<const double2*>(eta + o) : z;
      h2[tb] = (HETA && ok) ? *reinterpret_cast<const double2*>(Heta + o) : z;
      r2[tb] = ok ? *reinterpret_cast<const double2*>(r + o) : z;
    }
#pragma unroll
    for (int tb = 0; tb < KT; ++tb)
#pragma unroll
      for (int ta = 0; ta < KT; ++ta)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          dmma884(hd[tb][0], hd[tb][1], au[ta][ks], bm[ta][ks][tb]);
          dmma884(hd[tb][0], hd[tb][1], ad[ta][ks], bs[ta][ks][tb]);
          dmma884(r2[tb].x, r2[tb].y, au[ta][ks], bp[ta][ks][tb]);  // r - U MR (deferred pass C)
        }
#pragma unroll
    for (int tb = 0; tb < KT; ++tb) {
      e2[tb].x = fma(ce, d2[tb].x, e2[tb].x);
      e2[tb].y = fma(ce, d2[tb].y, e2[tb].y);
      h2[tb].x = fma(ce, hd[tb][0], h2[tb].x);
      h2[tb].y = fma(ce, hd[tb][1], h2[tb].y);
      r2[tb].x = fma(cr, hd[tb][0], r2[tb].x);
      r2[tb].y = fma(cr, hd[tb][1], r2[tb].y);
      zz = fma(r2[tb].x, r2[tb].x, zz);
      zz = fma(r2[tb].y, r2[tb].y, zz);
      *reinterpret_cast<double2*>(tl + g * K + 8 * tb + 2 * q) = r2[tb];
      if (ok) {
        const int64_t o = row * K + 8 * tb + 2 * q;
        *reinterpret_cast<double2*>(eta + o) = e2[tb];
        if constexpr (HETA) *reinterpret_cast<double2*>(Heta + o) = h2[tb];
        *reinterpret_cast<double2*>(r + o) = r2[tb];
      }
    }
    __syncwarp();
    // MR += U^T r over the block's 8 rows: A = U (row 4 ks + q, column 8 t + g), B = r likewise
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int64_t rr = 8 * b + 4 * ks + q;
      double bu[KT], br[KT];
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        bu[t] = rr < n ? __ldg(U + rr * K + 8 * t + g) : 0.0;
        br[t] = tl[(4 * ks + q) * K + 8 * t + g];
      }
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j) dmma884(mr[i][j][0], mr[i][j][1], bu[i], br[j]);
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) zz += __shfl_xor_sync(0xffffffffu, zz, o);
  __syncthreads();
  for (int w = 0; w < kTcgWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int i = 0; i < KT; ++i)
#pragma unroll
        for (int j = 0; j < KT; ++j)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) red[(8 * i + g) * K + 8 * j + 2 * q + hh] += mr[i][j][hh];
      if (lane == 0) red[KK] += zz;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < E; e += kTcgThreads) part[(int64_t)e * gridDim.x + blockIdx.x] = red[e];
}

// pass C over 8-row blocks: d <- ca (r - U MR) + cb d; r <- r - U MR stored only when WRITE_R
#ifndef PLP_TCG_MINB_C
#define PLP_TCG_MINB_C 5
#endif
template <int KT, bool WRITE_R>
__global__ void __launch_bounds__(kTcgThreads, KT == 1 ? PLP_TCG_MINB_C : 1) tcg_finish_kernel(int64_t n, const double* __restrict__ U,
                                                                 const double* __restrict__ sc,
                                                                 double* __restrict__ r,
                                                                 double* __restrict__ D) {
  constexpr int K = 8 * KT;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  double bm[KT][2][KT];
#pragma unroll
  for (int ta = 0; ta < KT; ++ta)
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int tb = 0; tb < KT; ++tb) bm[ta][ks][tb] = -sc[kMR + (8 * ta + 4 * ks + q) * K + 8 * tb + g];
  const double ca = sc[kCA], cb = sc[kCB];
  const int64_t blocks = (n + 7) / 8;
  const int64_t tw = (int64_t)gridDim.x * kTcgWarps, wid = (int64_t)blockIdx.x * kTcgWarps + warp;
  const int64_t b0 = blocks * wid / tw, b1 = blocks * (wid + 1) / tw;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t row = 8 * b + g;
    const bool ok = row < n;
    double au[KT][2];
#pragma unroll
    for (int ta = 0; ta < KT; ++ta)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) au[ta][ks] = ok ? __ldg(U + row * K + 8 * ta + 4 * ks + q) : 0.0;
    double rv[KT][2];
    double2 d2[KT];
#pragma unroll
    for (int tb = 0; tb < KT; ++tb) {
      const int64_t o = row * K + 8 * tb + 2 * q;
      const double2 z = make_double2(0.0, 0.0);
      const double2 x = ok ? *reinterpret_cast<const double2*>(r + o) : z;
      rv[tb][0] = x.x;
      rv[tb][1] = x.y;
      d2[tb] = ok ? *reinterpret_cast<const double2*>(D + o) : z;
    }
#pragma unroll
    for (int tb = 0; tb < KT; ++tb)
#pragma unroll
      for (int ta = 0; ta < KT; ++ta)
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) dmma884(rv[tb][0], rv[tb][1], au[ta][ks], bm[ta][ks][tb]);
    if (ok) {
#pragma unroll
      for (int tb = 0; tb < KT; ++tb) {
        const int64_t o = row * K + 8 * tb + 2 * q;
        if constexpr (WRITE_R) *reinterpret_cast<double2*>(r + o) = make_double2(rv[tb][0], rv[tb][1]);
        *reinterpret_cast<double2*>(D + o) =
            make_double2(fma(ca, rv[tb][0], cb * d2[tb].x), fma(ca, rv[tb][1], cb * d2[tb].y));
      }
    }
  }
}

// MODE 0 (after pass A): tot = [M1 | M2 | tr(d^T EH) | <d^T d, S>_F]; <d, Hd>, step length.
// MODE 1 (after pass B): tot = [MR | ||r||^2]; ||P r||^2 = ||r||^2 - ||MR||_F^2, convergence,
// conjugation; MR zeroed when the iteration stops (pass C then leaves r as it is).
// Folded k (kr = 1, 2, 4 < K = 8): the n x kr arrays are read as n kr / 8 rows of 8, so every 8 x 8
// Gram holds 8 / kr diagonal kr x kr blocks whose sum is the true Gram (off-diagonal blocks pair
// different nodes and are dropped); the k x k matrices the passes apply (M1, MR, S) are expanded
// block-diagonally.  kr = K: no folding.
__device__ void fold_blocks(const double* t, int K, int kr, double* f) {
  for (int i = threadIdx.x; i < kr * kr; i += blockDim.x) {
    const int a = i / kr, b = i % kr;
    double v = 0.0;
    for (int blk = 0; blk < K / kr; ++blk) v += t[(blk * kr + a) * K + blk * kr + b];
    f[i] = v;
  }
}
__device__ void expand_blocks(const double* f, int K, int kr, double* out) {
  for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
    const int row = e / K, col = e % K;
    out[e] = row / kr == col / kr ? f[(row % kr) * kr + col % kr] : 0.0;
  }
}

// The scalar step on the reduced totals (one CTA of 256 threads): fold / expand, <d, Hd> or
// ||P r||^2, tcg_scalar_a / _b, and the matrix the next pass applies.
template <int K, int MODE>
__device__ void tcg_reduce_tail(double* tot, double* sc, int* st, int max_iters, int kr) {
  constexpr int KK = K * K, E = MODE == 0 ? 2 * KK + 2 : KK + 1;
  __shared__ double t[E];
  __shared__ double f1[KK], f2[KK];
  __shared__ int go;
  for (int i = threadIdx.x; i < E; i += 256) t[i] = __ldcg(tot + i);
  __syncthreads();
  const bool fold = kr < K;
  const int kk = kr * kr;
  if (fold) {  // the true kr x kr Grams
    fold_blocks(t, K, kr, f1);
    if (MODE == 0) fold_blocks(t + KK, K, kr, f2);
  } else {
    for (int i = threadIdx.x; i < KK; i += 256) {
      f1[i] = t[i];
      if (MODE == 0) f2[i] = t[KK + i];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (MODE == 0) {
      double c1 = 0.0;
      for (int i = 0; i < kk; ++i) c1 = fma(f2[i], f1[i], c1);
      sc[kTrDE] = t[2 * KK];
      sc[kDHd] = (t[2 * KK] - c1) - t[2 * KK + 1];
      tcg_scalar_a(sc, st);
    } else {
      double m = 0.0;
      for (int i = 0; i < kk; ++i) m = fma(f1[i], f1[i], m);
      sc[kZraw] = t[KK];
      sc[kZnew] = t[KK] - m;
      go = tcg_scalar_b(sc, st, max_iters) ? 1 : 0;
    }
  }
  __syncthreads();
  // the matrix the next pass applies (M1 for pass B, MR for pass C), block-diagonal when folded
  if (MODE == 1 && !go) {
    for (int i = threadIdx.x; i < KK; i += 256) tot[i] = 0.0;
  } else if (fold) {
    expand_blocks(f1, K, kr, tot);
  }
}

// Multi-rank fused tCG: the scalar step after the totals were all-reduced over the ranks.
template <int K, int MODE>
__global__ void __launch_bounds__(256) tcg_step_kernel(double* tot, double* sc, int* st, int max_iters, int kr) {
  tcg_reduce_tail<K, MODE>(tot, sc, st, max_iters, kr);
}

// defer = 1 (multi-rank): the last CTA only resets the ticket; the caller all-reduces tot and
// launches tcg_step_kernel.
template <int K, int MODE>
__global__ void __launch_bounds__(256) tcg_reduce_kernel(int P, const double* __restrict__ part, double* tot,
                                                         unsigned* counter, double* sc, int* st, int max_iters,
                                                         int kr, int defer = 0) {
  constexpr int KK = K * K, E = MODE == 0 ? 2 * KK + 2 : KK + 1;
  __shared__ double ws[8];
  __shared__ unsigned ticket;
  const int e = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double v = 0.0;
  for (int b = threadIdx.x; b < P; b += 256) v += __ldcg(part + (int64_t)e * P + b);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) ws[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += ws[w];
    tot[e] = s;
    __threadfence();
    ticket = atomicAdd(counter, 1u);
  }
  __syncthreads();
  if (ticket != (unsigned)E - 1) return;
  __threadfence();
  if (threadIdx.x == 0) *counter = 0u;
  if (defer) return;
  tcg_reduce_tail<K, MODE>(tot, sc, st, max_iters, kr);
}

__global__ void tcg_expand_s_kernel(const double* __restrict__ S, int kr, double* __restrict__ out) {
  expand_blocks(S, 8, kr, out);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

static int fused_grid(plp_ctx* ctx, int64_t row_blocks, int E, int per_sm) {  // per_sm: one wave
  int64_t g = (int64_t)ctx->num_sms * per_sm;
  const int64_t cap = ((int64_t)ctx->max_ctas * 4 * PLP_MAX_K) / E;  // partials capacity
  if (g > cap) g = cap;
  const int64_t want = (row_blocks + kTcgWarps * 4 - 1) / (kTcgWarps * 4);  // >= 4 blocks per warp
  if (g > want) g = want;
  return (int)(g < 1 ? 1 : g);
}

template <int KT>
static plp_status fused_iteration(plp_ctx* ctx, int64_t n, const double* U, const double* S, double* eta,
                                  double* Heta, double* r, double* dlt, const double* EH, double* scal,
                                  int* status, int max_iters, int kr, int gram_grid, bool coll, bool last) {
  constexpr int K = 8 * KT, KK = K * K;
  static const int unr_a = env_int("PLP_TCG_UNR_A", 4);
  static const int per_sm_a = env_int("PLP_TCG_GRID_A", unr_a == 4 ? resident_ctas(tcg_gram_a_kernel<KT, 4>, kTcgThreads)
                                                                    : resident_ctas(tcg_gram_a_kernel<KT, 2>, kTcgThreads));
  static const int per_sm_b = env_int("PLP_TCG_GRID_B", resident_ctas(tcg_update_kernel<KT, true>, kTcgThreads));
  static const int per_sm_c = resident_ctas(tcg_finish_kernel<KT, true>, kTcgThreads);
  unsigned* counter = reinterpret_cast<unsigned*>(ctx->flag + 4);
  constexpr int EA = 2 * KK + 2, EB = KK + 1;
  int ga = gram_grid;  // > 0: the edge pass wrote pass A's partials (edge_halo.cuh, GRAM)
  if (ga == 0) {
    ga = fused_grid(ctx, (n + 3) / 4, EA, per_sm_a);
    if (unr_a == 4)
      tcg_gram_a_kernel<KT, 4><<<ga, kTcgThreads, 0, ctx->stream>>>(n, U, EH, dlt, S, ctx->partials);
    else
      tcg_gram_a_kernel<KT, 2><<<ga, kTcgThreads, 0, ctx->stream>>>(n, U, EH, dlt, S, ctx->partials);
    PLP_LAUNCH_CHECK("tcg_gram_a_kernel");
  }
  tcg_reduce_kernel<K, 0><<<EA, 256, 0, ctx->stream>>>(ga, ctx->partials, scal + kTotA, counter, scal, status,
                                                       max_iters, kr, coll ? 1 : 0);
  PLP_LAUNCH_CHECK("tcg_reduce_kernel");
  if (coll) {  // multi-rank: the totals over all ranks, then the scalar step
    plp_status s = comm_allreduce(ctx, scal + kTotA, EA);
    if (s) return s;
    tcg_step_kernel<K, 0><<<1, 256, 0, ctx->stream>>>(scal + kTotA, scal, status, max_iters, kr);
    PLP_LAUNCH_CHECK("tcg_step_kernel");
  }
  const int gb = fused_grid(ctx, (n + 7) / 8, EB, per_sm_b);
  auto upd = Heta ? tcg_update_kernel<KT, true> : tcg_update_kernel<KT, false>;
  upd<<<gb, kTcgThreads, 0, ctx->stream>>>(n, U, EH, dlt, S, scal, eta, Heta, r,
                                                             ctx->partials);
  PLP_LAUNCH_CHECK("tcg_update_kernel");
  tcg_reduce_kernel<K, 1><<<EB, 256, 0, ctx->stream>>>(gb, ctx->partials, scal + kTotB, counter + 1, scal, status,
                                                       max_iters, kr, coll ? 1 : 0);
  PLP_LAUNCH_CHECK("tcg_reduce_kernel");
  if (coll) {
    plp_status s = comm_allreduce(ctx, scal + kTotB, EB);
    if (s) return s;
    tcg_step_kernel<K, 1><<<1, 256, 0, ctx->stream>>>(scal + kTotB, scal, status, max_iters, kr);
    PLP_LAUNCH_CHECK("tcg_step_kernel");
  }
  int64_t gc = (int64_t)ctx->num_sms * per_sm_c;
  const int64_t bc = (n + 7) / 8;
  if (bc < gc * kTcgWarps) gc = std::max<int64_t>(1, (bc + kTcgWarps - 1) / kTcgWarps);
  if (last) {  // r projected for the caller; the next pass B must not apply MR again
    tcg_finish_kernel<KT, true><<<(int)gc, kTcgThreads, 0, ctx->stream>>>(n, U, scal, r, dlt);
    PLP_LAUNCH_CHECK("tcg_finish_kernel");
    PLP_CUDA(cudaMemsetAsync(scal + kMR, 0, sizeof(double) * KK, ctx->stream));
  } else {
    tcg_finish_kernel<KT, false><<<(int)gc, kTcgThreads, 0, ctx->stream>>>(n, U, scal, r, dlt);
    PLP_LAUNCH_CHECK("tcg_finish_kernel");
  }
  return PLP_OK;
}

// y = a x + b y with a, b read from the device (the host axpby's formula: fma(a, x, b * y))
__global__ void axpby_dev_kernel(int64_t total, const double* __restrict__ a, const double* __restrict__ x,
                                 const double* __restrict__ b, double* __restrict__ y) {
  const double av = *a, bv = b ? *b : 1.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(av, x[i], bv * y[i]);
}

static int axpby_grid(plp_ctx* ctx, int64_t total) {
  int64_t g = (total + 1023) / 1024;
  if (g > ctx->max_ctas) g = ctx->max_ctas;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace plp

using namespace plp;

extern "C" plp_status plp_tcg_init(plp_ctx* ctx, int64_t n, int k, const double* grad, double delta,
                                   double kappa, double theta, double* eta, double* Heta, double* r,
                                   double* dlt, double* scal, int* status) {
  PLP_NVTX("plp_tcg_init");
  if (!ctx || !grad || !eta || !r || !dlt || !scal || !status || n < 0)
    return set_error(PLP_ERR_ARG, "null argument");
  plp_status st = check_k(k);
  if (st) return st;
  if (!(delta > 0.0)) return set_error(PLP_ERR_DOMAIN, "trust radius must be positive");
  const size_t bytes = sizeof(double) * (size_t)n * k;
  PLP_CUDA(cudaMemcpyAsync(r, grad, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  PLP_CUDA(cudaMemsetAsync(eta, 0, bytes, ctx->stream));
  if (Heta) PLP_CUDA(cudaMemsetAsync(Heta, 0, bytes, ctx->stream));
  PLP_CUDA(cudaMemsetAsync(dlt, 0, bytes, ctx->stream));
  if ((st = plp_axpby(ctx, n, k, -1.0, r, 0.0, dlt))) return st;  // delta = -r
  if ((st = plp_dot(ctx, n, k, r, r, scal + kZr))) return st;
  PLP_CUDA(cudaMemsetAsync(scal + kMR, 0, sizeof(double) * PLP_MAX_K * PLP_MAX_K, ctx->stream));  // no MR to defer
  tcg_init_kernel<<<1, 1, 0, ctx->stream>>>(scal, status, delta, kappa, theta);
  PLP_LAUNCH_CHECK("tcg_init_kernel");
  return PLP_OK;
}

extern "C" plp_status plp_tcg_run(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                  const double* AB, const double* G_in, const double* S, double p,
                                  double eps, int mode, double* eta, double* Heta, double* r,
                                  double* dlt, double* Hd, double* scal, int* status, int max_iters,
                                  int iters, int fused) {
  PLP_NVTX("plp_tcg_run");
  if (!ctx || !g || !U || !AB || !S || !eta || !r || !dlt || !Hd || !scal || !status)
    return set_error(PLP_ERR_ARG, "null argument");
  if (iters < 0 || max_iters < 1) return set_error(PLP_ERR_ARG, "iters >= 0, max_iters >= 1");
  const int64_t n = g->n_rows;
  const int64_t total = n * k;
  const bool foldable = (k == 1 || k == 2 || k == 4) && (n * k) % 8 == 0;
  if (fused && k != 8 && k != 16 && !foldable)
    return set_error(PLP_ERR_ARG, "fused tCG needs k = 8 or 16, or k = 1, 2, 4 with n k divisible by 8");
  auto al16 = [](const void* x) { return ((uintptr_t)x & 15u) == 0; };
  if (!fused && !Heta) return set_error(PLP_ERR_ARG, "Heta may be NULL only with fused = 1");
  if (fused && !(al16(U) && al16(eta) && (!Heta || al16(Heta)) && al16(r) && al16(dlt) && al16(Hd)))
    return set_error(PLP_ERR_ARG, "fused tCG needs 16-byte aligned vectors");
  // multi-rank graph: the fused passes run on the owned rows, their k x k / scalar totals are
  // all-reduced before each scalar step (tcg_step_kernel), the direction's halo is exchanged by
  // the collective Hessian-vector product
  const bool coll = ctx->comm && g->dist;
  // on a multi-rank graph U's halo rows are current (the plp_fgrad at this iterate exchanged them):
  // each Hessian-vector product exchanges only the direction's halo
  if (ctx->comm && g->dist) mode |= PLP_U_HALO_CURRENT;
  const int grid = axpby_grid(ctx, total);
  plp_status st;
  if (fused) {
    if (k < 8) {
      tcg_expand_s_kernel<<<1, 64, 0, ctx->stream>>>(S, k, scal + kSx);
      PLP_LAUNCH_CHECK("tcg_expand_s_kernel");
    }
    // pass A folded into the Hessian-vector-only halo pass where it applies (k = 4, 8, sparse
    // mode, rank-local; PLP_TCG_GRAM_EDGE=0 keeps the separate pass for comparison)
    static const bool gram_edge = env_int("PLP_TCG_GRAM_EDGE", 1) != 0;
    const bool try_gram = gram_edge && (k == 8 || k == 4) && mode == PLP_HESS_SPARSE && !coll;
    const double* S8 = k == 8 ? S : scal + kSx;
    for (int it = 0; it < iters; ++it) {
      const bool last = it == iters - 1;
      int gram_grid = 0;
      if (try_gram) {
        bool used = false;
        int eg = 0;
        if ((st = hessvec_gram(ctx, g, k, U, dlt, p, AB, eps, S8, Hd, &eg, &used))) return st;
        gram_grid = used ? eg : 0;
      } else if ((st = plp_hessvec(ctx, g, k, U, dlt, p, AB, mode, eps, G_in, Hd))) {
        return st;
      }
      if (k == 16)
        st = fused_iteration<2>(ctx, n, U, S, eta, Heta, r, dlt, Hd, scal, status, max_iters, 16, 0, coll, last);
      else if (k == 8)
        st = fused_iteration<1>(ctx, n, U, S, eta, Heta, r, dlt, Hd, scal, status, max_iters, 8, gram_grid, coll, last);
      else  // k = 1, 2, 4: the n x k arrays as n k / 8 rows of 8, S block-diagonal
        st = fused_iteration<1>(ctx, n * k / 8, U, scal + kSx, eta, Heta, r, dlt, Hd, scal, status, max_iters, k,
                                gram_grid, coll, last);
      if (st) return st;
    }
    return PLP_OK;
  }
  for (int it = 0; it < iters; ++it) {
    // H(delta) = P(EucHess[delta]) - delta S
    if ((st = plp_hessvec(ctx, g, k, U, dlt, p, AB, mode, eps, G_in, Hd))) return st;
    if ((st = plp_project(ctx, n, k, U, Hd, Hd))) return st;
    if ((st = plp_apply_sub(ctx, n, k, dlt, S, Hd, Hd))) return st;
    if ((st = plp_dot(ctx, n, k, dlt, Hd, scal + kDHd))) return st;
    tcg_scalar_a_kernel<<<1, 1, 0, ctx->stream>>>(scal, status);
    PLP_LAUNCH_CHECK("tcg_scalar_a_kernel");
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCEta, dlt, nullptr, eta);
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCEta, Hd, nullptr, Heta);
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCR, Hd, nullptr, r);
    PLP_LAUNCH_CHECK("axpby_dev_kernel");
    if ((st = plp_project(ctx, n, k, U, r, r))) return st;  // keep the residual horizontal
    if ((st = plp_dot(ctx, n, k, r, r, scal + kZnew))) return st;
    tcg_scalar_b_kernel<<<1, 1, 0, ctx->stream>>>(scal, status, max_iters);
    PLP_LAUNCH_CHECK("tcg_scalar_b_kernel");
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCA, r, scal + kCB, dlt);
    PLP_LAUNCH_CHECK("axpby_dev_kernel");
  }
  return PLP_OK;
}

// ---------------------------------------------------------------------------------------------
// CUDA-graph capture of a batch of tCG iterations (SURVEY.md §8(f) NEXT-1 "CUDA-Graph the tCG
// iteration"): one graph launch replaces ~10 kernel launches per iteration.
// ---------------------------------------------------------------------------------------------
struct plp_tcg_graph {
  plp_ctx* ctx = nullptr;
  cudaGraphExec_t exec = nullptr;
  int nodes = 0;
};

extern "C" plp_status plp_tcg_graph_create(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                           const double* AB, const double* G_in, const double* S, double p,
                                           double eps, int mode, double* eta, double* Heta, double* r,
                                           double* dlt, double* Hd, double* scal, int* status, int max_iters,
                                           int iters, int fused, plp_tcg_graph** out) {
  PLP_NVTX("plp_tcg_graph_create");
  if (!ctx || !out) return set_error(PLP_ERR_ARG, "null argument");
  *out = nullptr;
  if (ctx->stream == nullptr || ctx->stream == cudaStreamLegacy || ctx->stream == cudaStreamPerThread)
    return set_error(PLP_ERR_ARG, "graph capture needs a created (non-default) stream on the context");
  if (iters < 1) return set_error(PLP_ERR_ARG, "iters >= 1");
  PLP_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
  const plp_status st = plp_tcg_run(ctx, g, k, U, AB, G_in, S, p, eps, mode, eta, Heta, r, dlt, Hd, scal, status,
                                    max_iters, iters, fused);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
  if (st != PLP_OK || e != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    return st != PLP_OK ? st : cuda_check(e, "cudaStreamEndCapture");
  }
  size_t nodes = 0;
  cudaGraphGetNodes(graph, nullptr, &nodes);
  cudaGraphExec_t exec = nullptr;
  const cudaError_t e2 = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e2 != cudaSuccess) return cuda_check(e2, "cudaGraphInstantiate");
  plp_tcg_graph* gr = new (std::nothrow) plp_tcg_graph();
  if (!gr) {
    cudaGraphExecDestroy(exec);
    return set_error(PLP_ERR_OOM, "host allocation failed");
  }
  gr->ctx = ctx;
  gr->exec = exec;
  gr->nodes = (int)nodes;
  *out = gr;
  return PLP_OK;
}

extern "C" plp_status plp_tcg_graph_launch(plp_tcg_graph* gr) {
  PLP_NVTX("plp_tcg_graph_launch");
  if (!gr) return set_error(PLP_ERR_ARG, "graph is null");
  PLP_CUDA(cudaGraphLaunch(gr->exec, gr->ctx->stream));
  return PLP_OK;
}

extern "C" plp_status plp_tcg_graph_nodes(const plp_tcg_graph* gr, int* nodes) {
  if (!gr || !nodes) return set_error(PLP_ERR_ARG, "null argument");
  *nodes = gr->nodes;
  return PLP_OK;
}

extern "C" plp_status plp_tcg_graph_destroy(plp_tcg_graph* gr) {
  if (!gr) return PLP_OK;
  cudaGraphExecDestroy(gr->exec);
  delete gr;
  return PLP_OK;
}
