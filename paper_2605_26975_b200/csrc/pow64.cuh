// fp64 power kernels for the edge pass: s = cap(a)^{p-2} and t = a^{p-1} for a = |u_i - u_j|
// (readings #6 and #8 of DESIGN.md §3).  One power per edge-column is shared by F (a^p = t a),
// the gradient (phi_p = copysign(t, d)) and the Hessian weight (s) -- SURVEY.md §8(a) a7.
//
// libdevice pow costs ~120 fp64-pipe slots per call on B200 (measured 134 G pow/s), which would
// make the edge pass fp64-ALU bound several times over the HBM roofline.  Three cheaper exact-
// to-rounding policies (DESIGN.md §5 "power"):
//   PowP2       p == 2:              s = 1, t = a                       (no power at all)
//   PowRoot<D>  p - 2 == -m/D:       y = x^{-1/D} from an fp32 MUFU seed + one cubic-corrected
//                                    Newton step (error O(e^3) ~ 1e-18), s = y^m
//   PowGeneric  any p in (1, 2]:     table-driven log2 (128 entries) + exp2 (64 entries),
//                                    degree-5 polynomials; max rel. error ~2e-15 (tested)
// Every policy computes s = pow_q(max(a, eps)), t = s * a; for the rare a < eps the exact
// t = a^{p-1} is recomputed with libdevice (t = 0 at a = 0), so F and the gradient never see the
// cap.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace plp {

struct PowTables {
  double2 logt[128];  // (1/c_j rounded, -log2(that value)) with c_j = 1 + (j + 0.5)/128
  double expt[64];    // 2^(j/64)
};

// ---- bit helpers (integer pipe only) ------------------------------------------------------------
// positive normal double (within float range) -> float, mantissa truncated to 20 bits
__device__ __forceinline__ float d2f_trunc(double x) {
  const unsigned hi = (unsigned)__double2hiint(x);
  return __uint_as_float((hi - (896u << 20)) << 3);
}
// positive normal float -> double (exact)
__device__ __forceinline__ double f2d_exact(float f) {
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((int)((b >> 3) + (896u << 20)), (int)(b << 29));
}
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int E>
__device__ __forceinline__ double ipow(double y) {
  if constexpr (E == 0) return 1.0;
  else if constexpr (E == 1) return y;
  else if constexpr (E % 2 == 0) { const double h = ipow<E / 2>(y); return h * h; }
  else return ipow<E - 1>(y) * y;
}

// runtime exponent 1 <= m < 16 by square-and-multiply (m is warp-uniform)
__device__ __forceinline__ double ipow_rt(double y, int m) {
  double r = (m & 1) ? y : 1.0;
  double b = y;
  m >>= 1;
  while (m) {
    b = b * b;
    if (m & 1) r = r * b;
    m >>= 1;
  }
  return r;
}

// ---- policies -------------------------------------------------------------------------------
struct PowBase {
  double eps;   // curvature cap (> 0 when p < 2)
  double pm1;   // p - 1 (rare branch)
  __device__ __forceinline__ void init_smem(void*) {}
};

struct PowP2 : PowBase {
  static constexpr bool kNeedsTables = false;
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    s = 1.0;
    t = a;
  }
};

template <int D>
struct PowRoot : PowBase {
  static constexpr bool kNeedsTables = false;
  int m;  // p - 2 = -m / D
  __device__ __forceinline__ double seed(double x) const {
    const float xf = d2f_trunc(x);
    float yf;
    if constexpr (D == 2) yf = rsqrt_approx(xf);
    else yf = ex2_approx(lg2_approx(xf) * (-1.0f / (float)D));
    return f2d_exact(yf);
  }
  // x^{-m/D} for x in [2^-100, 2^100]
  __device__ __forceinline__ double pow_q(double x) const {
    if (!(x > 7.888609052210118e-31 && x < 1.2676506002282294e30)) return pow(x, -(double)m / D);
    const double y0 = seed(x);
    const double e = fma(-x, ipow<D>(y0), 1.0);  // 1 - x y0^D  (|e| ~ 1e-6)
    constexpr double C1 = 1.0 / D, C2 = (D + 1.0) / (2.0 * D * D);
    const double c = fma(e, C2, C1);
    const double y = fma(y0 * e, c, y0);         // y0 (1 - e)^{-1/D} to O(e^3)
    return ipow_rt(y, m);
  }
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    const double ac = fmax(a, eps);
    s = pow_q(ac);
    t = s * a;
    if (a < eps) t = (a > 0.0) ? pow(a, pm1) : 0.0;
  }
};

struct PowGeneric : PowBase {
  static constexpr bool kNeedsTables = true;
  double q;    // p - 2
  double q64;  // 64 (p - 2)
  const PowTables* gtab;  // global copy
  const PowTables* tab;   // shared-memory copy (set by init_smem)
  __device__ __forceinline__ void init_smem(void* smem) {
    PowTables* st = reinterpret_cast<PowTables*>(smem);
    const double* src = reinterpret_cast<const double*>(gtab);
    double* dst = reinterpret_cast<double*>(st);
    for (int i = threadIdx.x; i < (int)(sizeof(PowTables) / 8); i += blockDim.x) dst[i] = src[i];
    tab = st;
  }
  __device__ __forceinline__ double pow_q(double x) const {
    if (!(x > 1.0e-300 && x < 1.0e300)) return pow(x, q);
    const int hi = __double2hiint(x);
    const int lo = __double2loint(x);
    const int ex = (hi >> 20) - 1023;
    const int j = (hi >> 13) & 127;
    const double m = __hiloint2double((hi & 0x000FFFFF) | 0x3FF00000, lo);  // [1, 2)
    const double2 tj = tab->logt[j];
    const double r = fma(m, tj.x, -1.0);  // |r| <= ~2^-8
    // log2(1 + r) = r * P(r),  P = log2(e) * (1 - r/2 + r^2/3 - r^3/4 + r^4/5 - r^5/6)
    constexpr double L0 = 1.4426950408889634, L1 = -0.7213475204444817,
                     L2 = 0.4808983469629878, L3 = -0.36067376022224085,
                     L4 = 0.28853900817779266, L5 = -0.2404491734814939;
    double P = fma(L5, r, L4);
    P = fma(P, r, L3);
    P = fma(P, r, L2);
    P = fma(P, r, L1);
    P = fma(P, r, L0);
    // (double)ex via the 2^52 + 2^31 magic (one DADD, no I2F)
    const double exd = __hiloint2double(0x43300000, ex ^ 0x80000000) - 4503601774854144.0;
    const double lg = fma(r, P, exd + tj.y);  // log2(x)
    // exp2(q * lg) with 64-entry table
    const double y64 = lg * q64;
    const double kd = y64 + 6755399441055744.0;  // 0x1.8p52: round to integer
    const int n = __double2loint(kd);
    const double rr = y64 - (kd - 6755399441055744.0);  // |rr| <= 0.5, exact
    // 2^(rr/64) = sum_k (rr ln2/64)^k / k!, degree 5
    constexpr double E1 = 0.010830424696249145, E2 = 5.86490495505617e-05,
                     E3 = 2.1173137155464776e-07, E4 = 5.732851688640402e-10,
                     E5 = 1.2417843701716925e-12;
    double Q = fma(E5, rr, E4);
    Q = fma(Q, rr, E3);
    Q = fma(Q, rr, E2);
    Q = fma(Q, rr, E1);
    Q = fma(Q, rr, 1.0);
    const double v = tab->expt[n & 63] * Q;
    return __hiloint2double(__double2hiint(v) + ((n >> 6) << 20), __double2loint(v));
  }
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    const double ac = fmax(a, eps);
    s = pow_q(ac);
    t = s * a;
    if (a < eps) t = (a > 0.0) ? pow(a, pm1) : 0.0;
  }
};

// Exact-series check of the constants above is in tests/test_gpu_pow.py (max rel. error vs
// libdevice pow over 2^20 random arguments).

}  // namespace plp
