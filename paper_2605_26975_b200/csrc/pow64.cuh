// fp64 power kernels for the edge pass (readings #6 and #8 of DESIGN.md §3).
//
// Per stored edge-column the fused pass needs ONE power, s_raw = |d|^{p-2} with d = u_i - u_j:
//   (Delta_p u)_i += w s_raw d            (= w phi_p(d) = w |d|^{p-1} sign(d); 0 at d = 0)
//   (H eta)_i     += w s_cap (eta_i - eta_j),   s_cap = cap(|d|)^{p-2} = (|d| < eps ? eps^{p-2} : s_raw)
// so F (through <u, Delta_p u> = A), the gradient and the Hessian share it.
//
// libdevice pow costs ~120 fp64-pipe slots per call on B200 (measured 134 G pow/s): many times
// the HBM roofline.  Cheaper policies, each accurate to a few ulp
// (tests/test_gpu_parity.py::test_power_policies_accuracy):
//   PowP2          p == 2:          s = 1                                (no power at all)
//   PowRoot<D, M>  p - 2 == -M/D:   y0 = x^{-1/D} from an fp32 MUFU seed, e = 1 - x y0^D, then
//                                   x^{-M/D} = y0^M (1 + c1 e + c2 e^2) + O(e^3): a second-order
//                                   expansion of the exact correction (|e| ~ 1e-6 so the error is
//                                   ~1e-18); 7 fp64 ops at p = 1.2 (D = 5, M = 4)
//   PowGeneric     any p in (1, 2]: table-driven log2 (128 entries) + exp2 (64 entries),
//                                   degree-5 polynomials, ~19 fp64 ops
// The edge form is branch-free on the fast domain {0} U [2^-120, 2^120): exact zeros (ties) give
// a finite s_raw that multiplies d = 0.  Anything else sets a flag and the row is recomputed with
// libdevice (edge_kernel.cuh), so every input follows the definitions.  The cap test runs on the
// integer pipe: for non-negative doubles the bit patterns order like the values.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace plp {

struct PowTables {
  double2 logt[128];  // (1/c_j rounded, -log2(that value)) with c_j = 1 + (j + 0.5)/128
  double expt[64];    // 2^(j/64)
};

constexpr unsigned kHiMin = (1023u - 120u) << 20;  // hi word of 2^-120
constexpr unsigned kHiMax = (1023u + 120u) << 20;  // hi word of 2^120

// ---- bit helpers (integer pipe only) ------------------------------------------------------------
__device__ __forceinline__ unsigned abs_hi(double d) {
  return (unsigned)__double2hiint(d) & 0x7FFFFFFFu;
}
// 1 if |d| is outside the fast domain {0} U [2^-120, 2^120) (|d| < 2^-1022 with a zero high word
// counts as 0)
__device__ __forceinline__ unsigned out_of_domain(unsigned ahi) {
  return (unsigned)(ahi - 1u < kHiMin - 1u) | (unsigned)(ahi >= kHiMax);
}
// float with the exponent and top 20 mantissa bits of the double whose |hi word| is `ahi`
// (ahi clamped to >= 2^-120 so the float is normal)
__device__ __forceinline__ float seed_float(unsigned ahi) {
  const unsigned h = ahi > kHiMin ? ahi : kHiMin;
  return __uint_as_float((h - (896u << 20)) << 3);
}
// positive normal float -> double (exact)
__device__ __forceinline__ double f2d_exact(float f) {
  const unsigned b = __float_as_uint(f);
  return __hiloint2double((int)((b >> 3) + (896u << 20)), (int)(b << 29));
}
__device__ __forceinline__ double scale_pow2(double v, int e) {  // v * 2^e, result normal
  return __hiloint2double(__double2hiint(v) + (e << 20), __double2loint(v));
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

// ---- policies -------------------------------------------------------------------------------
struct PowBase {
  double eps;          // curvature cap (> 0 when p < 2)
  long long eps_bits;  // bit pattern of eps (integer compare == value compare for >= 0)
  long long fast_lo;   // bit pattern of max(eps, 2^-120): |d| >= this (and < 2^120) is "fast"
  unsigned fast_lo2;   // (hi(fast_lo) + 1) << 1: the conservative hi-word form used by fast_hi
  unsigned fast_span2; // (kHiMax - (hi(fast_lo) + 1)) << 1
  double q;            // p - 2
  double pm1;          // p - 1
  double s_eps;        // eps^{p-2} (host glibc pow: the value the oracle's cap gives)
  double c1, c2;       // expansion coefficients of PowRoot (kernel parameters, not immediates)
  __device__ __forceinline__ void init_smem(void*) {}
  __device__ __forceinline__ bool below_cap(double a) const {  // a >= 0
    return __double_as_longlong(a) < eps_bits;
  }
  // |d| in [max(eps, 2^-120), 2^120): no cap and the branch-free power is valid (integer pipe)
  __device__ __forceinline__ bool fast(double d) const {
    const unsigned ahi = abs_hi(d);
    const unsigned long long a = ((unsigned long long)ahi << 32) | (unsigned)__double2loint(d);
    return (a >= (unsigned long long)fast_lo) & (ahi < kHiMax);
  }
  // Conservative two-instruction form of fast(): true only if |d| is in the fast domain (a |d|
  // sharing its high word with the lower bound counts as not fast and takes the exact path).
  __device__ __forceinline__ bool fast_hi(double d) const {
    const unsigned h2 = (unsigned)__double2hiint(d) << 1;  // drops the sign bit
    return h2 - fast_lo2 < fast_span2;
  }
  __device__ __forceinline__ bool abs_below_cap(double d) const {  // |d| < eps, integer pipe
    // compare (|hi|, lo) with eps's words; written on the words so the compiler cannot turn the
    // sign mask into an fp64 |d| (a DADD on the fp64 pipe)
    const unsigned long long a =
        ((unsigned long long)abs_hi(d) << 32) | (unsigned)__double2loint(d);
    return a < (unsigned long long)eps_bits;
  }
};

struct PowP2 : PowBase {
  static constexpr const char* kName = "P2";
  static constexpr bool kNeedsTables = false;
  static constexpr bool kIsP2 = true;
  __device__ __forceinline__ double pow_raw(double, unsigned&) const { return 1.0; }
  // node form: s = cap(a)^0 = 1, t = a^1
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    s = 1.0;
    t = a;
  }
};

// node form shared by the capped policies: s = cap(a)^{p-2}, t = a^{p-1} (a >= 0), with the
// exact libdevice results below the cap and outside the fast domain (rare, divergent).
template <class Derived>
struct PowCapped : PowBase {
  static constexpr bool kIsP2 = false;
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    unsigned bad = 0;
    s = static_cast<const Derived*>(this)->pow_raw(a, bad);
    t = s * a;
    if (bad | (unsigned)below_cap(a)) {
      if (below_cap(a)) {
        s = s_eps;
        t = (a != 0.0) ? pow(a, pm1) : 0.0;
      } else {
        s = pow(a, q);
        t = s * a;
      }
    }
  }
};

// y0^D and y0^M with shared products
template <int D, int M>
__device__ __forceinline__ void root_powers(double y, double& yD, double& yM) {
  const double y2 = y * y;
  if constexpr (D == 2) {
    yD = y2;
    yM = y;  // M = 1
  } else {
    const double y4 = y2 * y2;
    const double y5 = y4 * y;
    if constexpr (D == 5) {
      yD = y5;
      if constexpr (M == 1) yM = y;
      else if constexpr (M == 2) yM = y2;
      else if constexpr (M == 3) yM = y2 * y;
      else yM = y4;
    } else {  // D == 10
      yD = y5 * y5;
      if constexpr (M == 1) yM = y;
      else if constexpr (M == 3) yM = y2 * y;
      else if constexpr (M == 7) yM = y5 * y2;
      else yM = y5 * y4;
    }
  }
}

template <int D, int M>
struct PowRoot : PowCapped<PowRoot<D, M>> {
  static constexpr const char* kName = D == 2 ? "R2M1" : D == 5 ? (M == 1 ? "R5M1" : M == 2 ? "R5M2" : M == 3 ? "R5M3" : "R5M4")
                                     : (M == 1 ? "R10M1" : M == 3 ? "R10M3" : M == 7 ? "R10M7" : "R10M9");
  static constexpr bool kNeedsTables = false;
  // |d|^{-M/D}, valid on the fast domain only (no clamping: callers test fast_hi()); one IMAD
  // turns the high word into the float seed argument (the shift drops the sign bit)
  __device__ __forceinline__ double pow_fast(double d) const {
    const float xf = __uint_as_float(((unsigned)__double2hiint(d) << 3) + 0x40000000u);
    float yf;
    if constexpr (D == 2) yf = rsqrt_approx(xf);
    else yf = ex2_approx(lg2_approx(xf) * (-1.0f / (float)D));
    const double y0 = f2d_exact(yf);  // two integer instructions (F2F measured slower)
    double yD, yM;
    root_powers<D, M>(y0, yD, yM);
    const double e = fma(-fabs(d), yD, 1.0);  // 1 - x y0^D
    const double c = fma(this->c2, e, this->c1);
    return fma(yM * e, c, yM);
  }
  // |d|^{-M/D}; branch-free; sets `bad` outside the fast domain
  __device__ __forceinline__ double pow_raw(double d, unsigned& bad) const {
    const unsigned ahi = abs_hi(d);
    bad |= out_of_domain(ahi);
    const float xf = seed_float(ahi);
    float yf;
    if constexpr (D == 2) yf = rsqrt_approx(xf);
    else yf = ex2_approx(lg2_approx(xf) * (-1.0f / (float)D));
    const double y0 = f2d_exact(yf);
    double yD, yM;
    root_powers<D, M>(y0, yD, yM);
    const double e = fma(-fabs(d), yD, 1.0);  // 1 - x y0^D
    const double c = fma(this->c2, e, this->c1);
    return fma(yM * e, c, yM);
  }
};

struct PowGeneric : PowCapped<PowGeneric> {
  static constexpr const char* kName = "GEN";
  static constexpr bool kNeedsTables = true;
  double q64;             // 64 (p - 2)
  const PowTables* gtab;  // global copy
  const PowTables* tab;   // shared-memory copy (set by init_smem)
  __device__ __forceinline__ void init_smem(void* smem) {
    PowTables* st = reinterpret_cast<PowTables*>(smem);
    const double* src = reinterpret_cast<const double*>(gtab);
    double* dst = reinterpret_cast<double*>(st);
    for (int i = threadIdx.x; i < (int)(sizeof(PowTables) / 8); i += blockDim.x) dst[i] = src[i];
    tab = st;
  }
  __device__ __forceinline__ double pow_fast(double d) const {
    unsigned unused = 0;
    return pow_raw(d, unused);
  }
  // |d|^{p-2}; branch-free; sets `bad` outside the fast domain
  __device__ __forceinline__ double pow_raw(double d, unsigned& bad) const {
    const unsigned ahi = abs_hi(d);
    bad |= out_of_domain(ahi);
    const int hi = (int)(ahi > kHiMin ? ahi : kHiMin);
    const int lo = __double2loint(d);
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
    const double lg = fma(r, P, exd + tj.y);  // log2|d|
    // exp2(q * lg) with a 64-entry table
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
    return scale_pow2(tab->expt[n & 63] * Q, n >> 6);
  }
};

// the instantiated rational policies (p = 1.5; 1.8, 1.6, 1.4, 1.2; 1.9, 1.7, 1.3, 1.1)
using PowR2M1 = PowRoot<2, 1>;
using PowR5M1 = PowRoot<5, 1>;
using PowR5M2 = PowRoot<5, 2>;
using PowR5M3 = PowRoot<5, 3>;
using PowR5M4 = PowRoot<5, 4>;
using PowR10M1 = PowRoot<10, 1>;
using PowR10M3 = PowRoot<10, 3>;
using PowR10M7 = PowRoot<10, 7>;
using PowR10M9 = PowRoot<10, 9>;

#define PLP_POW_LIST(X)                                                                      \
  X(P2, PowP2) X(R2M1, PowR2M1) X(R5M1, PowR5M1) X(R5M2, PowR5M2) X(R5M3, PowR5M3)           \
  X(R5M4, PowR5M4) X(R10M1, PowR10M1) X(R10M3, PowR10M3) X(R10M7, PowR10M7)                  \
  X(R10M9, PowR10M9) X(GEN, PowGeneric)

}  // namespace plp
