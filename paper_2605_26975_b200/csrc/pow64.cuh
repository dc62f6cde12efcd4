// fp64 power kernels for the edge pass: s = cap(a)^{p-2} and t = a^{p-1} for a = |u_i - u_j|
// (readings #6 and #8 of DESIGN.md §3).  One power per edge-column is shared by F (a^p = t a),
// the gradient (phi_p = copysign(t, d)) and the Hessian weight (s) -- SURVEY.md §8(a) a7.
//
// libdevice pow costs ~120 fp64-pipe slots per call on B200 (measured 134 G pow/s), which would
// make the edge pass fp64-ALU bound many times over the HBM roofline.  Cheaper policies, each
// accurate to a few ulp (tests/test_gpu_parity.py::test_power_policies_accuracy):
//   PowP2          p == 2:            s = 1, t = a                         (no power at all)
//   PowRoot<D, M>  p - 2 == -M/D:     x = 2^(D q) x', x' in [1, 2^D) by integer exponent
//                                     arithmetic; y = x'^{-1/D} from an fp32 MUFU seed and one
//                                     cubic-corrected Newton step (error O(e^3) ~ 1e-18);
//                                     s = y^M 2^{-qM}  (7 + log2-chain fp64 ops)
//   PowGeneric     any p in (1, 2]:   table-driven log2 (128 entries) + exp2 (64 entries),
//                                     degree-5 polynomials, ~19 fp64 ops
// Every policy computes s = pow_q(max(a, eps)) and t = s * a; for the rare a < eps the exact
// t = a^{p-1} is recomputed with libdevice (t = 0 at a = 0), so F and the gradient never see the
// cap.  The max and the a < eps test run on the integer pipe: for non-negative doubles the bit
// patterns order like the values.  Domain: eps and every a are normal doubles below 2^1000
// (|U| entries < 1e150); eps >= 1e-300 is enforced by check_p.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace plp {

struct PowTables {
  double2 logt[128];  // (1/c_j rounded, -log2(that value)) with c_j = 1 + (j + 0.5)/128
  double expt[64];    // 2^(j/64)
};

// ---- bit helpers (integer pipe only) ------------------------------------------------------------
// positive normal double in [2^-126, 2^127] -> float, mantissa truncated to 20 bits
__device__ __forceinline__ float d2f_trunc(double x) {
  const unsigned hi = (unsigned)__double2hiint(x);
  return __uint_as_float((hi - (896u << 20)) << 3);
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

template <int E>
__device__ __forceinline__ double ipow(double y) {
  if constexpr (E == 0) return 1.0;
  else if constexpr (E == 1) return y;
  else if constexpr (E % 2 == 0) { const double h = ipow<E / 2>(y); return h * h; }
  else return ipow<E - 1>(y) * y;
}

// ---- policies -------------------------------------------------------------------------------
struct PowBase {
  double eps;         // curvature cap (> 0 when p < 2)
  long long eps_bits; // bit pattern of eps (integer compare == value compare for >= 0)
  double pm1;         // p - 1 (rare branch)
  __device__ __forceinline__ void init_smem(void*) {}
};

struct PowP2 : PowBase {
  static constexpr bool kNeedsTables = false;
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    s = 1.0;
    t = a;
  }
};

template <class Derived>
struct PowCapped : PowBase {
  __device__ __forceinline__ void eval(double a, double& s, double& t) const {
    const long long ab = __double_as_longlong(a);
    const bool small = ab < eps_bits;  // a < eps  (a >= 0)
    const double ac = __longlong_as_double(small ? eps_bits : ab);
    s = static_cast<const Derived*>(this)->pow_q(ac);
    t = s * a;
    if (small) t = (ab != 0) ? pow(a, pm1) : 0.0;  // rare: exact a^{p-1} below the cap
  }
};

template <int D, int M>
struct PowRoot : PowCapped<PowRoot<D, M>> {
  static constexpr bool kNeedsTables = false;
  // x^{-M/D} for a positive normal x
  __device__ __forceinline__ double pow_q(double x) const {
    const int hi = __double2hiint(x);
    const int ex = ((hi >> 20) & 0x7FF) - 1023;
    constexpr int OFF = 1100;  // divisible by D in {2, 5, 10}: floor division of ex by D
    const int qd = (int)((unsigned)(ex + OFF) / (unsigned)D) - OFF / D;
    const int r = ex - qd * D;  // 0 <= r < D
    const double xs = __hiloint2double((hi & 0x000FFFFF) | ((1023 + r) << 20), __double2loint(x));
    const float xf = d2f_trunc(xs);  // xs in [1, 2^D)
    float yf;
    if constexpr (D == 2) yf = rsqrt_approx(xf);
    else yf = ex2_approx(lg2_approx(xf) * (-1.0f / (float)D));
    const double y0 = f2d_exact(yf);
    const double e = fma(-xs, ipow<D>(y0), 1.0);  // 1 - xs y0^D  (|e| ~ 1e-6)
    constexpr double C1 = 1.0 / D, C2 = (D + 1.0) / (2.0 * D * D);
    const double c = fma(e, C2, C1);
    const double y = fma(y0 * e, c, y0);  // xs^{-1/D} to O(e^3)
    return scale_pow2(ipow<M>(y), -qd * M);
  }
};

struct PowGeneric : PowCapped<PowGeneric> {
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
