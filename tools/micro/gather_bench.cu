// Gather microbenchmark (standalone, not the product path): how fast can B200 gather the 64-byte
// neighbour rows U_j (and eta_j) of a CSR graph, with no arithmetic?  Isolates the memory side of
// the edge pass.  Built by tools/micro/gather_bench.py, called through ctypes.
#include <cstdint>
#include <cuda_runtime.h>

template <int VB>
struct Vec;
template <>
struct Vec<16> {
  double2 v;
  __device__ __forceinline__ void ld(const double* p) { v = __ldg(reinterpret_cast<const double2*>(p)); }
  __device__ __forceinline__ double sum() const { return v.x + v.y; }
};
template <>
struct Vec<32> {
  double a, b, c, d;
  __device__ __forceinline__ void ld(const double* p) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
  }
  __device__ __forceinline__ double sum() const { return a + b + c + d; }
};

// group of LPR lanes per row, each lane VB bytes of the 64-byte row; UNR edges per batch
template <int LPR, int VB, int UNR, bool ETA, int MINB>
__global__ void __launch_bounds__(256, MINB) gather_kernel(int n, const int* __restrict__ rp,
                                                         const int* __restrict__ col,
                                                         const double* __restrict__ U,
                                                         const double* __restrict__ E, double* out) {
  constexpr int RPW = 32 / LPR;
  const int lane = threadIdx.x & 31, grp = lane / LPR, li = lane % LPR;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x / 32) * RPW;
  const int c0 = li * (VB / 8);
  for (int64_t row = ((int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * RPW + grp; row < n;
       row += groups) {
    const int e0 = rp[row], e1 = rp[row + 1];
    double acc = 0.0;
    for (int e = e0; e < e1; e += UNR) {
      int j[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) j[u] = (e + u < e1) ? __ldg(col + e + u) : -1;
      Vec<VB> a[UNR], b[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (j[u] >= 0) {
          a[u].ld(U + (int64_t)j[u] * 8 + c0);
          if (ETA) b[u].ld(E + (int64_t)j[u] * 8 + c0);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u)
        if (j[u] >= 0) acc += a[u].sum() + (ETA ? b[u].sum() : 0.0);
    }
    out[row * LPR + li] = acc;
  }
}

template <int LPR, int VB, int UNR, bool ETA, int MINB>
static int launch(int n, const int* rp, const int* col, const double* U, const double* E, double* out,
                  int sms) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gather_kernel<LPR, VB, UNR, ETA, MINB>, 256, 0);
  gather_kernel<LPR, VB, UNR, ETA, MINB><<<occ * sms, 256>>>(n, rp, col, U, E, out);
  return occ;
}

extern "C" int gather_run(int variant, int n, const int* rp, const int* col, const double* U,
                          const double* E, double* out, int sms) {
  switch (variant) {
    case 0: return launch<4, 16, 1, true, 2>(n, rp, col, U, E, out, sms);
    case 1: return launch<4, 16, 2, true, 2>(n, rp, col, U, E, out, sms);
    case 2: return launch<4, 16, 4, true, 2>(n, rp, col, U, E, out, sms);
    case 3: return launch<4, 16, 8, true, 2>(n, rp, col, U, E, out, sms);
    case 4: return launch<2, 32, 1, true, 2>(n, rp, col, U, E, out, sms);
    case 5: return launch<2, 32, 4, true, 2>(n, rp, col, U, E, out, sms);
    case 6: return launch<4, 16, 4, true, 4>(n, rp, col, U, E, out, sms);
    case 7: return launch<4, 16, 8, true, 4>(n, rp, col, U, E, out, sms);
    case 8: return launch<4, 16, 4, false, 2>(n, rp, col, U, E, out, sms);
    case 9: return launch<4, 16, 8, false, 4>(n, rp, col, U, E, out, sms);
    case 10: return launch<2, 32, 4, true, 4>(n, rp, col, U, E, out, sms);
    case 11: return launch<4, 16, 2, true, 8>(n, rp, col, U, E, out, sms);
    default: return -1;
  }
}
