// Step-0 box-facts microbenchmarks: fp64 pipe rates on B200.
// Standalone; not part of the product path.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void k_dfma(double* out, int iters, double a, double b, long long* cyc) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == 12345.678f) out[0] = s;
}

__global__ void k_pow(double* out, int iters, double q) {
  double x = 0.5 + threadIdx.x * 1e-4 + blockIdx.x * 1e-6;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
    s += pow(x, q);
    x += 1e-7;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_rsqrt(double* out, int iters) {
  double x = 0.5 + threadIdx.x * 1e-4 + blockIdx.x * 1e-6;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
    s += rsqrt(x);
    x += 1e-7;
  }
  if (s == 12345.678) out[0] = s;
}

__global__ void k_cvt(double* out, int iters) {
  double x = 0.5 + threadIdx.x * 1e-4;
  float y = 0;
  for (int it = 0; it < iters; ++it) {
    y += __double2float_rn(x);
    x = (double)y * 1e-3 + 0.25;
  }
  if (y == 12345.678f) out[0] = y;
}

// fp64 tensor cores: mma.sync m8n8k4 f64 (DMMA), CH independent accumulators per warp
template <int CH>
__global__ void k_dmma(double* out, int iters) {
  double d[CH][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  int l2 = 0; CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  printf("device %s SMs %d L2 %d B smemPerSM %zu\n", pr.name, pr.multiProcessorCount, l2, pr.sharedMemPerMultiprocessor);
  double* dout; float* fout; long long* cyc;
  CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&fout, 64)); CK(cudaMalloc(&cyc, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = pr.multiProcessorCount;
  int blocks = sms * 8, threads = 256;
  const int iters = 4096;
  float ms;
  // warm
  k_dfma<8><<<blocks, threads>>>(dout, 16, 1.0000001, 1e-9, cyc);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_dfma<8><<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9, cyc);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double nf = (double)blocks * threads * iters * 8;
  printf("DFMA: %.3f ms, %.2f T DFMA/s, block0 cycles %lld -> eff clock %.0f MHz, DFMA/clk/SM %.1f\n", ms, nf / ms / 1e9, c,
         c / (ms * 1e3), nf / sms / (c * 1.0));
  k_dmma<8><<<blocks, threads>>>(dout, 16);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_dmma<8><<<blocks, threads>>>(dout, iters);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  {
    const double nm = (double)blocks * (threads / 32) * iters * 8;  // warp-level DMMA instructions
    printf("DMMA m8n8k4 f64: %.3f ms, %.2f T DMMA/s, %.2f TFLOP/s (512 flop each)\n", ms, nm / ms / 1e9,
           nm * 512.0 / ms / 1e9);
  }
  k_ffma<8><<<blocks, threads>>>(fout, 16, 1.0000001f, 1e-9f);
  cudaEventRecord(e0);
  k_ffma<8><<<blocks, threads>>>(fout, iters, 1.0000001f, 1e-9f);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FFMA: %.3f ms, %.2f T FFMA/s\n", ms, nf / ms / 1e9);
  const int piters = 512;
  k_pow<<<blocks, threads>>>(dout, 8, -0.8);
  cudaEventRecord(e0);
  k_pow<<<blocks, threads>>>(dout, piters, -0.8);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double np = (double)blocks * threads * piters;
  printf("pow(fp64): %.3f ms, %.2f G pow/s\n", ms, np / ms / 1e6);
  k_rsqrt<<<blocks, threads>>>(dout, 8);
  cudaEventRecord(e0);
  k_rsqrt<<<blocks, threads>>>(dout, piters);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("rsqrt(fp64): %.3f ms, %.2f G/s\n", ms, np / ms / 1e6);
  k_cvt<<<blocks, threads>>>(dout, 8);
  cudaEventRecord(e0);
  k_cvt<<<blocks, threads>>>(dout, piters);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cvt f64->f32 chain (latency-ish): %.3f ms, %.2f G/s\n", ms, np / ms / 1e6);
  size_t bytes = (size_t)2 << 30;
  double4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 0, bytes);
  size_t n4 = bytes / 32;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    k_copy<<<sms * 8, 512>>>(a, b, n4);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 2 GiB: %.3f ms, %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
  }
  return 0;
}
