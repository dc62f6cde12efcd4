#include <algorithm>
// Tall-skinny n x k kernels of the Grassmann solver: Gram products
// X^T Y with a fixed-order reduction, k x k Cholesky on one warp, row-block apply (X M, X - U M,
// (X+Y) R^-1), dot, axpby and row gathers.  All HBM-bound: k <= 32 doubles per row.
#include "dense_mma.cuh"
#include "plp_internal.h"

namespace plp {

constexpr int kGramThreads = 256;
constexpr int kGramRows = 32;  // rows per smem tile

// partials[block][k*k] = sum over this block's tiles of (X+Xa)^T (Y+Ya)
__global__ void __launch_bounds__(kGramThreads) gram_kernel(int64_t n, int k, const double* __restrict__ X,
                                                            const double* __restrict__ Xa,
                                                            const double* __restrict__ Y,
                                                            const double* __restrict__ Ya,
                                                            double* __restrict__ part) {
  __shared__ double xs[kGramRows * PLP_MAX_K];
  __shared__ double ys[kGramRows * PLP_MAX_K];
  __shared__ double red[kGramThreads];
  const int E = k * k;
  const int t = threadIdx.x;
  const int S = E <= kGramThreads ? kGramThreads / E : 1;  // row slices per entry
  const int per = E <= kGramThreads ? 1 : (E + kGramThreads - 1) / kGramThreads;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t tiles = (n + kGramRows - 1) / kGramRows;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * kGramRows;
    const int rows = (int)((n - r0) < kGramRows ? (n - r0) : kGramRows);
    __syncthreads();
    for (int idx = t; idx < kGramRows * k; idx += kGramThreads) {
      double xv = 0.0, yv = 0.0;
      if (idx < rows * k) {
        const int64_t g = r0 * k + idx;
        xv = X[g];
        if (Xa) xv += Xa[g];
        yv = Y[g];
        if (Ya) yv += Ya[g];
      }
      xs[idx] = xv;
      ys[idx] = yv;
    }
    __syncthreads();
    if (per == 1) {
      const int e = t % E, sl = t / E;
      if (sl < S) {
        const int a = e / k, b = e % k;
        for (int r = sl; r < rows; r += S) acc[0] = fma(xs[r * k + a], ys[r * k + b], acc[0]);
      }
    } else {
      for (int q = 0; q < per; ++q) {
        const int e = t + q * kGramThreads;
        if (e < E) {
          const int a = e / k, b = e % k;
          for (int r = 0; r < rows; ++r) acc[q] = fma(xs[r * k + a], ys[r * k + b], acc[q]);
        }
      }
    }
  }
  if (per == 1) {
    __syncthreads();
    red[t] = acc[0];
    __syncthreads();
    if (t < E) {
      double s = 0.0;
      for (int sl = 0; sl < S; ++sl) s += red[sl * E + t];
      part[(int64_t)blockIdx.x * E + t] = s;
    }
  } else {
    for (int q = 0; q < per; ++q) {
      const int e = t + q * kGramThreads;
      if (e < E) part[(int64_t)blockIdx.x * E + e] = acc[q];
    }
  }
}

// out[e] = sum_b part[b][e] (lane-strided then xor tree: fixed order)
__global__ void __launch_bounds__(1024) sum_partials_kernel(int grid, int E, const double* part,
                                                            double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = warp; e < E; e += (blockDim.x >> 5)) {
    double s = 0.0;
    for (int b = lane; b < grid; b += 32) s += part[(int64_t)b * E + e];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[e] = s;
  }
}

// Column `lane` of the inverse of an upper-triangular r (smem, k x k) by back substitution.
__device__ void upper_inverse(int k, const double* r, double* Rinv, int lane) {
  if (lane >= k) return;
  double v[PLP_MAX_K];
  for (int i = 0; i < k; ++i) v[i] = 0.0;
  v[lane] = 1.0 / r[lane * k + lane];
  for (int i = lane - 1; i >= 0; --i) {
    double s = 0.0;
    for (int m = i + 1; m <= lane; ++m) s += r[i * k + m] * v[m];
    v[i] = -s / r[i * k + i];
  }
  for (int i = 0; i < k; ++i) Rinv[i * k + lane] = v[i];
}

// Upper Cholesky C = R^T R (R_ii > 0) and R^-1 on one warp; info = 0 or the failing pivot (1-based).
__global__ void chol_kernel(int k, const double* __restrict__ C, double* __restrict__ R,
                            double* __restrict__ Rinv, int* info) {
  __shared__ double c[PLP_MAX_K * PLP_MAX_K];
  __shared__ double r[PLP_MAX_K * PLP_MAX_K];
  __shared__ int bad;
  const int lane = threadIdx.x;
  for (int i = lane; i < k * k; i += 32) {
    c[i] = C[i];
    r[i] = 0.0;
  }
  if (lane == 0) bad = 0;
  __syncwarp();
  for (int j = 0; j < k; ++j) {
    if (lane == 0) {
      double d = c[j * k + j];
      for (int m = 0; m < j; ++m) d -= r[m * k + j] * r[m * k + j];
      if (!(d > 0.0) && bad == 0) bad = j + 1;
      r[j * k + j] = d > 0.0 ? sqrt(d) : 1.0;
    }
    __syncwarp();
    if (lane > j && lane < k) {
      double s = c[j * k + lane];
      for (int m = 0; m < j; ++m) s -= r[m * k + j] * r[m * k + lane];
      r[j * k + lane] = s / r[j * k + j];
    }
    __syncwarp();
  }
  if (Rinv) upper_inverse(k, r, Rinv, lane);
  __syncwarp();
  for (int i = lane; i < k * k; i += 32) R[i] = r[i];
  if (lane == 0 && info) *info = bad;
}

__global__ void trinv_kernel(int k, const double* __restrict__ R, double* __restrict__ Rinv) {
  __shared__ double r[PLP_MAX_K * PLP_MAX_K];
  for (int i = threadIdx.x; i < k * k; i += 32) r[i] = R[i];
  __syncwarp();
  upper_inverse(k, r, Rinv, threadIdx.x);
}

// out = R2 R1 (k x k, both upper triangular)
__global__ void rmul_kernel(int k, const double* R2, const double* R1, double* out) {
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e / k, j = e % k;
    double s = 0.0;
    for (int m = 0; m < k; ++m) s += R2[i * k + m] * R1[m * k + j];
    out[e] = s;
  }
}

// out_i = S_i + sgn * (X_i + Xa_i) M for each row i; a group of G lanes per row, lane l < k owns
// column l; the row is shared through shuffles, so out may alias S, X or Xa.
template <int G>
__global__ void __launch_bounds__(256) apply_kernel(int64_t n, int k, const double* S, double sgn,
                                                    const double* X, const double* Xa,
                                                    const double* __restrict__ M, double* out) {
  __shared__ double m[PLP_MAX_K * PLP_MAX_K];
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) m[i] = M[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int l = lane % G;
  const int base = lane - l;
  const int64_t rows_per_iter = (int64_t)(blockDim.x / 32) * (32 / G);
  const int64_t first = (int64_t)blockIdx.x * rows_per_iter + (threadIdx.x >> 5) * (32 / G) + lane / G;
  const int64_t stride = (int64_t)gridDim.x * rows_per_iter;
  const int64_t iters = (n + stride - 1) / stride;  // uniform trip count: all lanes shuffle
  for (int64_t it = 0; it < iters; ++it) {
    const int64_t i = first + it * stride;
    const bool ok = i < n && l < k;
    double x = 0.0, s = 0.0;
    if (ok) {
      x = X[i * k + l];
      if (Xa) x += Xa[i * k + l];
      if (S) s = S[i * k + l];
    }
    double acc = 0.0;
    for (int q = 0; q < k; ++q) {
      const double xq = __shfl_sync(0xffffffffu, x, base + q);
      if (ok) acc = fma(xq, m[q * k + l], acc);
    }
    if (ok) out[i * k + l] = fma(sgn, acc, s);
  }
}

__global__ void __launch_bounds__(256) dot_kernel(int64_t total, const double* __restrict__ x,
                                                  const double* __restrict__ y, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], y[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void axpby_kernel(int64_t total, double a, const double* __restrict__ x, double b,
                             double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}

__global__ void gather_rows_kernel(int64_t m, int k, const int64_t* __restrict__ idx,
                                   const double* __restrict__ X, double* __restrict__ out) {
  const int64_t total = m * k;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / k;
    const int l = (int)(t % k);
    out[t] = X[idx[r] * k + l];
  }
}

static int grid_for(plp_ctx* ctx, int64_t work_items, int per_block) {
  int64_t g = (work_items + per_block - 1) / per_block;
  if (g > ctx->max_ctas) g = ctx->max_ctas;
  if (g < 1) g = 1;
  return (int)g;
}

// scratch layout (doubles) for the dense path: [256 + s*1024, ...) slot s
static double* dslot(plp_ctx* ctx, int s) { return ctx->scratch + 256 + (size_t)s * 1024; }

static plp_status gram(plp_ctx* ctx, int64_t n, int k, const double* X, const double* Xa,
                       const double* Y, const double* Ya, double* out) {
  if (k == 8 || k == 16) {  // fp64 tensor cores (dense_mma.cuh)
    static const int res1 = resident_ctas(gram_mma_kernel<1, false>, kMmaThreads),
                     res2 = resident_ctas(gram_mma_kernel<2, false>, kMmaThreads);
    int grid = ctx->num_sms * (k == 8 ? res1 : res2);  // one full wave
    const int cap = (int)(((int64_t)ctx->max_ctas * 4 * PLP_MAX_K) / (k * k));
    if (grid > cap) grid = cap;
    const int64_t blocks = (n + 3) / 4;
    if (blocks < (int64_t)grid * 8) grid = (int)std::max<int64_t>(1, (blocks + 7) / 8);
    const bool sym = X == Y && Xa == Ya;
    if (k == 8 && sym) gram_mma_kernel<1, true><<<grid, kMmaThreads, 0, ctx->stream>>>(n, X, Xa, Y, Ya, ctx->partials);
    else if (k == 8) gram_mma_kernel<1, false><<<grid, kMmaThreads, 0, ctx->stream>>>(n, X, Xa, Y, Ya, ctx->partials);
    else if (sym) gram_mma_kernel<2, true><<<grid, kMmaThreads, 0, ctx->stream>>>(n, X, Xa, Y, Ya, ctx->partials);
    else gram_mma_kernel<2, false><<<grid, kMmaThreads, 0, ctx->stream>>>(n, X, Xa, Y, Ya, ctx->partials);
    PLP_LAUNCH_CHECK("gram_mma_kernel");
    sum_partials_kernel<<<1, 1024, 0, ctx->stream>>>(grid, k * k, ctx->partials, out);
    PLP_LAUNCH_CHECK("sum_partials_kernel");
    return PLP_OK;
  }
  int grid = grid_for(ctx, (n + kGramRows - 1) / kGramRows, 1);
  const int cap = (int)(((int64_t)ctx->max_ctas * 4 * PLP_MAX_K) / (k * k));  // partials capacity
  if (grid > cap) grid = cap;
  gram_kernel<<<grid, kGramThreads, 0, ctx->stream>>>(n, k, X, Xa, Y, Ya, ctx->partials);
  PLP_LAUNCH_CHECK("gram_kernel");
  sum_partials_kernel<<<1, 1024, 0, ctx->stream>>>(grid, k * k, ctx->partials, out);
  PLP_LAUNCH_CHECK("sum_partials_kernel");
  return PLP_OK;
}

static plp_status apply(plp_ctx* ctx, int64_t n, int k, const double* S, double sgn,
                        const double* X, const double* Xa, const double* M, double* out) {
  auto al16 = [](const void* p) { return ((uintptr_t)p & 15u) == 0; };
  if ((k == 8 || k == 16) && al16(out) && (S == nullptr || al16(S))) {  // fp64 tensor cores
    const int64_t blocks = (n + 7) / 8;
    static const int res1 = resident_ctas(apply_mma_kernel<1>, kMmaThreads),
                     res2 = resident_ctas(apply_mma_kernel<2>, kMmaThreads);
    int64_t grid = (int64_t)ctx->num_sms * (k == 8 ? res1 : res2);  // one full wave
    if (blocks < grid * 8) grid = std::max<int64_t>(1, (blocks + 7) / 8);
    if (k == 8) apply_mma_kernel<1><<<(int)grid, kMmaThreads, 0, ctx->stream>>>(n, S, sgn, X, Xa, M, out);
    else apply_mma_kernel<2><<<(int)grid, kMmaThreads, 0, ctx->stream>>>(n, S, sgn, X, Xa, M, out);
    PLP_LAUNCH_CHECK("apply_mma_kernel");
    return PLP_OK;
  }
  int G = 1;
  while (G < k) G <<= 1;
  const int rows_per_block = 8 * (32 / G);
  const int grid = grid_for(ctx, n, rows_per_block);
#define PLP_APPLY(GG) apply_kernel<GG><<<grid, 256, 0, ctx->stream>>>(n, k, S, sgn, X, Xa, M, out)
  switch (G) {
    case 1: PLP_APPLY(1); break;
    case 2: PLP_APPLY(2); break;
    case 4: PLP_APPLY(4); break;
    case 8: PLP_APPLY(8); break;
    case 16: PLP_APPLY(16); break;
    default: PLP_APPLY(32); break;
  }
#undef PLP_APPLY
  PLP_LAUNCH_CHECK("apply_kernel");
  return PLP_OK;
}

}  // namespace plp

using namespace plp;

#define PLP_REQ(cond, msg) \
  do {                     \
    if (!(cond)) return set_error(PLP_ERR_ARG, msg); \
  } while (0)

extern "C" plp_status plp_gram(plp_ctx* ctx, int64_t n, int k, const double* X, const double* Y,
                               double* out) {
  PLP_NVTX("plp_gram");
  PLP_REQ(ctx && X && Y && out && n >= 0, "bad argument");
  plp_status st = check_k(k);
  if (st) return st;
  st = gram(ctx, n, k, X, nullptr, Y, nullptr, out);
  if (st) return st;
  return comm_allreduce(ctx, out, (size_t)k * k);  // collective on a multi-rank ctx
}

extern "C" plp_status plp_apply_sub(plp_ctx* ctx, int64_t n, int k, const double* U,
                                    const double* M, const double* X, double* out) {
  PLP_REQ(ctx && U && M && X && out && n >= 0, "bad argument");
  plp_status st = check_k(k);
  if (st) return st;
  return apply(ctx, n, k, X, -1.0, U, nullptr, M, out);
}

extern "C" plp_status plp_project(plp_ctx* ctx, int64_t n, int k, const double* U, const double* G,
                                  double* out) {
  PLP_NVTX("plp_project");
  PLP_REQ(ctx && U && G && out && n >= 0, "bad argument");
  plp_status st = check_k(k);
  if (st) return st;
  double* M = dslot(ctx, 0);
  st = gram(ctx, n, k, U, nullptr, G, nullptr, M);  // M = U^T G
  if (st) return st;
  if ((st = comm_allreduce(ctx, M, (size_t)k * k))) return st;  // global Gram (multi-rank ctx)
  return apply(ctx, n, k, G, -1.0, U, nullptr, M, out);  // G - U M
}

extern "C" plp_status plp_cholesky(plp_ctx* ctx, int k, const double* C, double* R, int* info) {
  PLP_REQ(ctx && C && R, "bad argument");
  plp_status st = check_k(k);
  if (st) return st;
  chol_kernel<<<1, 32, 0, ctx->stream>>>(k, C, R, nullptr, info ? info : ctx->flag);
  PLP_LAUNCH_CHECK("chol_kernel");
  return PLP_OK;
}

extern "C" plp_status plp_apply_rinv(plp_ctx* ctx, int64_t n, int k, const double* X,
                                     const double* Y, const double* R, double* Q) {
  PLP_REQ(ctx && X && R && Q && n >= 0, "bad argument");
  plp_status st = check_k(k);
  if (st) return st;
  double* Rinv = dslot(ctx, 5);
  trinv_kernel<<<1, 32, 0, ctx->stream>>>(k, R, Rinv);
  PLP_LAUNCH_CHECK("trinv_kernel");
  return apply(ctx, n, k, nullptr, 1.0, X, Y, Rinv, Q);  // Q = (X + Y) R^-1
}

extern "C" plp_status plp_retract(plp_ctx* ctx, int64_t n, int k, const double* U, const double* xi,
                                  double* Q, double* R_out) {
  PLP_NVTX("plp_retract");
  PLP_REQ(ctx && U && xi && Q && n >= 0, "bad argument");
  plp_status st = check_k(k);
  if (st) return st;
  double *C1 = dslot(ctx, 0), *R1 = dslot(ctx, 1), *R1i = dslot(ctx, 2);
  double *C2 = dslot(ctx, 3), *R2 = dslot(ctx, 4), *R2i = dslot(ctx, 5);
  PLP_CUDA(cudaMemsetAsync(ctx->flag, 0, 2 * sizeof(int), ctx->stream));
  // Cholesky-QR2: Y = U + xi; Q1 = Y R1^-1; Q = Q1 R2^-1; R = R2 R1
  if ((st = gram(ctx, n, k, U, xi, U, xi, C1))) return st;
  if ((st = comm_allreduce(ctx, C1, (size_t)k * k))) return st;  // global Grams (multi-rank ctx)
  chol_kernel<<<1, 32, 0, ctx->stream>>>(k, C1, R1, R1i, ctx->flag);
  PLP_LAUNCH_CHECK("chol_kernel");
  if ((st = apply(ctx, n, k, nullptr, 1.0, U, xi, R1i, Q))) return st;
  if ((st = gram(ctx, n, k, Q, nullptr, Q, nullptr, C2))) return st;
  if ((st = comm_allreduce(ctx, C2, (size_t)k * k))) return st;
  chol_kernel<<<1, 32, 0, ctx->stream>>>(k, C2, R2, R2i, ctx->flag + 1);
  PLP_LAUNCH_CHECK("chol_kernel");
  if ((st = apply(ctx, n, k, nullptr, 1.0, Q, nullptr, R2i, Q))) return st;
  if (R_out) {
    rmul_kernel<<<1, 256, 0, ctx->stream>>>(k, R2, R1, R_out);
    PLP_LAUNCH_CHECK("rmul_kernel");
  }
  int info[2] = {0, 0};
  PLP_CUDA(cudaMemcpyAsync(info, ctx->flag, sizeof(info), cudaMemcpyDeviceToHost, ctx->stream));
  PLP_CUDA(cudaStreamSynchronize(ctx->stream));
  if (info[0] || info[1])
    return set_error(PLP_ERR_RANK, "Cholesky-QR: Gram not positive definite at pivot %d (pass %d)",
                     info[0] ? info[0] : info[1], info[0] ? 1 : 2);
  return PLP_OK;
}

extern "C" plp_status plp_dot(plp_ctx* ctx, int64_t n, int k, const double* x, const double* y,
                              double* out) {
  PLP_NVTX("plp_dot");
  PLP_REQ(ctx && x && y && out && n >= 0 && k >= 1, "bad argument");
  const int64_t total = n * k;
  const int grid = grid_for(ctx, total, 256 * 8);
  dot_kernel<<<grid, 256, 0, ctx->stream>>>(total, x, y, ctx->partials);
  PLP_LAUNCH_CHECK("dot_kernel");
  sum_partials_kernel<<<1, 32, 0, ctx->stream>>>(grid, 1, ctx->partials, out);
  PLP_LAUNCH_CHECK("sum_partials_kernel");
  return comm_allreduce(ctx, out, 1);  // collective on a multi-rank ctx
}

extern "C" plp_status plp_axpby(plp_ctx* ctx, int64_t n, int k, double a, const double* x, double b,
                                double* y) {
  PLP_NVTX("plp_axpby");
  PLP_REQ(ctx && x && y && n >= 0 && k >= 1, "bad argument");
  const int64_t total = n * k;
  const int grid = grid_for(ctx, total, 256 * 4);
  axpby_kernel<<<grid, 256, 0, ctx->stream>>>(total, a, x, b, y);
  PLP_LAUNCH_CHECK("axpby_kernel");
  return PLP_OK;
}

extern "C" plp_status plp_gather_rows(plp_ctx* ctx, int64_t m, int k, const int64_t* idx,
                                      const double* X, double* out) {
  PLP_REQ(ctx && idx && X && out && m >= 0 && k >= 1, "bad argument");
  if (m == 0) return PLP_OK;
  const int grid = grid_for(ctx, m * k, 256 * 4);
  gather_rows_kernel<<<grid, 256, 0, ctx->stream>>>(m, k, idx, X, out);
  PLP_LAUNCH_CHECK("gather_rows_kernel");
  return PLP_OK;
}
