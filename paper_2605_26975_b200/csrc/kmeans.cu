#include <algorithm>
// k-means discretisation of the embedding (reading #13).
// Device kernels for k-means++ seeding (D^2 update, chunked cumulative sums, pick), the fused
// Lloyd assign + per-CTA centroid/count/SSE partials (fixed order, no atomics), empty-cluster
// repair (farthest point, lowest index), driven by a host loop with one small D2H per iteration.
#include <cstring>
#include <vector>

#include "dense_mma.cuh"
#include "plp_internal.h"

namespace plp {

constexpr int kKmThreads = 128;  // points per tile
constexpr int kChunk = 256;      // seeding cumsum chunk

// squared distance, ascending coordinates, no FMA contraction (same rounding as a plain loop)
__device__ __forceinline__ double km_dist2(const double* x, int xs, const double* c, int dim) {
  double s = 0.0;
  for (int d = 0; d < dim; ++d) {
    const double t = __dsub_rn(x[d * xs], c[d]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// D2[i] = dist2(x_i, c) (first) or min(D2[i], dist2(x_i, c)), and per chunk of kChunk = 256
// points (one CTA iteration) the chunk sum cs[chunk] (warp xor trees, warps in order)
__global__ void __launch_bounds__(kChunk) km_d2_kernel(int64_t n, int dim, const double* __restrict__ X,
                                                      const double* __restrict__ c, double* __restrict__ D2,
                                                      double* __restrict__ cs_out, int first) {
  __shared__ double cs[PLP_MAX_K];
  __shared__ double ws[kChunk / 32];
  if (threadIdx.x < dim) cs[threadIdx.x] = c[threadIdx.x];
  __syncthreads();
  const int64_t nch = (n + kChunk - 1) / kChunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool vec8 = dim == 8 && (reinterpret_cast<uintptr_t>(X) & 15u) == 0;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const int64_t i = ch * kChunk + threadIdx.x;
    double v = 0.0;
    if (i < n) {
      double d;
      if (vec8) {  // the row as four 16-byte loads (half the L1 wavefronts of eight 8-byte ones); same order
        const double2* xr = reinterpret_cast<const double2*>(X + i * 8);
        d = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 t = __ldg(xr + q);
          const double t0 = __dsub_rn(t.x, cs[2 * q]), t1 = __dsub_rn(t.y, cs[2 * q + 1]);
          d = __dadd_rn(d, __dmul_rn(t0, t0));
          d = __dadd_rn(d, __dmul_rn(t1, t1));
        }
      } else {
        d = km_dist2(X + i * dim, 1, cs, dim);
      }
      v = first ? d : (d < D2[i] ? d : D2[i]);
      D2[i] = v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) ws[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kChunk / 32; ++w) t += ws[w];
      cs_out[ch] = t;
    }
    __syncthreads();
  }
}

// Block-wide inclusive prefix sum (blockDim.x = 1024) of one value per thread, offset by base:
// warp shuffle scans, warp totals scanned by warp 0; every thread's result lands in pre[t].
__device__ void block_scan_to(double v, double base, double* wsum, double* pre) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wsum[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double w = lane < nw ? wsum[lane] : 0.0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) wsum[lane] = w;
  }
  __syncthreads();
  pre[threadIdx.x] = base + (v + (warp > 0 ? wsum[warp - 1] : 0.0));
  __syncthreads();
}

// First index e in [0, cnt) of a monotone running sum pre[] (exclusive value ex = pre[e - 1], or
// base at e = 0) with ex <= target < pre[e]; -1 if none.  Also the last e with a positive term.
__device__ void block_find(int cnt, double base, double target, const double* pre, int* s_hit, int* s_last) {
  const int t = threadIdx.x;
  if (t == 0) {
    *s_hit = -1;
    *s_last = -1;
  }
  __syncthreads();
  if (t < cnt) {
    const double ex = t > 0 ? pre[t - 1] : base;
    if (ex <= target && target < pre[t]) *s_hit = t;  // unique: pre is nondecreasing
    if (pre[t] > ex) atomicMax(s_last, t);
  }
  __syncthreads();
}

// D^2 pick (k-means++): the smallest i with cumsum(D^2)_i > u * sum(D^2), found top-down with
// parallel prefix sums: 1024 thread ranges of chunk sums, then the chunk sums of the chosen range
// (in slices of 1024), then the D^2 values of the chosen chunk.  The running sums differ from the
// oracle's sequential sum only in rounding order (reading #13); where rounding leaves no crossing
// inside the chosen range, its last positive entry is taken.
// Multi-rank seeding (plp_kmeans_dist) splits the pick: S_out != nullptr writes this rank's sum S
// and returns; target_in >= 0 replaces u * S by a given threshold (the global u * S less the
// lower ranks' sums) on the rank that owns the crossing.
__global__ void __launch_bounds__(1024) km_pick_kernel(int64_t n, int dim, const double* __restrict__ X,
                                                       const double* __restrict__ D2,
                                                       const double* __restrict__ cs, double u,
                                                       double* __restrict__ cent_row,
                                                       int64_t* pick_out, double target_in = -1.0,
                                                       double* S_out = nullptr) {
  __shared__ double wsum[32];
  __shared__ double pre[1024];
  __shared__ int s_hit, s_last;
  const int64_t nch = (n + kChunk - 1) / kChunk;
  const int T = blockDim.x, t = threadIdx.x;
  const int64_t per = (nch + T - 1) / T;
  double v = 0.0;
  for (int64_t c = t * per; c < (t + 1) * per && c < nch; ++c) v += cs[c];
  block_scan_to(v, 0.0, wsum, pre);
  const double S = pre[T - 1];
  if (S_out) {
    if (t == 0) *S_out = S;
    return;
  }
  int64_t pick;
  if (!(S > 0.0)) {
    pick = (int64_t)floor(u * (double)n);
    if (pick >= n) pick = n - 1;
  } else {
    const double target = target_in >= 0.0 ? target_in : u * S;
    // level 1: thread range q
    block_find(T, 0.0, target, pre, &s_hit, &s_last);
    const int q = s_hit >= 0 ? s_hit : s_last;
    double base = q > 0 ? pre[q - 1] : 0.0;
    __syncthreads();
    // level 2: chunk inside range q, slices of T chunks
    const int64_t c0 = (int64_t)q * per, c1 = ((int64_t)q + 1) * per < nch ? ((int64_t)q + 1) * per : nch;
    int64_t chosen = -1, lastpos = -1;
    double lastbase = base;
    for (int64_t cb = c0; cb < c1; cb += T) {
      const int cnt = (int)(c1 - cb < T ? c1 - cb : T);
      block_scan_to(t < cnt ? cs[cb + t] : 0.0, base, wsum, pre);
      block_find(cnt, base, target, pre, &s_hit, &s_last);
      if (s_last >= 0) {
        lastpos = cb + s_last;
        lastbase = s_last > 0 ? pre[s_last - 1] : base;
      }
      if (s_hit >= 0) {
        chosen = cb + s_hit;
        base = s_hit > 0 ? pre[s_hit - 1] : base;
        break;
      }
      base = pre[cnt - 1];
      __syncthreads();
    }
    if (chosen < 0) {  // rounding left no crossing: the last positive chunk of the range
      chosen = lastpos;
      base = lastbase;
    }
    __syncthreads();
    // level 3: point inside chunk `chosen`
    const int64_t i0 = chosen * kChunk, i1 = (chosen + 1) * kChunk < n ? (chosen + 1) * kChunk : n;
    const int cnt = (int)(i1 - i0);
    block_scan_to(t < cnt ? D2[i0 + t] : 0.0, base, wsum, pre);
    block_find(cnt, base, target, pre, &s_hit, &s_last);
    pick = i0 + (s_hit >= 0 ? s_hit : (s_last >= 0 ? s_last : cnt - 1));
  }
  if (t == 0 && pick_out) *pick_out = pick;
  if (t < dim) cent_row[t] = X[pick * dim + t];
}

// Fused assign (nearest centroid, ties -> lowest index) + per-CTA partials:
// part[b][0 .. K*dim) sums, [K*dim, K*dim+K) counts, [K*dim+K] sse.
__global__ void __launch_bounds__(kKmThreads) km_assign_kernel(int64_t n, int dim, int K,
                                                               const double* __restrict__ X,
                                                               const double* __restrict__ cent,
                                                               int32_t* __restrict__ lab,
                                                               double* __restrict__ best_d,
                                                               double* __restrict__ part) {
  __shared__ double cs[PLP_MAX_K * PLP_MAX_K];
  __shared__ double xs[kKmThreads * (PLP_MAX_K + 1)];
  __shared__ int ls[kKmThreads];
  __shared__ double bs[kKmThreads];
  const int pitch = dim | 1;
  for (int i = threadIdx.x; i < K * dim; i += blockDim.x) cs[i] = cent[i];
  const int E = K * dim + K + 1;
  double acc[9];
  for (int q = 0; q < 9; ++q) acc[q] = 0.0;
  const int64_t tiles = (n + kKmThreads - 1) / kKmThreads;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t p0 = tile * kKmThreads;
    const int np = (int)((n - p0) < kKmThreads ? (n - p0) : kKmThreads);
    __syncthreads();
    for (int idx = threadIdx.x; idx < np * dim; idx += blockDim.x)
      xs[(idx / dim) * pitch + idx % dim] = X[p0 * dim + idx];
    __syncthreads();
    const int t = threadIdx.x;
    if (t < np) {
      int bc = 0;
      double bd = km_dist2(xs + t * pitch, 1, cs, dim);
      for (int c = 1; c < K; ++c) {
        const double d = km_dist2(xs + t * pitch, 1, cs + c * dim, dim);
        if (d < bd) { bd = d; bc = c; }
      }
      lab[p0 + t] = bc;
      best_d[p0 + t] = bd;
      ls[t] = bc;
      bs[t] = bd;
    }
    __syncthreads();
    for (int q = 0; q * kKmThreads + threadIdx.x < E; ++q) {
      const int e = q * kKmThreads + threadIdx.x;
      double s = 0.0;
      if (e < K * dim) {
        const int c = e / dim, d = e % dim;
        for (int p = 0; p < np; ++p)
          if (ls[p] == c) s += xs[p * pitch + d];
      } else if (e < K * dim + K) {
        const int c = e - K * dim;
        for (int p = 0; p < np; ++p)
          if (ls[p] == c) s += 1.0;
      } else {
        for (int p = 0; p < np; ++p) s += bs[p];
      }
      acc[q] += s;
    }
  }
  for (int q = 0; q * kKmThreads + threadIdx.x < E; ++q)
    part[(int64_t)blockIdx.x * E + q * kKmThreads + threadIdx.x] = acc[q];
}

// Lloyd assign + centroid partials for K <= 8 clusters and dim <= 8 (the configs' C1, C2, C5):
// one thread per point for the distances (same exact rounding as km_dist2, ties -> lowest index),
// and the per-cluster sums / counts as one-hot^T X products on the fp64 tensor cores (DMMA
// m8n8k4: A[c][q] = [label of point q == c], B[q][d] = X[q][d] or 1), 4 points per instruction.
// Each warp owns a contiguous range of 32-point groups; per-CTA partials in a fixed order, layout
// [sums K*dim | counts K | sse] like km_assign_kernel.
#ifndef PLP_KM_PPL
#define PLP_KM_PPL 2  // points per lane and loop iteration (1: 78 / 64 registers at 3 / 4 CTAs per SM, but twice the
                     // centroid reads per point: 0.221 / 0.225 vs 0.208 ms per Lloyd iteration, r02t)
#endif
#ifndef PLP_KM_PREFETCH
#define PLP_KM_PREFETCH 1  // next group's point loads issued before the current group's DMMA phase
#endif
#ifndef PLP_KM_MINB
#define PLP_KM_MINB 2  // 128 registers with the prefetch (146 unbounded: one CTA per SM); 3 (80 registers,
                       // spills) measured slower before the prefetch: Lloyd 0.223 vs 0.211 ms
#endif
template <int DIM, int KC>  // DIM = 8: vectorised point loads; DIM = 0: runtime dim <= 8;
                           // KC = 8: K = 8 at compile time (unrolled); KC = 0: runtime K <= 8
__global__ void __launch_bounds__(256, KC == 8 ? PLP_KM_MINB : 1) km_assign_mma_kernel(int64_t n, int dim_rt, int K_rt,
                                                            const double* __restrict__ X,
                                                            const double* __restrict__ cent,
                                                            int32_t* __restrict__ lab,
                                                            double* __restrict__ best_d,
                                                            double* __restrict__ part) {
  constexpr int NW = 8, PPL = PLP_KM_PPL;  // two points per lane: each centroid load serves both
  const int dim = DIM > 0 ? DIM : dim_rt;
  const int K = KC > 0 ? KC : K_rt;
  __shared__ __align__(16) double cs[8 * 8];
  __shared__ double red[NW][8 * 8 + 8 + 1];
  for (int i = threadIdx.x; i < K * dim; i += blockDim.x) cs[i] = cent[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, q = lane & 3;
  const int64_t groups = (n + 32 * PPL - 1) / (32 * PPL);
  const int64_t tw = (int64_t)gridDim.x * NW, wid = (int64_t)blockIdx.x * NW + warp;
  const int64_t g0 = groups * wid / tw, g1 = groups * (wid + 1) / tw;
  double s0 = 0.0, s1 = 0.0, sse = 0.0;
  int cnt = 0;  // lane c < K counts cluster c
  // the lane's PPL points of group gr (rows past n read as zeros)
  double x[PPL][8];
  bool ok[PPL];
  auto load_group = [&](int64_t gr) {
#pragma unroll
    for (int h = 0; h < PPL; ++h) {
      const int64_t i = gr * 32 * PPL + 32 * h + lane;
      ok[h] = i < n;
      if constexpr (DIM == 8) {
        if (ok[h]) {
#pragma unroll
          for (int d = 0; d < 8; d += 2) {
            const double2 t = __ldg(reinterpret_cast<const double2*>(X + i * 8 + d));
            x[h][d] = t.x;
            x[h][d + 1] = t.y;
          }
        } else {
#pragma unroll
          for (int d = 0; d < 8; ++d) x[h][d] = 0.0;
        }
      } else {
#pragma unroll
        for (int d = 0; d < 8; ++d) x[h][d] = (ok[h] && d < dim) ? __ldg(X + i * dim + d) : 0.0;
      }
    }
  };
  // Software pipeline: the next group's point loads are issued as soon as the distances of the
  // current one are done (x is dead from there on), so their latency runs behind the label
  // stores, ballots and DMMAs of the current group.
  if (g0 < g1) load_group(g0);
  for (int64_t gr = g0; gr < g1; ++gr) {
    const int64_t p0 = gr * 32 * PPL;
    int bc[PPL];
    double bd[PPL];
#pragma unroll
    for (int h = 0; h < PPL; ++h) {
      bc[h] = 0;
      bd[h] = INFINITY;
    }
#pragma unroll(KC > 0 ? KC : 1)
    for (int c = 0; c < K; ++c) {
      double sd[PPL];
#pragma unroll
      for (int h = 0; h < PPL; ++h) sd[h] = 0.0;
      if constexpr (DIM == 8) {
        // centroid row as four 16-byte broadcasts (LDS.128), shared by the lane's points
        const double2* cr = reinterpret_cast<const double2*>(cs + c * 8);
#pragma unroll
        for (int d = 0; d < 8; d += 2) {
          const double2 cc = cr[d / 2];
#pragma unroll
          for (int h = 0; h < PPL; ++h) {
            const double t0 = __dsub_rn(x[h][d], cc.x);
            sd[h] = __dadd_rn(sd[h], __dmul_rn(t0, t0));
            const double t1 = __dsub_rn(x[h][d + 1], cc.y);
            sd[h] = __dadd_rn(sd[h], __dmul_rn(t1, t1));
          }
        }
      } else {
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          if (d < dim) {
            const double cv = cs[c * dim + d];
#pragma unroll
            for (int h = 0; h < PPL; ++h) {
              const double t = __dsub_rn(x[h][d], cv);
              sd[h] = __dadd_rn(sd[h], __dmul_rn(t, t));
            }
          }
        }
      }
#pragma unroll
      for (int h = 0; h < PPL; ++h)
        if (sd[h] < bd[h] || c == 0) {  // ties keep the lowest index
          bd[h] = sd[h];
          bc[h] = c;
        }
    }
    bool okc[PPL];
#pragma unroll
    for (int h = 0; h < PPL; ++h) okc[h] = ok[h];
#if PLP_KM_PREFETCH
    if (gr + 1 < g1) load_group(gr + 1);
#endif
#pragma unroll
    for (int h = 0; h < PPL; ++h) {
      const int64_t i = p0 + 32 * h + lane;
      if (okc[h]) {
        lab[i] = bc[h];
        best_d[i] = bd[h];
        sse += bd[h];
      } else {
        bc[h] = -1;
      }
    }
#pragma unroll
    for (int h = 0; h < PPL; ++h) {
      for (int c = 0; c < K; ++c) {
        const int m = __popc(__ballot_sync(0xffffffffu, bc[h] == c));
        if (lane == c) cnt += m;
      }
      const int64_t ph = p0 + 32 * h;
#pragma unroll
      for (int sb = 0; sb < 8; ++sb) {
        const int lq = __shfl_sync(0xffffffffu, bc[h], 4 * sb + q);
        const int64_t pq = ph + 4 * sb + q;
        const double a = (lq == g) ? 1.0 : 0.0;
        const double b = (pq < n && g < dim) ? __ldg(X + pq * dim + g) : 0.0;
        dmma884(s0, s1, a, b);
      }
    }
#if !PLP_KM_PREFETCH
    if (gr + 1 < g1) load_group(gr + 1);
#endif
  }
  // per-warp results -> shared, then a fixed-order sum over warps
  const int E = K * dim + K + 1;
  if (g < K) {
    if (2 * q < dim) red[warp][g * dim + 2 * q] = s0;
    if (2 * q + 1 < dim) red[warp][g * dim + 2 * q + 1] = s1;
  }
  if (lane < K) red[warp][K * dim + lane] = (double)cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sse += __shfl_xor_sync(0xffffffffu, sse, o);
  if (lane == 0) red[warp][E - 1] = sse;
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) t += red[w][e];
    part[(int64_t)blockIdx.x * E + e] = t;
  }
}

// red = [sums K*dim | counts K | sse]; cent[c] = sums/count where count > 0 (empty: unchanged)
__global__ void km_update_kernel(int K, int dim, const double* __restrict__ red, double* cent) {
  for (int e = threadIdx.x; e < K * dim; e += blockDim.x) {
    const int c = e / dim;
    const double cnt = red[K * dim + c];
    if (cnt > 0.0) cent[e] = red[e] / cnt;
  }
}

// argmax of best_d (lowest index on ties): per-block partials then a final pass
__global__ void km_argmax_kernel(int64_t n, const double* __restrict__ v, double* pv, int64_t* pi) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  double bv = -INFINITY;
  int64_t bi = n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (v[i] > bv) { bv = v[i]; bi = i; }
  sv[threadIdx.x] = bv;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double ov = sv[threadIdx.x + o];
      const int64_t oi = si[threadIdx.x + o];
      if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
        sv[threadIdx.x] = ov;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pv[blockIdx.x] = sv[0];
    pi[blockIdx.x] = si[0];
  }
}

__global__ void km_reseed_kernel(int grid, int dim, int c, const double* pv, const int64_t* pi,
                                 const double* __restrict__ X, double* cent, double* best_d) {
  __shared__ int64_t far;
  if (threadIdx.x == 0) {
    double bv = -INFINITY;
    int64_t bi = 0;
    for (int b = 0; b < grid; ++b)
      if (pv[b] > bv || (pv[b] == bv && pi[b] < bi)) { bv = pv[b]; bi = pi[b]; }
    far = bi;
  }
  __syncthreads();
  if (threadIdx.x < dim) cent[c * dim + threadIdx.x] = X[far * dim + threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) best_d[far] = -1.0;
}

// (value, index) of the argmax partials of km_argmax_kernel (largest value, lowest index)
__global__ void km_argmax_final_kernel(int grid, const double* pv, const int64_t* pi, double* out) {
  if (threadIdx.x == 0) {
    double bv = -INFINITY;
    int64_t bi = 0;
    for (int b = 0; b < grid; ++b)
      if (pv[b] > bv || (pv[b] == bv && pi[b] < bi)) { bv = pv[b]; bi = pi[b]; }
    out[0] = bv;
    out[1] = (double)bi;
  }
}

// out[e] = sum_b part[b][e]: one CTA per entry (thread-strided, warp xor trees, warps in order)
__global__ void __launch_bounds__(256) km_sum_kernel(int grid, int E, const double* part, double* out) {
  __shared__ double ws[8];
  const int e = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0.0;
  for (int b = threadIdx.x; b < grid; b += 256) s += part[(int64_t)b * E + e];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ws[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += ws[w];
    out[e] = t;
  }
}

}  // namespace plp

using namespace plp;

namespace plp {
// k-means over this rank's n rows; coll: the rows of all ranks of ctx in rank order (every
// reduction all-reduced, every pick made by the rank owning the point and broadcast), the
// single-rank computation when coll is false.
static plp_status kmeans_impl(plp_ctx* ctx, int64_t n, int dim, int K, const double* X,
                              const double* uniforms, int restarts, int max_iters, double rel_tol,
                              int32_t* labels, double* centroids, double* sse, int* iters, bool coll) {
  if (!ctx || (!X && n > 0) || !uniforms || (!labels && n > 0) || !centroids || !sse)
    return set_error(PLP_ERR_ARG, "null argument");
  if (dim < 1 || dim > PLP_MAX_K || K < 1 || K > PLP_MAX_K)
    return set_error(PLP_ERR_DOMAIN, "dim and clusters must be in [1, 32]");
  if (restarts < 1 || max_iters < 0) return set_error(PLP_ERR_ARG, "restarts >= 1, max_iters >= 0");
  if (n < 0) return set_error(PLP_ERR_SHAPE, "n >= 0");
  cudaStream_t st = ctx->stream;
  const int world = coll ? ctx->world : 1, rank = coll ? ctx->rank : 0;
  if (world > 512) return set_error(PLP_ERR_ARG, "plp_kmeans_dist: at most 512 ranks");
  // rank row offsets (all-reduce of a one-hot count vector: exact)
  std::vector<int64_t> cnt(world, 0), off(world + 1, 0);
  double* cscr = ctx->scratch + 4096;  // collective scratch: 2 x world doubles
  std::vector<double> hsc(2 * (size_t)world);
  if (coll) {
    double* dcnt = cscr + 1024;
    PLP_CUDA(cudaMemsetAsync(dcnt, 0, sizeof(double) * world, st));
    const double nd = (double)n;
    PLP_CUDA(cudaMemcpyAsync(dcnt + rank, &nd, sizeof(double), cudaMemcpyHostToDevice, st));
    plp_status s0 = comm_allreduce(ctx, dcnt, world);
    if (s0) return s0;
    PLP_CUDA(cudaMemcpyAsync(hsc.data(), dcnt, sizeof(double) * world, cudaMemcpyDeviceToHost, st));
    PLP_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < world; ++r) cnt[r] = (int64_t)hsc[r];
  } else {
    cnt[0] = n;
  }
  for (int r = 0; r < world; ++r) off[r + 1] = off[r] + cnt[r];
  const int64_t N = off[world], my0 = off[rank];
  if (N < K) return set_error(PLP_ERR_SHAPE, "need n >= clusters");
  auto owner_of = [&](int64_t gi) {
    int r = 0;
    while (r + 1 < world && gi >= off[r + 1]) ++r;
    return r;
  };
  // workspace: best_d (n), D2 (n), chunk sums, labels + centroids of the running restart
  const int64_t nch = (n + kChunk - 1) / kChunk;
  const size_t need = (size_t)(2 * n + nch + K * dim + (n + 1) / 2 + 64);
  // a point of this rank -> cent row (dev), and its all-reduce broadcast (others contribute 0)
  if (ctx->km_cap < need) {
    cudaFree(ctx->km_best);
    ctx->km_best = nullptr;
    ctx->km_cap = 0;
    PLP_CUDA(cudaMalloc(&ctx->km_best, need * sizeof(double)));
    ctx->km_cap = need;
  }
  double* best_d = ctx->km_best;
  double* D2 = best_d + n;
  double* csum = D2 + n;
  double* cent = csum + nch;
  int32_t* lab = reinterpret_cast<int32_t*>(cent + K * dim);
  const int E = K * dim + K + 1;
  int grid = (int)((n + kKmThreads - 1) / kKmThreads);
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  const int64_t part_cap = (int64_t)ctx->max_ctas * 4 * PLP_MAX_K;
  if ((int64_t)grid * E > part_cap) grid = (int)(part_cap / E);
  double* red = ctx->scratch + 256;  // E <= 32*32+33 doubles
  static const int res_d2 = resident_ctas(km_d2_kernel, kChunk);
  const int gridd = (int)std::min<int64_t>((int64_t)ctx->num_sms * res_d2, std::max<int64_t>(1, nch));
  int gridn = (int)((n + 255) / 256);
  if (gridn > ctx->max_ctas) gridn = ctx->max_ctas;
  double* pv = ctx->partials;
  int64_t* pi = reinterpret_cast<int64_t*>(ctx->partials + ctx->max_ctas);
  std::vector<double> host(E);
  double best = INFINITY;
  int best_iters = 0;
  // broadcast of centre row c from the rank that wrote it (the others zero it): exact
  auto bcast_row = [&](int c) -> plp_status { return comm_allreduce(ctx, cent + (int64_t)c * dim, dim); };
  auto zero_row = [&](int c) -> plp_status {
    PLP_CUDA(cudaMemsetAsync(cent + (int64_t)c * dim, 0, sizeof(double) * dim, st));
    return PLP_OK;
  };
  for (int r = 0; r < restarts; ++r) {
    const double* u = uniforms + (int64_t)r * K;
    plp_status s;
    // ---- k-means++ seeding ----
    int64_t c0 = (int64_t)floor(u[0] * (double)N);
    if (c0 >= N) c0 = N - 1;
    if (coll && (s = zero_row(0))) return s;
    if (c0 >= my0 && c0 < my0 + n)
      PLP_CUDA(cudaMemcpyAsync(cent, X + (c0 - my0) * dim, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
    if (coll && (s = bcast_row(0))) return s;
    for (int m = 1; m < K; ++m) {
      if (n > 0) {
        km_d2_kernel<<<gridd, kChunk, 0, st>>>(n, dim, X, cent + (int64_t)(m - 1) * dim, D2, csum, m == 1);
        PLP_LAUNCH_CHECK("km_d2_kernel");
      }
      if (!coll) {
        km_pick_kernel<<<1, 1024, 0, st>>>(n, dim, X, D2, csum, u[m], cent + (int64_t)m * dim, nullptr);
        PLP_LAUNCH_CHECK("km_pick_kernel");
        continue;
      }
      // every rank's sum of D^2, the global threshold u * sum, and the rank whose running sum
      // crosses it (where rounding leaves no crossing: the last rank with a positive sum)
      PLP_CUDA(cudaMemsetAsync(cscr, 0, sizeof(double) * world, st));
      if (n > 0) {
        km_pick_kernel<<<1, 1024, 0, st>>>(n, dim, X, D2, csum, u[m], nullptr, nullptr, -1.0, cscr + rank);
        PLP_LAUNCH_CHECK("km_pick_kernel");
      }
      if ((s = comm_allreduce(ctx, cscr, world))) return s;
      PLP_CUDA(cudaMemcpyAsync(hsc.data(), cscr, sizeof(double) * world, cudaMemcpyDeviceToHost, st));
      PLP_CUDA(cudaStreamSynchronize(st));
      double S = 0.0;
      for (int q = 0; q < world; ++q) S += hsc[q];
      if ((s = zero_row(m))) return s;
      if (!(S > 0.0)) {
        int64_t pk = (int64_t)floor(u[m] * (double)N);
        if (pk >= N) pk = N - 1;
        if (pk >= my0 && pk < my0 + n)
          PLP_CUDA(cudaMemcpyAsync(cent + (int64_t)m * dim, X + (pk - my0) * dim, sizeof(double) * dim,
                                   cudaMemcpyDeviceToDevice, st));
      } else {
        const double target = u[m] * S;
        int own = -1, lastpos = -1;
        double pre = 0.0, pre_own = 0.0, pre_last = 0.0;
        for (int q = 0; q < world; ++q) {
          const double nx = pre + hsc[q];
          if (hsc[q] > 0.0) { lastpos = q; pre_last = pre; }
          if (own < 0 && pre <= target && target < nx) { own = q; pre_own = pre; }
          pre = nx;
        }
        if (own < 0) { own = lastpos; pre_own = pre_last; }
        if (own == rank) {
          km_pick_kernel<<<1, 1024, 0, st>>>(n, dim, X, D2, csum, u[m], cent + (int64_t)m * dim, nullptr,
                                             target - pre_own, nullptr);
          PLP_LAUNCH_CHECK("km_pick_kernel");
        }
      }
      if ((s = bcast_row(m))) return s;
    }
    // ---- Lloyd ----
    const bool mma = K <= 8 && dim <= 8;
    static const int res_mma88 = resident_ctas(km_assign_mma_kernel<8, 8>, 256);
    static const int res_mma0 = std::min(resident_ctas(km_assign_mma_kernel<8, 0>, 256),
                                         resident_ctas(km_assign_mma_kernel<0, 0>, 256));
    const bool mma88 = dim == 8 && K == 8 && ((uintptr_t)X & 15u) == 0;
    int grid_mma = ctx->num_sms * (mma88 ? res_mma88 : res_mma0);  // one full wave
    if ((int64_t)grid_mma * E > part_cap) grid_mma = (int)(part_cap / E);
    const int64_t groups = (n + 63) / 64;
    if (groups < (int64_t)grid_mma * 8) grid_mma = (int)std::max<int64_t>(1, (groups + 7) / 8);
    auto assign = [&](double* sse_out, std::vector<double>& h) -> plp_status {
      if (n == 0) {
        PLP_CUDA(cudaMemsetAsync(red, 0, sizeof(double) * E, st));
      } else {
        if (mma) {
          if (mma88)
            km_assign_mma_kernel<8, 8><<<grid_mma, 256, 0, st>>>(n, dim, K, X, cent, lab, best_d, ctx->partials);
          else if (dim == 8 && ((uintptr_t)X & 15u) == 0)
            km_assign_mma_kernel<8, 0><<<grid_mma, 256, 0, st>>>(n, dim, K, X, cent, lab, best_d, ctx->partials);
          else
            km_assign_mma_kernel<0, 0><<<grid_mma, 256, 0, st>>>(n, dim, K, X, cent, lab, best_d, ctx->partials);
          PLP_LAUNCH_CHECK("km_assign_mma_kernel");
        } else {
          km_assign_kernel<<<grid, kKmThreads, 0, st>>>(n, dim, K, X, cent, lab, best_d, ctx->partials);
          PLP_LAUNCH_CHECK("km_assign_kernel");
        }
        km_sum_kernel<<<E, 256, 0, st>>>(mma ? grid_mma : grid, E, ctx->partials, red);
        PLP_LAUNCH_CHECK("km_sum_kernel");
      }
      if (coll) {  // sums, counts and sse over the ranks
        plp_status s2 = comm_allreduce(ctx, red, E);
        if (s2) return s2;
      }
      PLP_CUDA(cudaMemcpyAsync(h.data(), red, sizeof(double) * E, cudaMemcpyDeviceToHost, st));
      PLP_CUDA(cudaStreamSynchronize(st));
      *sse_out = h[E - 1];
      return PLP_OK;
    };
    double cur = 0.0;
    s = assign(&cur, host);
    if (s) return s;
    int it = 0;
    while (it < max_iters) {
      km_update_kernel<<<1, 256, 0, st>>>(K, dim, red, cent);
      PLP_LAUNCH_CHECK("km_update_kernel");
      for (int c = 0; c < K; ++c) {
        if (host[K * dim + c] > 0.0) continue;  // empty cluster -> farthest point
        if (!coll) {
          km_argmax_kernel<<<gridn, 256, 0, st>>>(n, best_d, pv, pi);
          PLP_LAUNCH_CHECK("km_argmax_kernel");
          km_reseed_kernel<<<1, 32, 0, st>>>(gridn, dim, c, pv, pi, X, cent, best_d);
          PLP_LAUNCH_CHECK("km_reseed_kernel");
          continue;
        }
        // every rank's farthest point (value, global index); largest value, lowest index wins
        std::vector<double> vi(2 * (size_t)world);
        PLP_CUDA(cudaMemsetAsync(cscr, 0, sizeof(double) * 2 * world, st));
        if (n > 0) {
          km_argmax_kernel<<<gridn, 256, 0, st>>>(n, best_d, pv, pi);
          PLP_LAUNCH_CHECK("km_argmax_kernel");
          km_argmax_final_kernel<<<1, 32, 0, st>>>(gridn, pv, pi, cscr + 2 * rank);
          PLP_LAUNCH_CHECK("km_argmax_final_kernel");
        }
        if ((s = comm_allreduce(ctx, cscr, 2 * (size_t)world))) return s;
        PLP_CUDA(cudaMemcpyAsync(vi.data(), cscr, sizeof(double) * 2 * world, cudaMemcpyDeviceToHost, st));
        PLP_CUDA(cudaStreamSynchronize(st));
        int own = -1;
        for (int q = 0; q < world; ++q)
          if (cnt[q] > 0 && (own < 0 || vi[2 * q] > vi[2 * own])) own = q;
        if ((s = zero_row(c))) return s;
        if (own == rank) {
          km_reseed_kernel<<<1, 32, 0, st>>>(gridn, dim, c, pv, pi, X, cent, best_d);
          PLP_LAUNCH_CHECK("km_reseed_kernel");
        }
        if ((s = bcast_row(c))) return s;
      }
      double nxt = 0.0;
      if ((s = assign(&nxt, host))) return s;
      ++it;
      const bool conv = (cur == 0.0) || (fabs(cur - nxt) < rel_tol * cur);
      cur = nxt;
      if (conv) break;
    }
    if (cur < best) {
      best = cur;
      best_iters = it;
      if (n > 0) PLP_CUDA(cudaMemcpyAsync(labels, lab, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
      PLP_CUDA(cudaMemcpyAsync(centroids, cent, sizeof(double) * K * dim, cudaMemcpyDeviceToDevice, st));
    }
  }
  PLP_CUDA(cudaStreamSynchronize(st));
  *sse = best;
  if (iters) *iters = best_iters;
  return PLP_OK;
}
}  // namespace plp

extern "C" plp_status plp_kmeans(plp_ctx* ctx, int64_t n, int dim, int K, const double* X,
                                 const double* uniforms, int restarts, int max_iters,
                                 double rel_tol, int32_t* labels, double* centroids, double* sse,
                                 int* iters) {
  PLP_NVTX("plp_kmeans");
  if (n < 1) return set_error(PLP_ERR_SHAPE, "need n >= clusters");
  return kmeans_impl(ctx, n, dim, K, X, uniforms, restarts, max_iters, rel_tol, labels, centroids, sse, iters,
                     false);
}

extern "C" plp_status plp_kmeans_dist(plp_ctx* ctx, int64_t n_local, int dim, int K, const double* X,
                                      const double* uniforms, int restarts, int max_iters, double rel_tol,
                                      int32_t* labels, double* centroids, double* sse, int* iters) {
  PLP_NVTX("plp_kmeans_dist");
  if (!ctx) return set_error(PLP_ERR_ARG, "null argument");
  return kmeans_impl(ctx, n_local, dim, K, X, uniforms, restarts, max_iters, rel_tol, labels, centroids, sse,
                     iters, ctx->comm != nullptr);
}
