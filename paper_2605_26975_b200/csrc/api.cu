// Context, graph handle, error reporting and argument checks of libplp (plp.h).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <new>
#include <vector>

#include "plp_internal.h"
#include "pow64.cuh"

namespace plp {

static thread_local char g_err[512] = "";

plp_status set_error(plp_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

plp_status cuda_check(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation)
    return set_error(PLP_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
  return set_error(PLP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

plp_status check_p(double p, double eps) {
  if (!(p > 1.0 && p <= 2.0)) return set_error(PLP_ERR_DOMAIN, "p = %g not in (1, 2]", p);
  if (p < 2.0 && !(eps >= 1e-300 && eps < 1e300))
    return set_error(PLP_ERR_DOMAIN, "eps = %g must be a normal double in [1e-300, 1e300) when p < 2",
                     eps);
  return PLP_OK;
}

plp_status check_k(int k) {
  if (k < 1 || k > PLP_MAX_K) return set_error(PLP_ERR_DOMAIN, "k = %d not in [1, 32]", k);
  return PLP_OK;
}

// Tables of the generic power (pow64.cuh), computed on the host in long double.
static void fill_pow_tables(PowTables* t) {
  for (int j = 0; j < 128; ++j) {
    const long double c = 1.0L + (j + 0.5L) / 128.0L;
    const double invc = (double)(1.0L / c);
    t->logt[j].x = invc;
    t->logt[j].y = (double)(-log2l((long double)invc));
  }
  for (int j = 0; j < 64; ++j) t->expt[j] = (double)exp2l((long double)j / 64.0L);
}

}  // namespace plp

using namespace plp;

extern "C" const char* plp_last_error(void) { return g_err; }
extern "C" const char* plp_version(void) { return "libplp 0.3 (sm_100a)"; }
extern "C" int plp_halo_tile_rows(void) { return PLP_HALO_TILE; }

static char g_last_edge_kernel[160] = "";
void plp::note_edge_kernel(const char* family, int kc, int cpl, int lpr, int unr, const char* pow,
                           int eta) {
  snprintf(g_last_edge_kernel, sizeof(g_last_edge_kernel), "%s<K=%d,CPL=%d,LPR=%d,UNR=%d,pow=%s,eta=%d>",
           family, kc, cpl, lpr, unr, pow, eta);
}
extern "C" const char* plp_last_edge_kernel(void) { return g_last_edge_kernel; }

extern "C" plp_status plp_ctx_create(int device, void* stream, int rank, int world,
                                     const void* nccl_id, plp_ctx** out) {
  if (!out) return set_error(PLP_ERR_ARG, "out is null");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return set_error(PLP_ERR_ARG, "bad rank/world");
  if (world > 1 && !nccl_id) return set_error(PLP_ERR_ARG, "world > 1 needs an NCCL unique id");
  PLP_CUDA(cudaSetDevice(device));
  plp_ctx* c = new (std::nothrow) plp_ctx();
  if (!c) return set_error(PLP_ERR_OOM, "host allocation failed");
  c->device = device;
  c->stream = (cudaStream_t)stream;
  cudaDeviceProp pr;
  cudaError_t e = cudaGetDeviceProperties(&pr, device);
  if (e != cudaSuccess) { delete c; return cuda_check(e, "cudaGetDeviceProperties"); }
  c->num_sms = pr.multiProcessorCount;
  c->max_ctas = c->num_sms * 8;
  const size_t part = (size_t)c->max_ctas * 4 * PLP_MAX_K * sizeof(double);
  const size_t scr = (size_t)16 * PLP_MAX_K * PLP_MAX_K * sizeof(double);
  if ((e = cudaMalloc(&c->partials, part)) != cudaSuccess ||
      (e = cudaMalloc(&c->scratch, scr)) != cudaSuccess ||
      (e = cudaMalloc(&c->flag, 64)) != cudaSuccess ||
      (e = cudaMalloc(&c->iscratch, 64 * sizeof(int64_t))) != cudaSuccess ||
      (e = cudaMalloc(&c->pow_tables, sizeof(PowTables))) != cudaSuccess) {
    plp_ctx_destroy(c);
    return cuda_check(e, "cudaMalloc(ctx workspace)");
  }
  PowTables t;
  fill_pow_tables(&t);
  if ((e = cudaMemcpy(c->pow_tables, &t, sizeof(t), cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemset(c->scratch, 0, scr)) != cudaSuccess ||
      (e = cudaMemset(c->flag, 0, 64)) != cudaSuccess) {
    plp_ctx_destroy(c);
    return cuda_check(e, "ctx init");
  }
  plp_status st = comm_init(c, rank, world, nccl_id);  // collective when an id is given
  if (st) {
    plp_ctx_destroy(c);
    return st;
  }
  *out = c;
  return PLP_OK;
}

extern "C" plp_status plp_ctx_set_stream(plp_ctx* ctx, void* stream) {
  if (!ctx) return set_error(PLP_ERR_ARG, "ctx is null");
  ctx->stream = (cudaStream_t)stream;
  return PLP_OK;
}

extern "C" plp_status plp_ctx_destroy(plp_ctx* ctx) {
  if (!ctx) return PLP_OK;
  comm_destroy(ctx);
  cudaFree(ctx->partials);
  cudaFree(ctx->scratch);
  cudaFree(ctx->flag);
  cudaFree(ctx->iscratch);
  cudaFree(ctx->pow_tables);
  cudaFree(ctx->km_best);
  delete ctx;
  return PLP_OK;
}

extern "C" plp_status plp_ctx_info(const plp_ctx* ctx, int* num_sms, int* max_ctas) {
  if (!ctx) return set_error(PLP_ERR_ARG, "ctx is null");
  if (num_sms) *num_sms = ctx->num_sms;
  if (max_ctas) *max_ctas = ctx->max_ctas;
  return PLP_OK;
}

// Halo tiles for edge_halo.cuh (see plp_graph): per tile of PLP_HALO_TILE consecutive rows its
// sorted distinct outside columns, and per stored edge the tile-local neighbour index.  Skipped
// (nullptr halo_enc) when a tile's buffers could not fit in shared memory even at k = 8.
static plp_status build_halo_tiles(plp_graph* g, const int64_t* rp, const int32_t* col,
                                   const double* w) {
  const int64_t n = g->n_rows;
  const int T = PLP_HALO_TILE;
  const int64_t nt = (n + T - 1) / T;
  if (nt == 0) return PLP_OK;
  std::vector<int64_t> xoff((size_t)nt + 1, 0);
  std::vector<int32_t> xs;
  int max_ext = 0, max_nnz = 0;
  std::vector<int32_t> tmp;
  std::vector<std::pair<int32_t, int32_t>> cnt;  // (-references, column)
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t r0 = t * T, r1 = std::min<int64_t>(n, r0 + T);
    tmp.clear();
    for (int64_t e = rp[r0]; e < rp[r1]; ++e)
      if (col[e] < r0 || col[e] >= r1) tmp.push_back(col[e]);
    std::sort(tmp.begin(), tmp.end());
    // halo rows by decreasing number of references (ties: column order), so that when a tile's
    // halo overflows shared memory (overflow mode) the rows left in L2 are the least used ones
    cnt.clear();
    for (size_t q = 0; q < tmp.size();) {
      size_t r = q;
      while (r < tmp.size() && tmp[r] == tmp[q]) ++r;
      cnt.emplace_back(-(int32_t)(r - q), tmp[q]);
      q = r;
    }
    std::sort(cnt.begin(), cnt.end());
    tmp.resize(cnt.size());
    for (size_t q = 0; q < cnt.size(); ++q) tmp[q] = cnt[q].second;
    xs.insert(xs.end(), tmp.begin(), tmp.end());
    xoff[t + 1] = (int64_t)xs.size();
    max_ext = std::max<int>(max_ext, (int)tmp.size());
    max_nnz = std::max<int64_t>(max_nnz, rp[r1] - rp[r0]);
  }
  // no locality (generator-order graphs, C4's 10-D kNN graph: ~7-10 outside rows per tile row):
  // halo tiles would mostly overflow to L2, and the staged / row kernels do better (measured
  // 3.5 ms against 3.1 ms at C5 in generator order); C3's 3-D grid (1.6 halo rows per tile row)
  // keeps them (overflow mode, 0.24 against 0.34 ms staged)
  if ((double)xs.size() > 3.0 * (double)T * (double)nt) return PLP_OK;
  const int ext_cap = (max_ext + 3) & ~3, nnz_cap = (max_nnz + 3) & ~3;
#ifndef PLP_HALO_NBUF
#define PLP_HALO_NBUF 2
#endif
  // skipped only if not even 64 halo rows per tile fit next to the tile's own data at k = 8 (the
  // launcher stages what fits and reads the rest from L2: overflow mode)
  const double bytes_k8 = PLP_HALO_NBUF * ((T + 64) * 128.0 + nnz_cap * 12.0 + 4096.0);
#ifndef PLP_HALO_CTAS
#define PLP_HALO_CTAS 1
#endif
  if (bytes_k8 > 224.0 * 1024.0 / PLP_HALO_CTAS) return PLP_OK;
  std::vector<int32_t> enc((size_t)g->nnz + 16, 0);
  // per tile a slot of ext_cap + 4 ints: n_ext, rp[r0], rp[r1], 0, then the halo columns
  const int64_t LS = ext_cap + 4;
  std::vector<int32_t> ext((size_t)(nt * LS + 16), -1);
  for (int64_t t = 0; t < nt; ++t) {
    const int64_t r0 = t * T, r1 = std::min<int64_t>(n, r0 + T);
    const int32_t* xb = xs.data() + xoff[t];
    const int32_t* xe = xs.data() + xoff[t + 1];
    ext[t * LS + 0] = (int32_t)(xe - xb);
    ext[t * LS + 1] = (int32_t)rp[r0];
    ext[t * LS + 2] = (int32_t)rp[r1];
    ext[t * LS + 3] = 0;
    std::copy(xb, xe, ext.begin() + t * LS + 4);
    // tile-local index of each halo column (the list is ordered by references, not by column)
    std::vector<std::pair<int32_t, int32_t>> pos;
    pos.reserve(xe - xb);
    for (const int32_t* q = xb; q < xe; ++q) pos.emplace_back(*q, (int32_t)(q - xb));
    std::sort(pos.begin(), pos.end());
    for (int64_t e = rp[r0]; e < rp[r1]; ++e) {
      const int32_t j = col[e];
      enc[e] = (j >= r0 && j < r1)
                   ? (int32_t)(j - r0)
                   : (int32_t)(T + std::lower_bound(pos.begin(), pos.end(), std::make_pair(j, INT32_MIN))->second);
    }
  }
  cudaError_t e;
  if ((e = cudaMalloc(&g->halo_enc, sizeof(int32_t) * enc.size())) != cudaSuccess ||
      (e = cudaMalloc(&g->halo_ext, sizeof(int32_t) * ext.size())) != cudaSuccess ||
      (e = cudaMemcpy(g->halo_enc, enc.data(), sizeof(int32_t) * enc.size(), cudaMemcpyHostToDevice)) !=
          cudaSuccess ||
      (e = cudaMemcpy(g->halo_ext, ext.data(), sizeof(int32_t) * ext.size(), cudaMemcpyHostToDevice)) !=
          cudaSuccess)
    return cuda_check(e, "cudaMalloc/cudaMemcpy(halo tiles)");
  g->halo_ext_cap = ext_cap;
  g->halo_nnz_cap = nnz_cap;
  // objective mode: square graph, sorted rows, symmetric with bitwise equal weights
  if (g->n_rows == g->n_cols) {
    std::vector<int32_t> nlow((size_t)n + 16, 0);
    bool ok = true;
    for (int64_t i = 0; i < n && ok; ++i) {
      int32_t cnt = 0;
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t j = col[e];
        if (e > rp[i] && col[e - 1] >= j) { ok = false; break; }
        cnt += j < i;
        const int32_t* b = col + rp[j];
        const int32_t* f = std::lower_bound(b, col + rp[j + 1], (int32_t)i);
        if (f == col + rp[j + 1] || *f != i || w[rp[j] + (f - b)] != w[e] || j == i) { ok = false; break; }
      }
      nlow[i] = cnt;
    }
    if (ok) {
      // objective-mode schedule: within each 32-row window, rows by decreasing upper-edge count
      // (the objective loop of a row pass runs over its rows' upper edges only)
      std::vector<int32_t> sup((size_t)n + 16, 0);
      for (int64_t w0 = 0; w0 < n; w0 += kSchedWindow) {
        const int64_t w1 = std::min<int64_t>(n, w0 + kSchedWindow);
        for (int64_t i = w0; i < w1; ++i) sup[i] = (int32_t)i;
        std::stable_sort(sup.begin() + w0, sup.begin() + w1, [&](int32_t x, int32_t y) {
          return (rp[x + 1] - rp[x] - nlow[x]) > (rp[y + 1] - rp[y] - nlow[y]);
        });
      }
      if ((e = cudaMalloc(&g->nlow, sizeof(int32_t) * nlow.size())) != cudaSuccess ||
          (e = cudaMemcpy(g->nlow, nlow.data(), sizeof(int32_t) * nlow.size(), cudaMemcpyHostToDevice)) !=
              cudaSuccess ||
          (e = cudaMalloc(&g->sched_up, sizeof(int32_t) * sup.size())) != cudaSuccess ||
          (e = cudaMemcpy(g->sched_up, sup.data(), sizeof(int32_t) * sup.size(), cudaMemcpyHostToDevice)) !=
              cudaSuccess)
        return cuda_check(e, "cudaMalloc/cudaMemcpy(nlow)");
      g->upper_ok = true;
    }
  }
  return PLP_OK;
}

extern "C" plp_status plp_create_graph(plp_ctx* ctx, int64_t n_rows, int64_t n_cols,
                                       const int64_t* row_ptr, const int32_t* col, const double* w,
                                       uint32_t flags, plp_graph** out) {
  PLP_NVTX("plp_create_graph");
  if (!ctx || !out || !row_ptr || (!col && row_ptr[n_rows] > 0) || (!w && row_ptr[n_rows] > 0))
    return set_error(PLP_ERR_ARG, "null argument");
  *out = nullptr;
  if (n_rows < 0 || n_cols < n_rows) return set_error(PLP_ERR_SHAPE, "need 0 <= n_rows <= n_cols");
  if (n_cols >= ((int64_t)1 << 31)) return set_error(PLP_ERR_SHAPE, "n_cols must be < 2^31");
  const int64_t nnz = row_ptr[n_rows];
  if (nnz < 0 || nnz >= ((int64_t)1 << 31)) return set_error(PLP_ERR_SHAPE, "nnz must be < 2^31");
  if (flags & (PLP_VALIDATE | PLP_VALIDATE_SYMMETRIC)) {
    plp_status st = plp_validate_csr(n_rows, n_cols, row_ptr, col, w,
                                     (flags & PLP_VALIDATE_SYMMETRIC) ? 1 : 0);
    if (st) return st;
  }
  PLP_CUDA(cudaSetDevice(ctx->device));
  plp_graph* g = new (std::nothrow) plp_graph();
  if (!g) return set_error(PLP_ERR_OOM, "host allocation failed");
  g->ctx = ctx;
  g->n_rows = n_rows;
  g->n_cols = n_cols;
  g->nnz = nnz;
  std::vector<int32_t> rp32((size_t)n_rows + 1);
  for (int64_t i = 0; i <= n_rows; ++i) rp32[i] = (int32_t)row_ptr[i];
  // Row schedule: within windows of kSchedWindow consecutive rows, rows by decreasing degree
  // (stable), so that the row groups of one warp see near-equal degrees (no divergence) while
  // the window keeps the U_j gathers L2-local.  Row results do not depend on it.
  // (+16 entries: the staged kernel's bulk copies round the schedule slice up to 16 bytes)
  std::vector<int32_t> sched((size_t)n_rows + 16, 0);
  for (int64_t c0 = 0; c0 < n_rows; c0 += kStagedChunk) {
    const int64_t c1 = std::min<int64_t>(n_rows, c0 + kStagedChunk);
    g->max_chunk_nnz = std::max<int>(g->max_chunk_nnz, rp32[c1] - rp32[c0]);
  }
  for (int64_t w0 = 0; w0 < n_rows; w0 += kSchedWindow) {
    const int64_t w1 = std::min<int64_t>(n_rows, w0 + kSchedWindow);
    for (int64_t i = w0; i < w1; ++i) sched[i] = (int32_t)i;
    std::stable_sort(sched.begin() + w0, sched.begin() + w1, [&](int32_t x, int32_t y) {
      return (rp32[x + 1] - rp32[x]) > (rp32[y + 1] - rp32[y]);
    });
  }
  cudaError_t e;
  if ((e = cudaMalloc(&g->sched, sizeof(int32_t) * sched.size())) != cudaSuccess ||
      (e = cudaMemcpy(g->sched, sched.data(), sizeof(int32_t) * sched.size(), cudaMemcpyHostToDevice)) !=
          cudaSuccess) {
    plp_destroy_graph(g);
    return cuda_check(e, "graph schedule");
  }
  // (+16 elements of padding: the tiled kernel's bulk copies round ranges up to 16 bytes)
  if ((e = cudaMalloc(&g->rp, sizeof(int32_t) * (n_rows + 1 + 16))) != cudaSuccess ||
      (e = cudaMalloc(&g->col, sizeof(int32_t) * (nnz + 16))) != cudaSuccess ||
      (e = cudaMalloc(&g->w, sizeof(double) * (nnz + 16))) != cudaSuccess) {
    plp_destroy_graph(g);
    return cuda_check(e, "cudaMalloc(graph)");
  }
  if ((e = cudaMemcpy(g->rp, rp32.data(), sizeof(int32_t) * (n_rows + 1), cudaMemcpyHostToDevice)) !=
          cudaSuccess ||
      (nnz > 0 && (e = cudaMemcpy(g->col, col, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice)) !=
                      cudaSuccess) ||
      (nnz > 0 && (e = cudaMemcpy(g->w, w, sizeof(double) * nnz, cudaMemcpyHostToDevice)) !=
                      cudaSuccess)) {
    plp_destroy_graph(g);
    return cuda_check(e, "cudaMemcpy(graph)");
  }
  plp_status st = build_halo_tiles(g, row_ptr, col, w);
  if (st) {
    plp_destroy_graph(g);
    return st;
  }
  *out = g;
  return PLP_OK;
}

extern "C" plp_status plp_graph_info(const plp_graph* g, int64_t* n_rows, int64_t* n_cols,
                                     int64_t* nnz) {
  if (!g) return set_error(PLP_ERR_ARG, "graph is null");
  if (n_rows) *n_rows = g->n_rows;
  if (n_cols) *n_cols = g->n_cols;
  if (nnz) *nnz = g->nnz;
  return PLP_OK;
}

extern "C" plp_status plp_destroy_graph(plp_graph* g) {
  if (!g) return PLP_OK;
  cudaFree(g->rp);
  cudaFree(g->col);
  cudaFree(g->w);
  cudaFree(g->sched);
  cudaFree(g->halo_enc);
  cudaFree(g->halo_ext);
  cudaFree(g->nlow);
  cudaFree(g->sched_up);
  dist_destroy(g->dist);
  delete g;
  return PLP_OK;
}
