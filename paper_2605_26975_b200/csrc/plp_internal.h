// Internal declarations of libplp (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "plp.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: a no-op unless a profiler injects itself

#define PLP_MAX_K 32
// Cap used by passes that need no curvature (objective, gradient, full-mode epilogue): s is then
// unused and t = a^{p-1} must stay on the fast path for every a > 0 (pow64.cuh).
constexpr double kNoCap = 1e-300;

// Resident CTAs per SM of a kernel at this block size (grids sized to whole waves: a grid of
// num_sms x this many CTAs runs in one wave, with no partial second wave).
template <class Kernel>
inline int resident_ctas(Kernel kernel, int threads, size_t smem = 0) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem) != cudaSuccess || b < 1) {
    cudaGetLastError();
    b = 1;
  }
  return b;
}

struct plp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  int max_ctas = 0;          // edge/dense kernels' fixed reduction grid upper bound
  double* partials = nullptr;  // max_ctas * 4 * PLP_MAX_K doubles
  double* scratch = nullptr;   // 8 * PLP_MAX_K * PLP_MAX_K doubles (Grams, R, AB, dots)
  int* flag = nullptr;         // device status flags (Cholesky info, ...)
  int64_t* iscratch = nullptr; // device int64 scratch (argmax index, sizes)
  void* pow_tables = nullptr;  // device PowTables for the generic power (pow64.cuh)
  // k-means workspace (grown at plp_kmeans entry if needed; not a hot edge call)
  double* km_best = nullptr;
  size_t km_cap = 0;
  // collective layer (comm.cu): rank / world and the NCCL communicator (ncclComm_t; nullptr on a
  // single-rank context created without an id)
  int rank = 0, world = 1;
  void* comm = nullptr;
  cudaStream_t comm_stream = nullptr;       // halo exchanges overlapped with interior tiles
  cudaEvent_t ev_in = nullptr, ev_halo = nullptr;
};

// Halo plan of a graph created by plp_create_graph_dist (comm.cu): this rank owns global rows
// [row_begin, row_end); its dense arrays hold those rows followed by the n_halo halo rows (sorted
// global ids, local ids n_own + h).  Per peer q: recv slice [recv_off[q], + recv_cnt[q]) of the
// halo; send_cnt[q] rows listed from send_idx[send_off[q]] (local row ids, in q's halo order).
struct plp_dist {
  int64_t n_global = 0, row_begin = 0, row_end = 0, n_own = 0, n_halo = 0;
  std::vector<int64_t> bounds, send_off, send_cnt, recv_off, recv_cnt;
  int64_t total_send = 0;
  int32_t* send_idx = nullptr;  // device
  void* sendbuf = nullptr;      // device, total_send rows of up to PLP_MAX_K doubles
  size_t sendbuf_bytes = 0;
  // halo-kernel tiles (PLP_HALO_TILE rows) with no halo column first, then the boundary tiles:
  // the interior ones run while the halo exchange is in flight
  int32_t* tile_order = nullptr;  // device, n_interior + n_boundary entries
  int64_t n_interior = 0, n_boundary = 0;
};

struct plp_graph {
  plp_ctx* ctx = nullptr;
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  int32_t* rp = nullptr;     // device int32 row_ptr[n_rows+1]
  int32_t* col = nullptr;    // device int32 col[nnz]
  double* w = nullptr;       // device fp64 w[nnz]
  int32_t* sched = nullptr;  // device row schedule: rows sorted by degree within windows
  int max_chunk_nnz = 0;  // max nnz over chunks of kStagedChunk rows (staged kernel ring slots)
  // Halo tiles (edge_halo.cuh): tiles of PLP_HALO_TILE rows; per stored edge the tile-local index
  // (j - r0 inside the tile, PLP_HALO_TILE + x for the x-th halo row); per tile a slot of
  // halo_ext_cap + 4 ints at halo_ext[t * (halo_ext_cap + 4)]: n_ext, rp[r0], rp[r1], 0, then the
  // halo columns (-1 padded).  nullptr halo_enc: no halo tiles.
  int32_t* halo_enc = nullptr;
  int32_t* halo_ext = nullptr;
  int halo_ext_cap = 0;  // max halo rows per tile (rounded up to 4)
  int halo_nnz_cap = 0;  // max stored edges per tile (rounded up to 4)
  // objective mode (A over the upper triangle): the graph is square, symmetric with bitwise equal
  // weights and sorted rows; nlow[i] = stored edges of row i with col < i
  bool upper_ok = false;
  int32_t* nlow = nullptr;
  int32_t* sched_up = nullptr;  // rows by decreasing upper-edge count within 32-row windows
  plp_dist* dist = nullptr;     // multi-rank halo plan (plp_create_graph_dist), else nullptr
};
// rows per degree-sorting window: small enough that a CTA's rows per iteration stay contiguous
// (neighbour rows of a tile-ordered graph then hit L1)
#ifndef PLP_SCHED_WINDOW
#define PLP_SCHED_WINDOW 16  // degree-sorting window (the halo kernel's tiles are whole windows)
#endif
constexpr int kSchedWindow = PLP_SCHED_WINDOW;
// rows per chunk of the staged kernel (a union of whole degree-sorting windows)
constexpr int kStagedChunk = 32;
static_assert(kStagedChunk % kSchedWindow == 0, "staged chunks hold whole schedule windows");
namespace plp {

// NVTX range over one C-ABI call (named after it), for nsys / ncu --nvtx timelines of the solver
// (SURVEY.md §5 tracing).  Host-side push / pop only: nothing is enqueued on the stream.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define PLP_NVTX(name) ::plp::NvtxRange plp_nvtx_range_(name)

plp_status set_error(plp_status st, const char* fmt, ...);
plp_status cuda_check(cudaError_t e, const char* what);

#define PLP_CUDA(x)                                              \
  do {                                                           \
    cudaError_t e_ = (x);                                        \
    if (e_ != cudaSuccess) return ::plp::cuda_check(e_, #x);     \
  } while (0)

#define PLP_LAUNCH_CHECK(what)                                   \
  do {                                                           \
    cudaError_t e_ = cudaGetLastError();                         \
    if (e_ != cudaSuccess) return ::plp::cuda_check(e_, what);   \
  } while (0)

plp_status check_p(double p, double eps);
// collective layer (comm.cu)
plp_status comm_init(plp_ctx* ctx, int rank, int world, const void* nccl_id);
void comm_destroy(plp_ctx* ctx);
plp_status comm_allreduce(plp_ctx* ctx, double* buf, size_t count);  // in place, no-op on one rank
plp_status comm_allreduce_i64(plp_ctx* ctx, int64_t* buf, size_t count);
plp_status halo_exchange_bytes(plp_ctx* ctx, const plp_graph* g, void* X, int row_bytes,
                               cudaStream_t stream = nullptr);  // nullptr: ctx->stream
void dist_destroy(plp_dist* d);
// records the last launched edge kernel's name (plp_last_edge_kernel)
void note_edge_kernel(const char* family, int kc, int cpl, int lpr, int unr, const char* pow, int eta);
plp_status check_k(int k);

// Edge kernel launcher (edge.cu).
struct EdgeArgs {
  int64_t n_rows;
  int64_t n_cols;  // rows of U / eta (owned + halo)
  const int32_t* rp;
  const int32_t* sched;
  const int32_t* col;
  const double* w;
  int k;
  const double* U;
  const double* eta;
  const double* AB;     // global A,B for the coefficients (nullptr: objective only)
  double* G;
  double* Hv;
  double p, eps;
  double* partials;     // [grid][4][k]: A, B, alpha, gamma partial sums
  int want_dots;
  int need_ab;   // the caller reduces the A, B partials (0: a Hessian-vector-only pass may skip them)
  // staged kernel (edge_staged.cuh): largest chunk nnz of the graph, ring slot capacity
  int max_chunk_nnz, chunk_cap;
  int ldx;  // row stride (elements) of U and eta in the staged kernel; 0 = k (contiguous)
  // halo-tile kernel (edge_halo.cuh)
  const int32_t* halo_enc;
  const int32_t* halo_ext;
  int halo_ext_cap, halo_nnz_cap;
  int halo_stage;  // halo rows staged per tile (< halo_ext_cap: overflow mode); set by the launcher
  // optional work list of the halo kernel: tiles tile_list[tile_begin, + tile_count) only (the
  // interior / boundary launches of a multi-rank call); other kernels refuse a list
  const int32_t* tile_list;
  int64_t tile_begin, tile_count;
  const int32_t* nlow;  // objective mode (edge_halo.cuh)
  const int32_t* sched_up;
  int upper_ok;
  // fused tCG (tcg.cu): a Hessian-vector-only halo pass at k = 4 / 8 may also accumulate pass A's
  // sums (M1 = U^T EH, M2 = U^T eta, sum eta (EH - eta S)) into `partials`, entry-major per CTA;
  // gram_S is the 8 x 8 S (k = 4: block-diagonal), *gram_used (host) tells the caller it did
  const double* gram_S;
  int* gram_used;
};
plp_status launch_edge(plp_ctx* ctx, const EdgeArgs& a, int* grid_out);
plp_status hessvec_gram(plp_ctx* ctx, const plp_graph* g, int k, const double* U, const double* eta,
                        double p, const double* AB_in, double eps, const double* S8, double* Hv,
                        int* grid, bool* used);
// Fixed-order reduction of edge partials: AB_out (2k), dots_out (2k), F (1); any may be null.
plp_status launch_edge_finalize(plp_ctx* ctx, int grid, int k, const double* partials,
                                double* AB_out, double* dots_out, double* F);

}  // namespace plp
