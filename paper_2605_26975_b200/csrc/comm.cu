// Collective layer of libplp (SURVEY.md §8(b) "on P ranks each call is collective", §8(e)):
// the NCCL communicator lives in the context, graphs created with plp_create_graph_dist carry
// their halo plan (who sends which rows to whom), and the edge / dense entry points exchange the
// halo rows of U and eta and all-reduce their small partial outputs (A, B, dots, k x k Grams)
// themselves, on the ctx stream.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"; in a process that already loaded PyTorch's
// NCCL the same library is reused), so libplp has no link-time NCCL dependency and the host-only
// entry points work without it.  One process per GPU; over NVLink 5 / NVSwitch NCCL's P2P
// send/recv and its all-reduce (NVLS where available) carry the halo rows and the <= 3 KB
// reductions.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "plp_internal.h"

namespace plp {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;
static std::once_flag g_nccl_once;
static std::string g_nccl_err;

static void load_nccl() {
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* nm : names) {
    h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);  // already in the process (torch)?
    if (!h) h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (h) break;
  }
  if (!h) {
    g_nccl_err = std::string("dlopen(libnccl.so.2) failed: ") + (dlerror() ? dlerror() : "?");
    return;
  }
  NcclApi a;
  a.h = h;
#define PLP_SYM(field, name)                                               \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));           \
  if (!a.field) {                                                          \
    g_nccl_err = std::string("NCCL symbol missing: ") + name;              \
    return;                                                                \
  }
  PLP_SYM(GetUniqueId, "ncclGetUniqueId");
  PLP_SYM(CommInitRank, "ncclCommInitRank");
  PLP_SYM(CommDestroy, "ncclCommDestroy");
  PLP_SYM(AllReduce, "ncclAllReduce");
  PLP_SYM(AllGather, "ncclAllGather");
  PLP_SYM(Send, "ncclSend");
  PLP_SYM(Recv, "ncclRecv");
  PLP_SYM(GroupStart, "ncclGroupStart");
  PLP_SYM(GroupEnd, "ncclGroupEnd");
  PLP_SYM(GetErrorString, "ncclGetErrorString");
#undef PLP_SYM
  g_nccl = a;
}

static const NcclApi* nccl() {
  std::call_once(g_nccl_once, load_nccl);
  return g_nccl.h && g_nccl.GetErrorString ? &g_nccl : nullptr;
}

#define PLP_NCCL(x)                                                                      \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      return set_error(PLP_ERR_NCCL, "%s: %s", #x, nccl()->GetErrorString(r_));          \
  } while (0)

static ncclComm_t comm_of(const plp_ctx* ctx) { return reinterpret_cast<ncclComm_t>(ctx->comm); }

plp_status comm_init(plp_ctx* ctx, int rank, int world, const void* id) {
  ctx->rank = rank;
  ctx->world = world;
  if (!id) {
    if (world != 1) return set_error(PLP_ERR_ARG, "world > 1 needs an NCCL unique id");
    return PLP_OK;
  }
  const NcclApi* api = nccl();
  if (!api) return set_error(PLP_ERR_NCCL, "%s", g_nccl_err.c_str());
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  PLP_NCCL(api->CommInitRank(&c, world, uid, rank));
  ctx->comm = c;
  // side stream + events: halo exchanges run there while the interior tiles compute
  PLP_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  PLP_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  PLP_CUDA(cudaEventCreateWithFlags(&ctx->ev_halo, cudaEventDisableTiming));
  return PLP_OK;
}

void comm_destroy(plp_ctx* ctx) {
  if (ctx->comm && nccl()) nccl()->CommDestroy(comm_of(ctx));
  ctx->comm = nullptr;
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_halo) cudaEventDestroy(ctx->ev_halo);
  ctx->comm_stream = nullptr;
  ctx->ev_in = ctx->ev_halo = nullptr;
}

// In-place sum over the ranks of `count` doubles (device), on the ctx stream.  No-op without a
// communicator (single rank).
plp_status comm_allreduce(plp_ctx* ctx, double* buf, size_t count) {
  if (!ctx->comm || count == 0) return PLP_OK;
  PLP_NCCL(nccl()->AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm_of(ctx), ctx->stream));
  return PLP_OK;
}

plp_status comm_allreduce_i64(plp_ctx* ctx, int64_t* buf, size_t count) {
  if (!ctx->comm || count == 0) return PLP_OK;
  PLP_NCCL(nccl()->AllReduce(buf, buf, count, ncclInt64, ncclSum, comm_of(ctx), ctx->stream));
  return PLP_OK;
}

__global__ void gather_rows_bytes_kernel(int64_t m, int row_words, const int32_t* __restrict__ idx,
                                         const uint32_t* __restrict__ X, uint32_t* __restrict__ out) {
  const int64_t total = m * row_words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / row_words, c = t - r * row_words;
    out[t] = X[(int64_t)idx[r] * row_words + c];
  }
}

// Halo exchange of an n_cols x row_bytes array X (rows [0, n_own) owned, [n_own, n_cols) halo):
// pack the rows each peer needs (one gather launch), then grouped NCCL send/recv; a received
// peer slice lands in place in X's halo rows (the halo is sorted and ownership ranges are
// contiguous, so each peer's rows form one slice).
plp_status halo_exchange_bytes(plp_ctx* ctx, const plp_graph* g, void* X, int row_bytes, cudaStream_t stream) {
  const plp_dist* d = g->dist;
  if (!d || !ctx->comm) return PLP_OK;
  if (!stream) stream = ctx->stream;
  if (row_bytes % 4) return set_error(PLP_ERR_ARG, "halo rows must be a multiple of 4 bytes");
  const size_t need = (size_t)d->total_send * (size_t)row_bytes;
  if (need > d->sendbuf_bytes)
    return set_error(PLP_ERR_SHAPE, "halo rows of %d bytes exceed the send buffer (PLP_MAX_K doubles)", row_bytes);
  const int words = row_bytes / 4;
  if (d->total_send > 0) {
    const int64_t total = d->total_send * words;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)ctx->num_sms * 8);
    gather_rows_bytes_kernel<<<grid, 256, 0, stream>>>(d->total_send, words, d->send_idx,
                                                            static_cast<const uint32_t*>(X),
                                                            static_cast<uint32_t*>(d->sendbuf));
    PLP_LAUNCH_CHECK("gather_rows_bytes_kernel");
  }
  const NcclApi* api = nccl();
  char* xb = static_cast<char*>(X);
  const char* sb = static_cast<const char*>(d->sendbuf);
  PLP_NCCL(api->GroupStart());
  for (int q = 0; q < ctx->world; ++q) {
    if (d->send_cnt[q] > 0)
      PLP_NCCL(api->Send(sb + (size_t)d->send_off[q] * row_bytes, (size_t)d->send_cnt[q] * words,
                         ncclUint32, q, comm_of(ctx), stream));
    if (d->recv_cnt[q] > 0)
      PLP_NCCL(api->Recv(xb + (size_t)(d->n_own + d->recv_off[q]) * row_bytes,
                         (size_t)d->recv_cnt[q] * words, ncclUint32, q, comm_of(ctx), stream));
  }
  PLP_NCCL(api->GroupEnd());
  return PLP_OK;
}

}  // namespace plp

using namespace plp;

extern "C" plp_status plp_get_nccl_unique_id(void* out128) {
  if (!out128) return set_error(PLP_ERR_ARG, "out is null");
  const NcclApi* api = nccl();
  if (!api) return set_error(PLP_ERR_NCCL, "%s", g_nccl_err.c_str());
  ncclUniqueId id;
  PLP_NCCL(api->GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return PLP_OK;
}

extern "C" plp_status plp_ctx_comm_info(const plp_ctx* ctx, int* rank, int* world, int* has_comm) {
  if (!ctx) return set_error(PLP_ERR_ARG, "ctx is null");
  if (rank) *rank = ctx->rank;
  if (world) *world = ctx->world;
  if (has_comm) *has_comm = ctx->comm != nullptr;
  return PLP_OK;
}

extern "C" plp_status plp_allreduce_sum(plp_ctx* ctx, double* buf, int64_t count) {
  PLP_NVTX("plp_allreduce_sum");
  if (!ctx || (!buf && count > 0) || count < 0) return set_error(PLP_ERR_ARG, "bad argument");
  return comm_allreduce(ctx, buf, (size_t)count);
}

extern "C" plp_status plp_halo_exchange(plp_ctx* ctx, const plp_graph* g, int row_bytes, void* X) {
  PLP_NVTX("plp_halo_exchange");
  if (!ctx || !g || !X || row_bytes <= 0) return set_error(PLP_ERR_ARG, "bad argument");
  if (g->ctx != ctx) return set_error(PLP_ERR_ARG, "graph belongs to another ctx");
  return halo_exchange_bytes(ctx, g, X, row_bytes);
}

// Host part of the plan: the per-peer slices of this rank's sorted halo (owner by the ranks' row
// bounds).  Pure host code (tests/test_dist_gloo.py exercises it with gloo on CPU).
extern "C" plp_status plp_dist_recv_plan(int world, const int64_t* bounds, int64_t n_halo,
                                         const int64_t* halo, int64_t* recv_off, int64_t* recv_cnt) {
  if (world < 1 || !bounds || (n_halo > 0 && !halo) || !recv_off || !recv_cnt)
    return set_error(PLP_ERR_ARG, "bad argument");
  for (int q = 0; q < world; ++q) {
    if (bounds[q + 1] < bounds[q]) return set_error(PLP_ERR_ARG, "bounds not monotone");
    const int64_t* b = std::lower_bound(halo, halo + n_halo, bounds[q]);
    const int64_t* e = std::lower_bound(halo, halo + n_halo, bounds[q + 1]);
    recv_off[q] = b - halo;
    recv_cnt[q] = e - b;
  }
  int64_t tot = 0;
  for (int q = 0; q < world; ++q) tot += recv_cnt[q];
  if (tot != n_halo) return set_error(PLP_ERR_ARG, "halo column outside [bounds[0], bounds[world])");
  return PLP_OK;
}

extern "C" plp_status plp_create_graph_dist(plp_ctx* ctx, int64_t n_global, int64_t row_begin,
                                            int64_t row_end, const int64_t* row_ptr, const int32_t* col,
                                            const double* w, uint32_t flags, plp_graph** out) {
  PLP_NVTX("plp_create_graph_dist");
  if (!ctx || !row_ptr || !out || row_begin < 0 || row_end < row_begin || row_end > n_global)
    return set_error(PLP_ERR_ARG, "bad argument");
  *out = nullptr;
  const int world = ctx->world, rank = ctx->rank;
  if (world > 1 && !ctx->comm) return set_error(PLP_ERR_ARG, "world > 1 without a communicator");
  const int64_t n_own = row_end - row_begin;
  const int64_t base = row_ptr[0], nnz = row_ptr[n_own] - base;
  for (int64_t e = 0; e < nnz; ++e)
    if (col[e] < 0 || col[e] >= n_global) return set_error(PLP_ERR_GRAPH, "column %d outside [0, %lld)", col[e], (long long)n_global);
  // halo: sorted distinct columns outside [row_begin, row_end); local column ids
  std::vector<int64_t> halo;
  for (int64_t e = 0; e < nnz; ++e)
    if (col[e] < row_begin || col[e] >= row_end) halo.push_back(col[e]);
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  const int64_t n_halo = (int64_t)halo.size();
  std::vector<int32_t> col_loc((size_t)std::max<int64_t>(nnz, 1));
  for (int64_t e = 0; e < nnz; ++e) {
    const int64_t j = col[e];
    col_loc[e] = (j >= row_begin && j < row_end)
                     ? (int32_t)(j - row_begin)
                     : (int32_t)(n_own + (std::lower_bound(halo.begin(), halo.end(), j) - halo.begin()));
  }
  std::vector<int64_t> rp((size_t)n_own + 1);
  for (int64_t i = 0; i <= n_own; ++i) rp[i] = row_ptr[i] - base;

  plp_dist* d = new (std::nothrow) plp_dist();
  if (!d) return set_error(PLP_ERR_OOM, "host allocation failed");
  d->n_global = n_global;
  d->row_begin = row_begin;
  d->row_end = row_end;
  d->n_own = n_own;
  d->n_halo = n_halo;
  d->send_off.assign(world, 0);
  d->send_cnt.assign(world, 0);
  d->recv_off.assign(world, 0);
  d->recv_cnt.assign(world, 0);
  d->bounds.assign(world + 1, 0);
  plp_status st = PLP_OK;
  int64_t* dbuf = nullptr;
  auto fail = [&](plp_status s) {
    cudaFree(dbuf);
    delete d;
    return s;
  };
  if (ctx->comm) {
    // (1) everybody's row range, (2) the request-count matrix, (3) the request lists
    const NcclApi* api = nccl();
    const size_t cap = (size_t)std::max<int64_t>(2 * world + 2, 8);
    if (cudaMalloc(&dbuf, sizeof(int64_t) * cap * (world + 1)) != cudaSuccess)
      return fail(set_error(PLP_ERR_OOM, "cudaMalloc(plan scratch)"));
    int64_t mine[2] = {row_begin, row_end};
    std::vector<int64_t> all((size_t)2 * world);
    if (cudaMemcpy(dbuf, mine, sizeof(mine), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_error(PLP_ERR_CUDA, "plan copy"));
    ncclResult_t r = api->AllGather(dbuf, dbuf + 2, 2, ncclInt64, comm_of(ctx), ctx->stream);
    if (r != ncclSuccess) return fail(set_error(PLP_ERR_NCCL, "ncclAllGather(bounds): %s", api->GetErrorString(r)));
    if (cudaMemcpyAsync(all.data(), dbuf + 2, sizeof(int64_t) * 2 * world, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return fail(set_error(PLP_ERR_CUDA, "plan copy"));
    for (int q = 0; q < world; ++q) {
      if (all[2 * q] != (q == 0 ? 0 : all[2 * q - 1]))
        return fail(set_error(PLP_ERR_ARG, "row ranges are not contiguous in rank order (rank %d)", q));
      d->bounds[q] = all[2 * q];
    }
    d->bounds[world] = all[2 * world - 1];
    if (d->bounds[world] != n_global) return fail(set_error(PLP_ERR_ARG, "row ranges do not cover n_global"));
    st = plp_dist_recv_plan(world, d->bounds.data(), n_halo, halo.data(), d->recv_off.data(), d->recv_cnt.data());
    if (st) return fail(st);
    if (d->recv_cnt[rank] != 0) return fail(set_error(PLP_ERR_ARG, "halo row owned by this rank"));
    // request-count matrix M[r][q] = rows rank r needs from rank q
    std::vector<int64_t> M((size_t)world * world);
    cudaFree(dbuf);
    dbuf = nullptr;
    if (cudaMalloc(&dbuf, sizeof(int64_t) * (size_t)world * (world + 1)) != cudaSuccess)
      return fail(set_error(PLP_ERR_OOM, "cudaMalloc(plan scratch)"));
    if (cudaMemcpy(dbuf, d->recv_cnt.data(), sizeof(int64_t) * world, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_error(PLP_ERR_CUDA, "plan copy"));
    r = api->AllGather(dbuf, dbuf + world, world, ncclInt64, comm_of(ctx), ctx->stream);
    if (r != ncclSuccess) return fail(set_error(PLP_ERR_NCCL, "ncclAllGather(counts): %s", api->GetErrorString(r)));
    if (cudaMemcpyAsync(M.data(), dbuf + world, sizeof(int64_t) * world * world, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return fail(set_error(PLP_ERR_CUDA, "plan copy"));
    int64_t tot_send = 0;
    for (int q = 0; q < world; ++q) {
      d->send_off[q] = tot_send;
      d->send_cnt[q] = M[(size_t)q * world + rank];
      tot_send += d->send_cnt[q];
    }
    d->total_send = tot_send;
    // request lists: my halo slice owned by q goes to q; q's request for my rows comes back
    cudaFree(dbuf);
    dbuf = nullptr;
    const size_t nreq = (size_t)std::max<int64_t>(n_halo, 1), nsend = (size_t)std::max<int64_t>(tot_send, 1);
    if (cudaMalloc(&dbuf, sizeof(int64_t) * (nreq + nsend)) != cudaSuccess)
      return fail(set_error(PLP_ERR_OOM, "cudaMalloc(plan scratch)"));
    if (n_halo && cudaMemcpy(dbuf, halo.data(), sizeof(int64_t) * n_halo, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(set_error(PLP_ERR_CUDA, "plan copy"));
    int64_t* rq = dbuf + nreq;
    api->GroupStart();
    for (int q = 0; q < world; ++q) {
      if (d->recv_cnt[q] > 0) api->Send(dbuf + d->recv_off[q], d->recv_cnt[q], ncclInt64, q, comm_of(ctx), ctx->stream);
      if (d->send_cnt[q] > 0) api->Recv(rq + d->send_off[q], d->send_cnt[q], ncclInt64, q, comm_of(ctx), ctx->stream);
    }
    r = api->GroupEnd();
    if (r != ncclSuccess) return fail(set_error(PLP_ERR_NCCL, "request exchange: %s", api->GetErrorString(r)));
    std::vector<int64_t> req((size_t)nsend);
    if (cudaMemcpyAsync(req.data(), rq, sizeof(int64_t) * nsend, cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
        cudaStreamSynchronize(ctx->stream) != cudaSuccess)
      return fail(set_error(PLP_ERR_CUDA, "plan copy"));
    std::vector<int32_t> sidx((size_t)nsend, 0);
    for (int64_t t = 0; t < tot_send; ++t) {
      if (req[t] < row_begin || req[t] >= row_end) return fail(set_error(PLP_ERR_ARG, "peer requested a row this rank does not own"));
      sidx[t] = (int32_t)(req[t] - row_begin);
    }
    cudaFree(dbuf);
    dbuf = nullptr;
    // send buffer for rows up to PLP_MAX_K doubles, allocated here so that no exchange allocates
    // (the calls may be captured into CUDA graphs)
    d->sendbuf_bytes = nsend * PLP_MAX_K * sizeof(double);
    if (cudaMalloc(&d->send_idx, sizeof(int32_t) * nsend) != cudaSuccess ||
        cudaMemcpy(d->send_idx, sidx.data(), sizeof(int32_t) * nsend, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMalloc(&d->sendbuf, d->sendbuf_bytes) != cudaSuccess) {
      cudaFree(d->send_idx);
      cudaFree(d->sendbuf);
      return fail(set_error(PLP_ERR_OOM, "cudaMalloc(send_idx / sendbuf)"));
    }
  } else {
    if (n_halo) return fail(set_error(PLP_ERR_ARG, "single rank: the graph has columns outside [row_begin, row_end)"));
    d->bounds[0] = 0;
    d->bounds[1] = n_global;
  }
  plp_graph* g = nullptr;
  st = plp_create_graph(ctx, n_own, n_own + n_halo, rp.data(), col_loc.data(), w, flags & ~(uint32_t)PLP_VALIDATE_SYMMETRIC, &g);
  if (st) {
    cudaFree(d->send_idx);
    return fail(st);
  }
  // interior tiles (no column in the halo) first, then the boundary tiles (SURVEY.md §8(e):
  // interior rows compute while the halo is in flight).  PLP_DEBUG_SPLIT=1 also lists every third
  // interior tile as a boundary tile (exercises the two-launch path on one GPU; tests).
  g->dist = d;
  if (g->halo_enc) {
    const int64_t T = PLP_HALO_TILE, nt = (n_own + T - 1) / T;
    std::vector<int32_t> inter, bnd;
    static const bool dbg = getenv("PLP_DEBUG_SPLIT") != nullptr;
    for (int64_t t = 0; t < nt; ++t) {
      const int64_t r0 = t * T, r1 = std::min<int64_t>(n_own, r0 + T);
      bool b = false;
      for (int64_t e = rp[r0]; e < rp[r1] && !b; ++e) b = col_loc[e] >= n_own;
      if (dbg && t % 3 == 1) b = true;
      (b ? bnd : inter).push_back((int32_t)t);
    }
    d->n_interior = (int64_t)inter.size();
    d->n_boundary = (int64_t)bnd.size();
    inter.insert(inter.end(), bnd.begin(), bnd.end());
    if (!inter.empty() &&
        (cudaMalloc(&d->tile_order, sizeof(int32_t) * inter.size()) != cudaSuccess ||
         cudaMemcpy(d->tile_order, inter.data(), sizeof(int32_t) * inter.size(), cudaMemcpyHostToDevice) !=
             cudaSuccess)) {
      plp_destroy_graph(g);
      return set_error(PLP_ERR_OOM, "cudaMalloc(tile order)");
    }
  }
  *out = g;
  return PLP_OK;
}

extern "C" plp_status plp_graph_dist_info(const plp_graph* g, int64_t* n_own, int64_t* n_halo,
                                          int64_t* row_begin, int64_t* send_rows) {
  if (!g) return set_error(PLP_ERR_ARG, "graph is null");
  const plp_dist* d = g->dist;
  if (n_own) *n_own = d ? d->n_own : g->n_rows;
  if (n_halo) *n_halo = d ? d->n_halo : g->n_cols - g->n_rows;
  if (row_begin) *row_begin = d ? d->row_begin : 0;
  if (send_rows) *send_rows = d ? d->total_send : 0;
  return PLP_OK;
}

namespace plp {
void dist_destroy(plp_dist* d) {
  if (!d) return;
  cudaFree(d->tile_order);
  cudaFree(d->send_idx);
  cudaFree(d->sendbuf);
  delete d;
}
}  // namespace plp
