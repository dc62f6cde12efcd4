// C-ABI entry points of the edge path: F_p, EucGrad, EucHessianEta, the
// full-mode epilogue (a6) and RCut (a12).  Kernels: edge_kernel.cuh; power policies: pow64.cuh.
#include <cmath>
#include <cstdlib>

#include "edge_inst.cuh"
#include "plp_internal.h"

namespace plp {

// ---- power-policy dispatch (DESIGN.md §5 "power") ----------------------------------------------
// p - 2 == -m/D (within 4 ulp: the configs' decimal p = 1.8, 1.2, 1.1 are not exact binary
// fractions; the exponent difference is < 1e-16, reading #20) selects the root-Newton policy.
static bool match_root(double p, int D, int* m_out) {
  const double q = p - 2.0;
  const long m = lround(-q * D);
  if (m < 1 || m >= D) return false;
  const double r = -(double)m / D;
  const double ulp = std::nextafter(std::fabs(q), INFINITY) - std::fabs(q);
  if (std::fabs(q - r) > 4.0 * ulp) return false;
  *m_out = (int)m;
  return true;
}

template <class P>
static P base_pol(double p, double eps) {
  P pw{};
  pw.eps = eps;
  pw.eps_bits = __builtin_bit_cast(long long, eps);
  pw.fast_lo = __builtin_bit_cast(long long, std::fmax(eps, 0x1p-120));
  const unsigned lo1 = (unsigned)(pw.fast_lo >> 32) + 1u;
  pw.fast_lo2 = lo1 << 1;
  pw.fast_span2 = (kHiMax - lo1) << 1;
  pw.q = p - 2.0;
  pw.pm1 = p - 1.0;
  pw.s_eps = std::pow(eps, p - 2.0);  // cap(a)^{p-2} for a < eps, as the oracle computes it
  return pw;
}

template <int D, int M>
static PowRoot<D, M> root_pol(double p, double eps) {
  PowRoot<D, M> pw = base_pol<PowRoot<D, M>>(p, eps);
  pw.c1 = (double)M / D;                   // (1 - e)^{-M/D} = 1 + c1 e + c2 e^2 + O(e^3)
  pw.c2 = pw.c1 * (pw.c1 + 1.0) / 2.0;
  return pw;
}

template <class F>
static plp_status with_pow(plp_ctx* ctx, double p, double eps, F&& f) {
  int m = 0;
  if (p == 2.0) return f(base_pol<PowP2>(p, eps));
  if (match_root(p, 2, &m)) return f(root_pol<2, 1>(p, eps));
  if (match_root(p, 5, &m)) {
    switch (m) {
      case 1: return f(root_pol<5, 1>(p, eps));
      case 2: return f(root_pol<5, 2>(p, eps));
      case 3: return f(root_pol<5, 3>(p, eps));
      default: return f(root_pol<5, 4>(p, eps));
    }
  }
  if (match_root(p, 10, &m)) {
    switch (m) {
      case 1: return f(root_pol<10, 1>(p, eps));
      case 3: return f(root_pol<10, 3>(p, eps));
      case 7: return f(root_pol<10, 7>(p, eps));
      case 9: return f(root_pol<10, 9>(p, eps));
      default: break;  // even m matched D = 5, m = 5 matched D = 2
    }
  }
  PowGeneric pw = base_pol<PowGeneric>(p, eps);
  pw.q64 = 64.0 * (p - 2.0);
  pw.gtab = reinterpret_cast<const PowTables*>(ctx->pow_tables);
  pw.tab = nullptr;
  return f(pw);
}

plp_status launch_edge(plp_ctx* ctx, const EdgeArgs& a, int* grid) {
  return with_pow(ctx, a.p, a.eps,
                  [&](const auto& pw) -> plp_status { return launch_edge_pol(ctx, a, pw, grid); });
}

static plp_status launch_epilogue(plp_ctx* ctx, const EpiArgs& a, double eps) {
  return with_pow(ctx, a.p, eps,
                  [&](const auto& pw) -> plp_status { return launch_epi_pol(ctx, a, pw); });
}

// ---- fixed-order reduction of CTA partials ------------------------------------------------------
// One warp per output sum: lane l adds CTAs l, l+32, ... in order, then a fixed xor-tree.
__global__ void __launch_bounds__(1024) edge_finalize_kernel(int grid, int k, const double* part,
                                                             double* AB_out, double* dots_out,
                                                             double* F) {
  __shared__ double sAB[2 * PLP_MAX_K];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = warp; t < 4 * k; t += (blockDim.x >> 5)) {
    const int q = t / k, cl = t % k;
    double s = 0.0;
    for (int b = lane; b < grid; b += 32) s += part[((int64_t)b * 4 + q) * k + cl];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (q < 2) {
        sAB[q * k + cl] = s;
        if (AB_out) AB_out[q * k + cl] = s;
      } else if (dots_out) {
        dots_out[(q - 2) * k + cl] = s;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && F) {
    double f = 0.0;
    for (int l = 0; l < k; ++l) f += sAB[l] / sAB[k + l];
    *F = f;
  }
}

plp_status launch_edge_finalize(plp_ctx* ctx, int grid, int k, const double* partials,
                                double* AB_out, double* dots_out, double* F) {
  edge_finalize_kernel<<<1, 1024, 0, ctx->stream>>>(grid, k, partials, AB_out, dots_out, F);
  PLP_LAUNCH_CHECK("edge_finalize_kernel");
  return PLP_OK;
}

__global__ void objective_from_ab_kernel(int k, const double* AB, double* F) {
  if (threadIdx.x == 0) {
    double f = 0.0;
    for (int l = 0; l < k; ++l) f += AB[l] / AB[k + l];
    *F = f;
  }
}

// ---- RCut (a12): per-CTA cut/size partials by label, fixed-order --------------------------------
// One thread per row (32 rows in flight per warp: the row_ptr -> col -> label chain is latency-bound);
// per cluster c the warp sums its rows' cuts with a shuffle tree and counts them with a ballot
// (lane c keeps cluster c), then the CTA's warps are added in order.  No atomics, fixed order.
constexpr int kRcutThreads = 256, kRcutLanes = 1;
__global__ void __launch_bounds__(kRcutThreads) rcut_kernel(int64_t n, const int32_t* __restrict__ rp,
                                                           const int32_t* __restrict__ col,
                                                           const double* __restrict__ w, int K,
                                                           const int32_t* __restrict__ lab,
                                                           double* part_cut, int64_t* part_size,
                                                           int* bad) {
  constexpr int NW = kRcutThreads / 32, RPW = 32 / kRcutLanes;
  __shared__ double s_cut[NW][PLP_MAX_K];
  __shared__ int64_t s_cnt[NW][PLP_MAX_K];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int grp = lane / kRcutLanes, gl = lane % kRcutLanes;
  double acc_cut = 0.0;  // lane c < K: cluster c
  int64_t acc_cnt = 0;
  const int64_t steps = (n + RPW - 1) / RPW;
  const int64_t tw = (int64_t)gridDim.x * NW, wid = (int64_t)blockIdx.x * NW + warp;
  const int64_t s0 = steps * wid / tw, s1 = steps * (wid + 1) / tw;
  for (int64_t st = s0; st < s1; ++st) {
    const int64_t i = st * RPW + grp;
    int li = -1;
    double cut = 0.0;
    if (i < n) {
      li = __ldg(lab + i);
      if (gl == 0 && (li < 0 || li >= K)) atomicExch(bad, 1);
      const int e1 = __ldg(rp + i + 1);
      for (int e = __ldg(rp + i) + gl; e < e1; e += kRcutLanes)
        if (__ldg(lab + __ldg(col + e)) != li) cut += __ldg(w + e);
    }
#pragma unroll
    for (int o = kRcutLanes / 2; o > 0; o >>= 1) cut += __shfl_xor_sync(0xffffffffu, cut, o);
    const bool lead = gl == 0 && i < n;
    for (int c = 0; c < K; ++c) {
      double v = (lead && li == c) ? cut : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      const int cnt = __popc(__ballot_sync(0xffffffffu, lead && li == c));
      if (lane == c) {
        acc_cut += v;
        acc_cnt += cnt;
      }
    }
  }
  if (lane < K) {
    s_cut[warp][lane] = acc_cut;
    s_cnt[warp][lane] = acc_cnt;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double c = 0.0;
    int64_t m = 0;
    for (int q = 0; q < NW; ++q) {
      c += s_cut[q][threadIdx.x];
      m += s_cnt[q][threadIdx.x];
    }
    part_cut[(int64_t)blockIdx.x * K + threadIdx.x] = c;
    part_size[(int64_t)blockIdx.x * K + threadIdx.x] = m;
  }
}

// cut / sizes per cluster (one warp per cluster, lanes over the CTAs, xor tree), then RCut
__global__ void __launch_bounds__(1024) rcut_finalize_kernel(int grid, int K, const double* part_cut,
                                                             const int64_t* part_size, double* cut,
                                                             int64_t* sizes, double* rcut) {
  __shared__ double s_c[PLP_MAX_K];
  __shared__ int64_t s_n[PLP_MAX_K];
  const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (c < K) {
    double sc = 0.0;
    int64_t sn = 0;
    for (int b = lane; b < grid; b += 32) {
      sc += part_cut[(int64_t)b * K + c];
      sn += part_size[(int64_t)b * K + c];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sc += __shfl_xor_sync(0xffffffffu, sc, o);
      sn += __shfl_xor_sync(0xffffffffu, sn, o);
    }
    if (lane == 0) {
      s_c[c] = sc;
      s_n[c] = sn;
      if (cut) cut[c] = sc;
      if (sizes) sizes[c] = sn;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && rcut) {
    double r = 0.0;
    for (int q = 0; q < K; ++q) r += (s_n[q] > 0) ? s_c[q] / (double)s_n[q] : NAN;
    *rcut = r;
  }
}

}  // namespace plp

using namespace plp;

static EdgeArgs graph_args(const plp_graph* g) {
  EdgeArgs a{};
  a.need_ab = 1;
  a.n_rows = g->n_rows;
  a.n_cols = g->n_cols;
  a.rp = g->rp;
  a.sched = g->sched;
  a.col = g->col;
  a.w = g->w;
  a.max_chunk_nnz = g->max_chunk_nnz;
  a.halo_enc = g->halo_enc;
  a.halo_ext = g->halo_ext;
  a.halo_ext_cap = g->halo_ext_cap;
  a.halo_nnz_cap = g->halo_nnz_cap;
  a.nlow = g->nlow;
  a.sched_up = g->sched_up;
  a.upper_ok = g->upper_ok ? 1 : 0;
#ifdef PLP_DEBUG_LDX
  a.ldx = PLP_DEBUG_LDX;  // layout experiments only (compile-time)
#endif
  return a;
}

static plp_status check_graph_call(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                   double p, double eps) {
  if (!ctx || !g || !U) return set_error(PLP_ERR_ARG, "null ctx/graph/U");
  if (g->ctx != ctx) return set_error(PLP_ERR_ARG, "graph belongs to another ctx");
  plp_status st = check_k(k);
  if (st) return st;
  return check_p(p, eps);
}

// Multi-rank graph on a ctx with a communicator: the calls below exchange halo rows and
// all-reduce their partial sums (on P ranks each call is collective).
static bool collective(const plp_ctx* ctx, const plp_graph* g) { return ctx->comm && g->dist; }
static plp_status exchange(plp_ctx* ctx, const plp_graph* g, const double* X, int k) {
  // the halo rows [n_own, n_cols) of X are library-written slots (plp_create_graph_dist)
  return halo_exchange_bytes(ctx, g, const_cast<double*>(X), k * (int)sizeof(double));
}

// One edge pass of a collective call with its halo exchange (arrays xU, xE: nullptr = not needed).
// With interior and boundary tiles (plp_dist::tile_order) and the halo kernel, the exchange runs on
// the context's comm stream while the interior tiles compute; the boundary tiles follow once the
// halo has landed.  Partial sums of the two launches are consecutive CTA blocks (*grid = both).
static plp_status overlapped_pass(plp_ctx* ctx, const plp_graph* g, const EdgeArgs& a, const double* xU,
                                  const double* xE, int* grid) {
  const plp_dist* d = g->dist;
  const int k = a.k;
  plp_status st;
  const bool split = d && ctx->comm && ctx->comm_stream && d->tile_order && d->n_interior > 0 &&
                     d->n_boundary > 0 && (xU || xE);
  if (!split) {
    if (xU && (st = exchange(ctx, g, xU, k))) return st;
    if (xE && (st = exchange(ctx, g, xE, k))) return st;
    return launch_edge(ctx, a, grid);
  }
  PLP_CUDA(cudaEventRecord(ctx->ev_in, ctx->stream));  // U / eta written by the caller's stream
  PLP_CUDA(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_in, 0));
  if (xU && (st = halo_exchange_bytes(ctx, g, const_cast<double*>(xU), k * 8, ctx->comm_stream))) return st;
  if (xE && (st = halo_exchange_bytes(ctx, g, const_cast<double*>(xE), k * 8, ctx->comm_stream))) return st;
  PLP_CUDA(cudaEventRecord(ctx->ev_halo, ctx->comm_stream));
  EdgeArgs ai = a;
  ai.tile_list = d->tile_order;
  ai.tile_begin = 0;
  ai.tile_count = d->n_interior;
  int g1 = 0, g2 = 0;
  st = launch_edge(ctx, ai, &g1);
  if (st == PLP_ERR_SHAPE) {  // the halo kernel does not apply (k, alignment): exchange, then one pass
    PLP_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
    return launch_edge(ctx, a, grid);
  }
  if (st) return st;
  PLP_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_halo, 0));
  EdgeArgs ab = ai;
  ab.tile_begin = d->n_interior;
  ab.tile_count = d->n_boundary;
  ab.partials = a.partials + (int64_t)g1 * 4 * k;
  if ((st = launch_edge(ctx, ab, &g2))) return st;
  *grid = g1 + g2;
  return PLP_OK;
}

extern "C" plp_status plp_edge_pass(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                    const double* eta, double p, double eps, const double* AB_in,
                                    double* AB_out, double* dots_out, double* G, double* Hv) {
  PLP_NVTX("plp_edge_pass");
  plp_status st = check_graph_call(ctx, g, k, U, p, eps);
  if (st) return st;
  if (!AB_in && (G || Hv || dots_out))
    return set_error(PLP_ERR_ARG, "G/Hv/dots need AB_in (the global A, B at U)");
  if ((Hv || dots_out) && !eta) return set_error(PLP_ERR_ARG, "Hv/dots need eta");
  EdgeArgs a = graph_args(g);
  a.k = k;
  a.U = U;
  a.eta = (Hv || dots_out) ? eta : nullptr;
  a.AB = AB_in;
  a.G = G;
  a.Hv = Hv;
  a.p = p;
  a.eps = Hv ? eps : kNoCap;  // the cap only enters the Hessian weights (reading #6)
  a.partials = ctx->partials;
  a.want_dots = dots_out != nullptr;
  int grid = 0;
  st = launch_edge(ctx, a, &grid);
  if (st) return st;
  if (AB_out || dots_out) return launch_edge_finalize(ctx, grid, k, ctx->partials, AB_out, dots_out, nullptr);
  return PLP_OK;
}

extern "C" plp_status plp_objective_from_ab(plp_ctx* ctx, int k, const double* AB, double* F) {
  if (!ctx || !AB || !F) return set_error(PLP_ERR_ARG, "null argument");
  plp_status st = check_k(k);
  if (st) return st;
  objective_from_ab_kernel<<<1, 32, 0, ctx->stream>>>(k, AB, F);
  PLP_LAUNCH_CHECK("objective_from_ab_kernel");
  return PLP_OK;
}

extern "C" plp_status plp_full_epilogue(plp_ctx* ctx, int64_t n_rows, int k, const double* U,
                                        double p, const double* AB, const double* dots,
                                        const double* G, double* Hv) {
  if (!ctx || !U || !AB || !dots || !G || !Hv) return set_error(PLP_ERR_ARG, "null argument");
  plp_status st = check_k(k);
  if (st) return st;
  st = check_p(p, 1.0);
  if (st) return st;
  if (n_rows <= 0) return PLP_OK;
  EpiArgs e{n_rows, k, U, p, AB, dots, G, Hv};
  // The epilogue needs phi_p(u) only (no curvature): the cap value is irrelevant, pass 1.
  return launch_epilogue(ctx, e, kNoCap);  // needs phi_p(u) only: no curvature cap
}

// scratch layout (doubles): [0, 2K) AB of an objective pass, [2K, 4K) dots, [4K, 6K) AB recomputed
// by a fused pass (when the caller passes no AB_out)
static double* scratch_ab(plp_ctx* ctx) { return ctx->scratch; }
static double* scratch_dots(plp_ctx* ctx) { return ctx->scratch + 2 * PLP_MAX_K; }
static double* scratch_ab2(plp_ctx* ctx) { return ctx->scratch + 4 * PLP_MAX_K; }

extern "C" plp_status plp_fgrad(plp_ctx* ctx, const plp_graph* g, int k, const double* U, double p,
                                double* F, double* AB_out, double* G) {
  PLP_NVTX("plp_fgrad");
  plp_status st = check_graph_call(ctx, g, k, U, p, 1.0);
  if (st) return st;
  const bool coll = collective(ctx, g);
  if (coll && (st = exchange(ctx, g, U, k))) return st;  // U halo (a new iterate)
  double* ab = AB_out ? AB_out : scratch_ab(ctx);
  EdgeArgs a = graph_args(g);
  a.k = k;
  a.U = U;
  a.p = p; a.eps = kNoCap; a.partials = ctx->partials;  // F and G never use the cap
  int grid = 0;
  st = launch_edge(ctx, a, &grid);  // objective pass
  if (st) return st;
  st = launch_edge_finalize(ctx, grid, k, ctx->partials, ab, nullptr, coll ? nullptr : F);
  if (st) return st;
  if (coll) {  // global A, B, then F = sum A / B
    if ((st = comm_allreduce(ctx, ab, 2 * (size_t)k))) return st;
    if (F && (st = plp_objective_from_ab(ctx, k, ab, F))) return st;
  }
  if (G) {
    EdgeArgs b = a;
    b.AB = ab;
    b.G = G;
    st = launch_edge(ctx, b, &grid);  // gradient pass with the fresh A, B
    if (st) return st;
  }
  return PLP_OK;
}

extern "C" plp_status plp_hessvec(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                  const double* eta, double p, const double* AB_in, int mode,
                                  double eps, const double* G_in, double* Hv) {
  PLP_NVTX("plp_hessvec");
  plp_status st = check_graph_call(ctx, g, k, U, p, eps);
  if (st) return st;
  const bool u_current = (mode & PLP_U_HALO_CURRENT) != 0;
  mode &= ~PLP_U_HALO_CURRENT;
  if (!eta || !AB_in || !Hv) return set_error(PLP_ERR_ARG, "hessvec needs eta, AB_in and Hv");
  if (mode != PLP_HESS_SPARSE && mode != PLP_HESS_FULL) return set_error(PLP_ERR_ARG, "bad mode");
  if (mode == PLP_HESS_FULL && !G_in)
    return set_error(PLP_ERR_ARG, "full mode needs G_in (the Euclidean gradient at U)");
  const bool full = mode == PLP_HESS_FULL;
  const bool coll = collective(ctx, g);
  if (!coll && full) {
    st = plp_edge_pass(ctx, g, k, U, eta, p, eps, AB_in, nullptr, scratch_dots(ctx), nullptr, Hv);
    if (st) return st;
  } else if (!coll) {  // sparse: a Hessian-vector-only pass (no gradient sum, no A, B partials)
    EdgeArgs a = graph_args(g);
    a.k = k; a.U = U; a.eta = eta; a.AB = AB_in; a.Hv = Hv; a.p = p; a.eps = eps;
    a.partials = ctx->partials;
    a.need_ab = 0;
    int grid = 0;
    return launch_edge(ctx, a, &grid);
  } else {
    EdgeArgs a = graph_args(g);
    a.k = k; a.U = U; a.eta = eta; a.AB = AB_in; a.Hv = Hv; a.p = p; a.eps = eps;
    a.partials = ctx->partials;
    a.want_dots = full;
    a.need_ab = 0;
    int grid = 0;
    if ((st = overlapped_pass(ctx, g, a, u_current ? nullptr : U, eta, &grid))) return st;
    if (!full) return PLP_OK;
    if ((st = launch_edge_finalize(ctx, grid, k, ctx->partials, nullptr, scratch_dots(ctx), nullptr))) return st;
    if ((st = comm_allreduce(ctx, scratch_dots(ctx), 2 * (size_t)k))) return st;
  }
  return plp_full_epilogue(ctx, g->n_rows, k, U, p, AB_in, scratch_dots(ctx), G_in, Hv);
}

namespace plp {
// The fused tCG's Hessian-vector product with pass A folded in (tcg.cu): a rank-local sparse
// plp_hessvec whose halo pass also writes pass A's CTA partials when it can (*used; *grid = the
// number of partial columns), else a plain one (*used = false: the caller runs pass A).
plp_status hessvec_gram(plp_ctx* ctx, const plp_graph* g, int k, const double* U, const double* eta,
                        double p, const double* AB_in, double eps, const double* S8, double* Hv,
                        int* grid, bool* used) {
  *used = false;
  plp_status st = check_graph_call(ctx, g, k, U, p, eps);
  if (st) return st;
  if (!eta || !AB_in || !Hv || !S8) return set_error(PLP_ERR_ARG, "hessvec_gram: null argument");
  if (collective(ctx, g)) return set_error(PLP_ERR_ARG, "hessvec_gram is rank-local");
  EdgeArgs a = graph_args(g);
  a.k = k; a.U = U; a.eta = eta; a.AB = AB_in; a.Hv = Hv; a.p = p; a.eps = eps;
  a.partials = ctx->partials;
  a.need_ab = 0;
  a.gram_S = S8;
  int gram_used = 0;
  a.gram_used = &gram_used;
  if ((st = launch_edge(ctx, a, grid))) return st;
  *used = gram_used != 0;
  return PLP_OK;
}
}  // namespace plp

extern "C" plp_status plp_fgrad_hessvec(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                        const double* eta, double p, const double* AB_in, int mode,
                                        double eps, double* F, double* AB_out, double* G,
                                        double* Hv) {
  PLP_NVTX("plp_fgrad_hessvec");
  plp_status st = check_graph_call(ctx, g, k, U, p, eps);
  if (st) return st;
  const bool u_current = (mode & PLP_U_HALO_CURRENT) != 0;
  mode &= ~PLP_U_HALO_CURRENT;
  if (mode != PLP_HESS_SPARSE && mode != PLP_HESS_FULL) return set_error(PLP_ERR_ARG, "bad mode");
  if (Hv && !eta) return set_error(PLP_ERR_ARG, "Hv needs eta");
  const bool full = mode == PLP_HESS_FULL && Hv != nullptr;
  if (full && !G) return set_error(PLP_ERR_ARG, "full mode needs the G output buffer");
  const bool coll = collective(ctx, g);
  const double* xU = coll && !u_current ? U : nullptr;  // halo exchanges this call still owes
  const double* xE = coll && Hv ? eta : nullptr;
  if (!AB_in) {  // objective pass first (two edge passes)
    if (xU && (st = exchange(ctx, g, U, k))) return st;
    xU = nullptr;
    st = plp_edge_pass(ctx, g, k, U, nullptr, p, eps, nullptr, scratch_ab(ctx), nullptr, nullptr,
                       nullptr);
    if (st) return st;
    if (coll && (st = comm_allreduce(ctx, scratch_ab(ctx), 2 * (size_t)k))) return st;
    AB_in = scratch_ab(ctx);
  }
  EdgeArgs a = graph_args(g);
  a.k = k;
  a.U = U;
  a.eta = Hv ? eta : nullptr;
  a.AB = AB_in; a.G = G; a.Hv = Hv; a.p = p; a.eps = eps; a.partials = ctx->partials;
  a.want_dots = full;
  int grid = 0;
  st = coll ? overlapped_pass(ctx, g, a, xU, xE, &grid) : launch_edge(ctx, a, &grid);
  if (st) return st;
  if (AB_out || full || F) {
    // F and AB_out come from the fused pass's own A', B' (all-reduced over the ranks)
    double* abo = AB_out ? AB_out : scratch_ab2(ctx);
    st = launch_edge_finalize(ctx, grid, k, ctx->partials, abo, full ? scratch_dots(ctx) : nullptr,
                              coll ? nullptr : F);
    if (st) return st;
    if (coll) {
      if ((st = comm_allreduce(ctx, abo, 2 * (size_t)k))) return st;
      if (full && (st = comm_allreduce(ctx, scratch_dots(ctx), 2 * (size_t)k))) return st;
      if (F && (st = plp_objective_from_ab(ctx, k, abo, F))) return st;
    }
  }
  if (full) return plp_full_epilogue(ctx, g->n_rows, k, U, p, AB_in, scratch_dots(ctx), G, Hv);
  return PLP_OK;
}

extern "C" plp_status plp_debug_pow(plp_ctx* ctx, int64_t n, const double* a, double p, double eps,
                                    double* s, double* t) {
  if (!ctx || !a || !s || !t || n < 0) return set_error(PLP_ERR_ARG, "bad argument");
  plp_status st = check_p(p, eps);
  if (st) return st;
  if (n == 0) return PLP_OK;
  return with_pow(ctx, p, eps, [&](const auto& pw) -> plp_status {
    return launch_dbg_pol(ctx, n, a, s, t, pw);
  });
}

__global__ void rcut_ratio_kernel(int K, const double* cut, const int64_t* sizes, double* rcut) {
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int q = 0; q < K; ++q) r += (sizes[q] > 0) ? cut[q] / (double)sizes[q] : NAN;
    *rcut = r;
  }
}

extern "C" plp_status plp_rcut(plp_ctx* ctx, const plp_graph* g, int clusters,
                               const int32_t* labels, double* cut, int64_t* sizes, double* rcut) {
  PLP_NVTX("plp_rcut");
  if (!ctx || !g || !labels) return set_error(PLP_ERR_ARG, "null argument");
  if (clusters < 1 || clusters > PLP_MAX_K) return set_error(PLP_ERR_DOMAIN, "clusters must be in [1, 32]");
  const bool coll = collective(ctx, g);
  plp_status st;
  // multi-rank: the halo rows' labels come from their owners (labels has n_cols entries)
  if (coll && (st = halo_exchange_bytes(ctx, g, const_cast<int32_t*>(labels), (int)sizeof(int32_t)))) return st;
  static const int res = resident_ctas(rcut_kernel, kRcutThreads);
  int grid = ctx->num_sms * res;  // one full wave
  const int64_t want = (g->n_rows + 255) / 256;
  if (grid > want) grid = (int)std::max<int64_t>(1, want);
  if (grid > ctx->max_ctas) grid = ctx->max_ctas;
  double* pc = ctx->partials;
  int64_t* ps = reinterpret_cast<int64_t*>(ctx->partials + (int64_t)ctx->max_ctas * PLP_MAX_K);
  PLP_CUDA(cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
  rcut_kernel<<<grid, kRcutThreads, 0, ctx->stream>>>(g->n_rows, g->rp, g->col, g->w, clusters, labels, pc,
                                              ps, ctx->flag);
  PLP_LAUNCH_CHECK("rcut_kernel");
  if (!coll) {
    rcut_finalize_kernel<<<1, 1024, 0, ctx->stream>>>(grid, clusters, pc, ps, cut, sizes, rcut);
    PLP_LAUNCH_CHECK("rcut_finalize_kernel");
    return PLP_OK;
  }
  // rank-local cut / sizes, summed over the ranks, then the ratio
  double* c = cut ? cut : ctx->scratch + 8 * PLP_MAX_K;
  int64_t* m = sizes ? sizes : ctx->iscratch + 16;
  rcut_finalize_kernel<<<1, 1024, 0, ctx->stream>>>(grid, clusters, pc, ps, c, m, nullptr);
  PLP_LAUNCH_CHECK("rcut_finalize_kernel");
  if ((st = comm_allreduce(ctx, c, clusters))) return st;
  if ((st = comm_allreduce_i64(ctx, m, clusters))) return st;
  if (rcut) {
    rcut_ratio_kernel<<<1, 32, 0, ctx->stream>>>(clusters, c, m, rcut);
    PLP_LAUNCH_CHECK("rcut_ratio_kernel");
  }
  return PLP_OK;
}
