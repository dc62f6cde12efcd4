/*
 * plp.h -- C ABI of libplp: the B200 (sm_100a) hot path of p-spectral clustering on the
 * Grassmann manifold (arxiv 2605.26975, "Nonlinear spectral clustering with C++ GraphBLAS").
 *
 * The entry points follow the paper's statement of the problem:
 *   Eq. (1)  F_p(U) = sum_l sum_{i,j} w_ij |u_i^l - u_j^l|^p / (2 ||u^l||_p^p)
 *   Delta_p, phi_p, ||.||_p
 *   EucGrad, EucHessianEta (Alg. 1)
 *   k-means discretisation
 *   RCut = sum_i cut(C_i, ~C_i)/|C_i|
 * Readings of the paper where it is silent or garbled are listed in DESIGN.md §3 (numbered #1..#19
 * as in SURVEY.md §8(c)); the ones that change numbers are cited at each call below.
 *
 * Conventions (all calls):
 *  - Dense arrays are fp64, contiguous, node-major (row-major) n x k: element (i, l) at [i*k + l].
 *    U, eta, G, Hv, xi, X and every other dense array are DEVICE pointers owned by the caller
 *    (e.g. torch tensors); libplp never frees them.  Small outputs (F, AB, dots, Grams, rcut) are
 *    device pointers too, so no hot call synchronises with the host.  Exceptions are stated.
 *  - libplp owns plp_ctx and plp_graph and everything inside them (device CSR, workspaces).
 *    Hot calls never allocate; all workspace is sized at plp_ctx_create / plp_create_graph.
 *  - Work is enqueued on the ctx's CUDA stream (plp_ctx_set_stream).  On P ranks (a ctx with an
 *    NCCL communicator, plp_ctx_create) each call is collective: every rank passes its own rows
 *    (dense arrays of a plp_create_graph_dist graph carry halo slots the calls fill), and scalar /
 *    k x k outputs (F, AB, dots, Grams) are global -- DESIGN.md §7.  plp_edge_pass and
 *    plp_full_epilogue stay rank-local building blocks.
 *  - 1 <= k <= 32.  p in (1, 2].  eps > 0 when p < 2 (curvature cap, reading #6).
 *  - Every call returns a plp_status; plp_last_error() gives a thread-local message.  No C++
 *    exception crosses the ABI.  Results are deterministic: every reduction runs in a fixed order
 *    (no floating-point atomics), so two identical calls are bitwise equal on a given device.
 */
#ifndef PLP_H_
#define PLP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PLP_OK = 0,
  PLP_ERR_ARG = 1,        /* null pointer / bad flag / bad size                                   */
  PLP_ERR_SHAPE = 2,      /* size mismatch or beyond a supported limit (e.g. nnz >= 2^31)          */
  PLP_ERR_DOMAIN = 3,     /* p not in (1,2], eps <= 0 with p < 2, k < 1, k > 32    */
  PLP_ERR_GRAPH = 4,      /* asymmetric, diagonal entry, w <= 0, unsorted/duplicate or
                             out-of-range column */
  PLP_ERR_DEGENERATE = 5, /* B_l = 0 (zero column)    */
  PLP_ERR_RANK = 6,       /* Cholesky of Y^T Y failed: the retraction step must be rejected        */
  PLP_ERR_NONFINITE = 7,  /* non-finite input or result detected                                    */
  PLP_ERR_CUDA = 8,       /* CUDA runtime error (message in plp_last_error)                        */
  PLP_ERR_OOM = 9,        /* device allocation failed                                               */
  PLP_ERR_EMPTY = 10,     /* empty cluster where the metric needs |C| > 0    */
  PLP_ERR_NCCL = 11       /* NCCL missing or an NCCL call failed (message in plp_last_error)       */
} plp_status;

enum { PLP_HESS_SPARSE = 0, PLP_HESS_FULL = 1 };          /* reading #5 */
/* OR-ed into `mode` of plp_hessvec / plp_fgrad_hessvec on a multi-rank graph: the halo rows of U
 * are already current (exchanged by an earlier call at the same U, e.g. plp_fgrad), so only the
 * eta halo is exchanged -- the tCG's Hessian-vector products at a fixed iterate.  Ignored on a
 * single-rank graph. */
enum { PLP_U_HALO_CURRENT = 16 };
enum { PLP_VALIDATE = 1u, PLP_VALIDATE_SYMMETRIC = 2u };  /* plp_create_graph flags */
enum { PLP_TILE_ROWS = 80 };  /* default BFS tile of plp_tile_order (three per halo-kernel tile) */
#ifndef PLP_HALO_TILE_ROWS
#define PLP_HALO_TILE_ROWS 240  /* 15 consumer warps x 2 slices of 8 rows: 16 warps per SM with the producer */
#endif
enum { PLP_HALO_TILE = PLP_HALO_TILE_ROWS };  /* rows per tile of the halo-tile edge kernel */

typedef struct plp_ctx plp_ctx;
typedef struct plp_graph plp_graph;

const char* plp_last_error(void);
const char* plp_version(void);
/* Rows per tile of the halo-tile edge kernel (PLP_HALO_TILE); multi-rank row blocks are aligned to
 * it (paper_2605_26975_b200/dist.py).  plp_tile_order takes its own BFS tile size. */
int plp_halo_tile_rows(void);

/* ---------------------------------------------------------------------------------------------- */
/* Context                                                                                          */
/* ---------------------------------------------------------------------------------------------- */
/* device: CUDA ordinal.  stream: a cudaStream_t (NULL = legacy default stream).  Allocates the
 * ctx workspaces (CTA partials, k x k scratch) on the device.
 * rank, world, nccl_id: one process per GPU.  nccl_id = the 128-byte id from
 * plp_get_nccl_unique_id on rank 0, broadcast by the caller (e.g. torch.distributed); the call is
 * then collective over the `world` ranks and the ctx owns an NCCL communicator: every call below
 * on a graph from plp_create_graph_dist, and every Gram / dot / projection / retraction, is then
 * collective (each rank passes its own rows; scalar and k x k outputs are global).  nccl_id NULL
 * requires world == 1 (single GPU, no communicator).  world == 1 with an id creates a one-rank
 * communicator (the collective code path on one GPU).  PLP_ERR_NCCL if NCCL cannot be loaded. */
plp_status plp_ctx_create(int device, void* stream, int rank, int world, const void* nccl_id,
                          plp_ctx** out);
/* Rank 0: a fresh NCCL unique id (128 bytes) for plp_ctx_create.  Loads NCCL (libnccl.so.2). */
plp_status plp_get_nccl_unique_id(void* out128);
/* rank, world, and whether the ctx holds a communicator. */
plp_status plp_ctx_comm_info(const plp_ctx* ctx, int* rank, int* world, int* has_comm);
/* In-place sum over the ranks of `count` device doubles, on the ctx stream (collective; no-op
 * without a communicator). */
plp_status plp_allreduce_sum(plp_ctx* ctx, double* buf, int64_t count);
plp_status plp_ctx_set_stream(plp_ctx* ctx, void* stream);
plp_status plp_ctx_destroy(plp_ctx* ctx);
/* Number of CTAs the edge kernel launches (the fixed reduction grid); informational. */
plp_status plp_ctx_info(const plp_ctx* ctx, int* num_sms, int* max_ctas);

/* ---------------------------------------------------------------------------------------------- */
/* Host-side graph utilities (no GPU needed; used for setup)                    */
/* ---------------------------------------------------------------------------------------------- */
/* Checks the CSR of rows [0, n_rows) with columns in [0, n_cols): row_ptr monotone with
 * row_ptr[0] = 0, columns strictly increasing per row, no diagonal entry (col == row for
 * row < n_rows), w > 0 and finite.  With symmetric != 0 (requires n_rows == n_cols) also checks
 * w_ij == w_ji bitwise (the paper's undirected graph G(V,E,W)).
 * Returns PLP_ERR_GRAPH with the first offending (i, j) in plp_last_error. */
plp_status plp_validate_csr(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                            const int32_t* col, const double* w, int symmetric);
/* Reverse Cuthill-McKee ordering of a symmetric CSR (n x n): perm[new] = old.  Per connected
 * component (components in order of their lowest-degree / lowest-id start node), BFS from a
 * pseudo-peripheral node with neighbours visited in (degree, id) order; the whole order is then
 * reversed.  Deterministic.  Used so that U_j gathers hit L2. */
plp_status plp_rcm_order(int64_t n, const int64_t* row_ptr, const int32_t* col, int64_t* perm);
/* Tile ordering for the halo-tile edge kernel: RCM sweep, then tiles of `tile`
 * nodes (PLP_TILE_ROWS = 80: three per 240-row halo-kernel tile) grown by BFS along
 * the sweep, the nodes of a tile sorted by decreasing degree.
 * perm[new] = old.  Relabel with plp_permute_csr; U and eta must then use the new order. */
plp_status plp_tile_order(int64_t n, const int64_t* row_ptr, const int32_t* col, int tile,
                          int64_t* perm);
/* Relabels a symmetric CSR: new node a is old node perm[a].  Output arrays are caller-allocated
 * (n+1, nnz, nnz); columns of each output row are sorted. */
plp_status plp_permute_csr(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* w,
                           const int64_t* perm, int64_t* row_ptr_out, int32_t* col_out,
                           double* w_out);
/* Contiguous row-block partition of n rows into `parts` blocks balancing the per-row cost
 * cost_row + cost_nnz * deg(i) (e.g. 32k and 12 bytes): bounds[0] = 0, bounds[parts] = n. */
plp_status plp_partition_rows(int64_t n, const int64_t* row_ptr, int parts, double cost_row,
                              double cost_nnz, int64_t* bounds);
/* Halo plan for the owned rows [r0, r1) of a global CSR: halo = sorted unique global ids of the
 * columns outside [r0, r1).  Call once with halo == NULL to get *n_halo, then again with a
 * caller array of that size.  Local column ids: owned j -> j - r0, halo h -> (r1 - r0) + index of
 * h in halo.  col_local (size row_ptr[r1] - row_ptr[r0]) is written when non-NULL.
 * Because ownership ranges are contiguous and halo is sorted, the halo rows owned by one peer
 * form one contiguous slice of it: a received peer message lands in place (no unpack). */
plp_status plp_halo_plan(const int64_t* row_ptr, const int32_t* col, int64_t r0, int64_t r1,
                         int64_t* n_halo, int64_t* halo, int32_t* col_local);

/* ---------------------------------------------------------------------------------------------- */
/* Graph                                                                                            */
/* ---------------------------------------------------------------------------------------------- */
/* Uploads a host CSR of n_rows rows whose columns index the n_cols rows of U/eta (n_cols ==
 * n_rows on one GPU; owned + halo rows on P ranks).  flags: PLP_VALIDATE runs plp_validate_csr
 * first (PLP_VALIDATE_SYMMETRIC adds the symmetry check).  Device storage: int32 row_ptr (nnz must
 * be < 2^31, else PLP_ERR_SHAPE), int32 col, fp64 w.  Holds its own workspace. */
plp_status plp_create_graph(plp_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                            const int32_t* col, const double* w, uint32_t flags, plp_graph** out);
plp_status plp_graph_info(const plp_graph* g, int64_t* n_rows, int64_t* n_cols, int64_t* nnz);
/* Collective graph creation on a ctx with a communicator: this rank owns the
 * global rows [row_begin, row_end) of an n_global-node graph; the ranks' ranges must be contiguous
 * in rank order and cover [0, n_global).  row_ptr (n_own + 1 entries, any base), col (GLOBAL
 * column ids) and w are the host CSR of the owned rows.  The call finds this rank's halo (the
 * sorted distinct columns outside the owned range), relabels columns locally (owned j ->
 * j - row_begin, halo h -> n_own + index of h), exchanges the request lists with the peers (NCCL)
 * and keeps the send/recv plan.  Dense arrays of this graph then have n_cols = n_own + n_halo rows:
 * rows [0, n_own) are the caller's, rows [n_own, n_cols) are halo slots that the collective calls
 * (plp_fgrad, plp_hessvec, plp_fgrad_hessvec, plp_rcut) fill from the peers before their edge
 * pass (grouped NCCL send/recv; a peer's rows land in place).  Outputs (G, Hv, labels) have n_own
 * rows.  flags: PLP_VALIDATE checks the local CSR (symmetry needs the whole graph: not checked).
 * Without a communicator (world == 1, no id) the graph must have no column outside the range. */
plp_status plp_create_graph_dist(plp_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                                 const int64_t* row_ptr, const int32_t* col, const double* w,
                                 uint32_t flags, plp_graph** out);
/* n_own, n_halo (the dense arrays' n_cols = n_own + n_halo), row_begin, and the number of rows this
 * rank sends per exchange.  A graph from plp_create_graph reports n_own = n_rows, send_rows = 0. */
plp_status plp_graph_dist_info(const plp_graph* g, int64_t* n_own, int64_t* n_halo, int64_t* row_begin,
                               int64_t* send_rows);
/* Halo exchange of an n_cols x row_bytes device array (row_bytes % 4 == 0): one gather launch packs
 * the rows the peers need, grouped NCCL send/recv fill rows [n_own, n_cols).  Collective; no-op on a
 * single-rank graph.  The edge calls run it themselves; exposed for other per-node arrays. */
plp_status plp_halo_exchange(plp_ctx* ctx, const plp_graph* g, int row_bytes, void* X);
/* Host part of the plan (no GPU): the slice of a sorted halo owned by each of `world` ranks with
 * row bounds bounds[0..world] -- recv_off[q], recv_cnt[q].  PLP_ERR_ARG if a halo column lies
 * outside [bounds[0], bounds[world]). */
plp_status plp_dist_recv_plan(int world, const int64_t* bounds, int64_t n_halo, const int64_t* halo,
                              int64_t* recv_off, int64_t* recv_cnt);
plp_status plp_destroy_graph(plp_graph* g);

/* ---------------------------------------------------------------------------------------------- */
/* F_p, EucGrad, EucHessianEta                                              */
/* ---------------------------------------------------------------------------------------------- */
/* Notation: A_l = 1/2 sum_i sum_{j in N(i)} w_ij |U_il - U_jl|^p (reading #1), B_l = sum_i
 * |U_il|^p, F = sum_l A_l / B_l.  AB arrays hold [A_0..A_{k-1}, B_0..B_{k-1}].
 *
 * plp_fgrad: F (device double[1]), AB_out (device double[2k]) and, if G != NULL, the Euclidean
 * gradient G_il = (p/B_l)((Delta_p u^l)_i - (A_l/B_l) phi_p(U_il))  (reading #4).  With G it runs
 * two edge passes (objective, then gradient with the fresh AB).  Rank-local: F and AB are sums over
 * this rank's rows (single GPU: the global values).  Hot calls do not synchronise, so B_l = 0
 * (PLP_ERR_DEGENERATE) shows up as a non-finite F on the device; the Python binding checks it. */
plp_status plp_fgrad(plp_ctx* ctx, const plp_graph* g, int k, const double* U, double p,
                     double* F, double* AB_out, double* G);

/* plp_hessvec: Hv = H eta at U, one edge pass.  AB_in (device, 2k): the GLOBAL A, B at the same U
 * and p (from plp_fgrad).  mode PLP_HESS_SPARSE: Alg. 1 with D[l] = diag(H^l), H[l] = diag(H^l) -
 * H^l for H^l = p(p-1)[Lap(w~)/B - (A/B^2) diag(cap(|u|)^{p-2})], w~_ij = w_ij cap(|u_i-u_j|)^{p-2},
 * cap(x) = max(x, eps) (readings #5, #6, #8).  mode PLP_HESS_FULL adds the rank-two terms of the
 * exact Hessian of A/B and then needs G_in = the Euclidean gradient at U (from plp_fgrad); single
 * rank only (P ranks: use plp_edge_pass + plp_full_epilogue).  eps: curvature cap (1e-9 default). */
plp_status plp_hessvec(plp_ctx* ctx, const plp_graph* g, int k, const double* U, const double* eta,
                       double p, const double* AB_in, int mode, double eps, const double* G_in,
                       double* Hv);

/* plp_fgrad_hessvec: the benchmark unit -- F, G and Hv in ONE edge pass (one power per
 * edge-column, shared by F, G and Hv).  AB_in (device) as for plp_hessvec; if AB_in == NULL the
 * objective pass runs first (two edge passes).  AB_out (device, nullable) receives the A, B
 * recomputed by the fused pass (equals AB_in up to rounding: a built-in consistency check).
 * G, Hv (device, n_rows x k, nullable).  mode as for plp_hessvec (FULL: single rank). */
plp_status plp_fgrad_hessvec(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                             const double* eta, double p, const double* AB_in, int mode, double eps,
                             double* F, double* AB_out, double* G, double* Hv);

/* Low-level pieces for P ranks.  plp_edge_pass runs one edge pass:
 *   AB_in == NULL: objective only (G, Hv, dots_out must be NULL); otherwise G / Hv when non-NULL.
 * AB_out (device 2k, nullable): this rank's A, B partial sums.  dots_out (device 2k, nullable,
 * needs eta and AB_in): this rank's [alpha_l = sum_i p phi_p(U_il) eta_il,
 * gamma_l = sum_i G_il eta_il] with G the gradient at U computed inside the pass (stored only if
 * G != NULL).  eta may be NULL when Hv and dots_out are NULL. */
plp_status plp_edge_pass(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                         const double* eta, double p, double eps, const double* AB_in,
                         double* AB_out, double* dots_out, double* G, double* Hv);
/* Full-mode rank-two epilogue, elementwise over n_rows x k with GLOBAL AB and dots:
 *   gB = p phi_p(u), gA = B G + (A/B) gB, beta = B gamma + (A/B) alpha,
 *   Hv += -(gA alpha + gB beta)/B^2 + 2 A gB alpha / B^3        (reading #5). */
plp_status plp_full_epilogue(plp_ctx* ctx, int64_t n_rows, int k, const double* U, double p,
                             const double* AB, const double* dots, const double* G, double* Hv);
/* F = sum_l A_l / B_l from a (global) AB, on the device. */
plp_status plp_objective_from_ab(plp_ctx* ctx, int k, const double* AB, double* F);

/* ---------------------------------------------------------------------------------------------- */
/* Tall-skinny Grassmann kernels                                           */
/* ---------------------------------------------------------------------------------------------- */
/* out (device k x k, row-major) = X^T Y over n rows; fixed-order reduction. */
plp_status plp_gram(plp_ctx* ctx, int64_t n, int k, const double* X, const double* Y, double* out);
/* Horizontal projection at U (Grassmann):
 *   out = G - U (U^T G).  out may alias G.  Single rank (P ranks: plp_gram + all-reduce +
 *   plp_apply_sub). */
plp_status plp_project(plp_ctx* ctx, int64_t n, int k, const double* U, const double* G,
                       double* out);
/* out = X - U M  (M device k x k).  out may alias X. */
plp_status plp_apply_sub(plp_ctx* ctx, int64_t n, int k, const double* U, const double* M,
                         const double* X, double* out);
/* QR retraction: Q = the Q factor of U + xi with R_ii > 0, by Cholesky-QR2
 * (C = Y^T Y, R = chol(C), Q = Y R^-1, twice).  R_out (device k x k, nullable) = the product of
 * both R factors.  If the Cholesky of a Gram is not positive definite returns PLP_ERR_RANK (this
 * call synchronises the stream to read the flag).  Q may alias U or xi.  Single rank. */
plp_status plp_retract(plp_ctx* ctx, int64_t n, int k, const double* U, const double* xi, double* Q,
                       double* R_out);
/* Pieces for P ranks: C (device k x k, all-reduced by the caller) -> R upper, R_ii > 0 (device);
 * *info (device int) = 0 or the 1-based failing pivot.  Then Q = (X [+ Y]) R^-1. */
plp_status plp_cholesky(plp_ctx* ctx, int k, const double* C, double* R, int* info);
plp_status plp_apply_rinv(plp_ctx* ctx, int64_t n, int k, const double* X, const double* Y,
                          const double* R, double* Q);
/* <x, y> = sum_{i,l} x_il y_il (device double[1]); y = a x + b y. */
plp_status plp_dot(plp_ctx* ctx, int64_t n, int k, const double* x, const double* y, double* out);
plp_status plp_axpby(plp_ctx* ctx, int64_t n, int k, double a, const double* x, double b,
                     double* y);
/* Row gather (halo packing, reordering): out[r] = X[idx[r]] for r < m (idx device int64). */
plp_status plp_gather_rows(plp_ctx* ctx, int64_t m, int k, const int64_t* idx, const double* X,
                           double* out);

/* ---------------------------------------------------------------------------------------------- */
/* k-means discretisation and RCut                                        */
/* ---------------------------------------------------------------------------------------------- */
/* k-means on the n rows of X (n x dim, device), `clusters` clusters (1 <= clusters, dim <= 32,
 * n >= clusters).  uniforms: HOST restarts x clusters values in [0,1) for k-means++ seeding (the
 * same array the oracle gets).  Algorithm (reading #13): per restart, seed (first centre
 * floor(u0 n); centre m = smallest i with cumsum(D^2)_i > u_m sum D^2; if sum D^2 = 0 then
 * floor(u_m n)), assign (nearest, ties -> lowest index), then repeat {update means (empty cluster
 * -> the point farthest from its own centroid, lowest index); assign} until sse == 0,
 * |sse_prev - sse| < rel_tol sse_prev, or max_iters updates.  Best restart = lowest sse.
 * Outputs: labels (device int32 n), centroids (device clusters x dim), *sse and *iters (HOST).
 * Synchronises (the loop is host-driven).  Single rank. */
plp_status plp_kmeans(plp_ctx* ctx, int64_t n, int dim, int clusters, const double* X,
                      const double* uniforms, int restarts, int max_iters, double rel_tol,
                      int32_t* labels, double* centroids, double* sse, int* iters);
/* Collective k-means (k x k / k x dim reductions all-reduced): the rows are the
 * ranks' X blocks (n_local x dim each, device) concatenated in rank order, n_local >= 0 with the
 * global n >= clusters.  The same algorithm and uniforms as plp_kmeans on the concatenated rows:
 * seeding picks use the global D^2 sum (each rank's sum all-reduced; the rank whose running sum
 * crosses u sum D^2 picks inside its block and broadcasts the point), Lloyd's per-cluster sums,
 * counts and sse are all-reduced, an empty cluster takes the globally farthest point (largest
 * distance, lowest global index).  Outputs: labels of this rank's rows (device int32 n_local);
 * centroids, *sse, *iters identical on every rank.  On one rank (a context without a
 * communicator, or world = 1) bitwise equal to plp_kmeans; across ranks equal up to the rounding
 * order of the all-reduced sums.  Collective: every rank calls it with the same arguments except
 * n_local, X and labels.  Synchronises. */
plp_status plp_kmeans_dist(plp_ctx* ctx, int64_t n_local, int dim, int clusters, const double* X,
                           const double* uniforms, int restarts, int max_iters, double rel_tol,
                           int32_t* labels, double* centroids, double* sse, int* iters);
/* RCut = sum_c cut(C_c, ~C_c) / |C_c| over the graph's rows; labels (device
 * int32, n_cols entries so halo labels resolve).  Outputs (device, nullable): cut[clusters],
 * sizes[clusters] (int64), rcut[1].  Empty cluster -> rcut = NaN (device; the binding raises). */
plp_status plp_rcut(plp_ctx* ctx, const plp_graph* g, int clusters, const int32_t* labels,
                    double* cut, int64_t* sizes, double* rcut);

/* ---------------------------------------------------------------------------------------------- */
/* Device-resident truncated CG ("truncated conjugate      */
/* gradient scheme")                                                                */
/* ---------------------------------------------------------------------------------------------- */
#define PLP_TCG_SCAL_LEN 4160 /* doubles in the tCG scalar/matrix workspace `scal` */
enum {
  PLP_TCG_RUNNING = 0, PLP_TCG_BOUNDARY = 1, PLP_TCG_NEGATIVE_CURVATURE = 2, PLP_TCG_CONVERGED = 3,
  PLP_TCG_MAXITER = 4, PLP_TCG_INTERIOR = 5
};
/* Steihaug-Toint tCG for min <grad, s> + <s, H s>/2, ||s|| <= delta, with the Riemannian Hessian
 * H(x) = P_U(EucHess[x]) - x S of solver.py (reading #21).  All vectors are device n x k (n =
 * the graph's rows), scal a device double[PLP_TCG_SCAL_LEN] and status a device int[2] =
 * {status, iterations}.
 * plp_tcg_init: eta = Heta = 0, r = grad, delta_dir = -grad, scalars (stop tolerance
 * ||g|| min(||g||^theta, kappa)); status INTERIOR if grad = 0.
 * plp_tcg_run: `iters` iterations (launches only, no synchronisation; iterations after the exit
 * condition leave eta, Heta and delta_dir unchanged), Hd a work array.  fused = 0: the
 * recurrences are bitwise those of solver.py's host loop (projection, curvature term, dots and
 * axpbys as separate passes).  fused = 1 (k = 8 or 16, or k = 1, 2, 4 with n k divisible by 8 --
 * the arrays then read as n k / 8 rows of 8 with block-diagonal k x k matrices --, 16-byte aligned
 * vectors; else PLP_ERR_ARG):
 * after the edge pass, three streaming passes on the fp64 tensor cores:
 * <d, Hd> = sum d (EH - d S) - <U^T d, U^T EH>_F element by element; the eta / Heta / r updates
 * with Hd = EH - U U^T EH - d S formed in registers, U^T r and ||r||^2; then r's re-projection and
 * the new direction -- the same iteration up to rounding order.  Errors: PLP_ERR_ARG for null
 * pointers (Heta only as below), iters < 0, max_iters < 1; CUDA errors as PLP_ERR_CUDA.  Read `status` to know when it stopped; eta / Heta are
 * the step and H step.  With fused = 1, Heta may be NULL (plp_tcg_init likewise): the update pass
 * then neither reads nor writes an H step (16 n k bytes less per iteration) and the caller forms
 * H(eta) once at the end (by linearity the same vector up to rounding). */
plp_status plp_tcg_init(plp_ctx* ctx, int64_t n, int k, const double* grad, double delta, double kappa,
                        double theta, double* eta, double* Heta, double* r, double* delta_dir,
                        double* scal, int* status);
plp_status plp_tcg_run(plp_ctx* ctx, const plp_graph* g, int k, const double* U, const double* AB,
                       const double* G_in, const double* S, double p, double eps, int mode, double* eta,
                       double* Heta, double* r, double* delta_dir, double* Hd, double* scal,
                       int* status, int max_iters, int iters, int fused);
/* CUDA graph of `iters` plp_tcg_run iterations with exactly these arguments (pointers and scalars
 * are baked in: refresh the buffers' contents, not the pointers, between launches).  Captured on
 * ctx's stream, which must be a created stream (not the legacy / per-thread default: PLP_ERR_ARG).
 * plp_tcg_graph_launch enqueues the whole batch on ctx's stream (one launch); _nodes reports the
 * captured kernel/memset node count; libplp owns the graph (destroy frees it). */
typedef struct plp_tcg_graph plp_tcg_graph;
plp_status plp_tcg_graph_create(plp_ctx* ctx, const plp_graph* g, int k, const double* U, const double* AB,
                                const double* G_in, const double* S, double p, double eps, int mode,
                                double* eta, double* Heta, double* r, double* delta_dir, double* Hd,
                                double* scal, int* status, int max_iters, int iters, int fused,
                                plp_tcg_graph** out);
plp_status plp_tcg_graph_launch(plp_tcg_graph* graph);
plp_status plp_tcg_graph_nodes(const plp_tcg_graph* graph, int* nodes);
plp_status plp_tcg_graph_destroy(plp_tcg_graph* graph);

/* ---------------------------------------------------------------------------------------------- */
/* Diagnostics                                                                                      */
/* ---------------------------------------------------------------------------------------------- */
/* Evaluates the edge kernel's power policy for this (p, eps) on n device values a[i] >= 0:
 * s[i] = cap(a_i)^{p-2}, t[i] = a_i^{p-1} (exactly what the fused pass uses per edge-column).
 * For accuracy tests of the custom fp64 powers. */
plp_status plp_debug_pow(plp_ctx* ctx, int64_t n, const double* a, double p, double eps, double* s,
                         double* t);

/* Name and template shape of the last edge kernel this process launched (any context), e.g.
 * "edge_staged_kernel<K=8,CPL=4,LPR=2,UNR=1,pow=R5M4,eta=1>"; "" before the first launch.  The
 * pointer refers to a static buffer, valid until the next edge launch.  Diagnostics only (the
 * bench reports which kernel its roofline figure belongs to; tests check the dispatch). */
const char* plp_last_edge_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* PLP_H_ */
