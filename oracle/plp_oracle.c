/*
 * plp_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for p-spectral clustering on
 * the Grassmann manifold (arxiv 2605.26975, "Nonlinear spectral clustering with C++ GraphBLAS").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load or call this library.  It shares no code, header, table or
 * constant with the CUDA path (paper_2605_26975_b200/csrc), and neither side includes the other.
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -fPIC -shared (no fast-math).  OpenMP only splits the
 * OUTER row loop; every reduction over rows is then done sequentially in ascending row order, so
 * results do not depend on the thread count.
 *
 * Conventions (DESIGN.md §3 "Readings"):
 *   Graph: CSR of the rows [0, n_rows) of W (both triangles stored), int64 rp[n_rows+1],
 *   int32 col[nnz], double w[nnz].  Column j indexes row j of U (U may have more rows than the
 *   graph has rows: a rank's owned rows followed by its halo rows).
 *   U, eta, outputs: node-major n x k, element (i, l) at [i*k + l].
 *   Optional `rows`/`nsel`: evaluate only the listed rows (outputs compacted in list order);
 *   rows == NULL means all rows 0..n_rows-1.
 *   Summation order: for each column l, row i ascending, then j in CSR order.
 *
 * Parity status per function: every function below is pinned by tests/test_oracle_*.py
 * (closed forms, finite differences, exact identities, worked examples); see DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_DEGENERATE = 4, OR_ERR_EMPTY = 5 };

void oracle_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int oracle_get_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* sign(x) with sign(0) = 0  (reading #7). */
static double sgn(double x) { return x > 0.0 ? 1.0 : (x < 0.0 ? -1.0 : 0.0); }

/* phi_p(x) = |x|^{p-1} sign(x)   (§II). */
double oracle_phi(double x, double p) { return pow(fabs(x), p - 1.0) * sgn(x); }

/* cap(x) = max(x, eps): curvature regularisation used ONLY in Hessian weights (reading #6). */
static double cap(double x, double eps) { return x > eps ? x : eps; }

static int64_t row_of(const int64_t* rows, int64_t s) { return rows ? rows[s] : s; }

/* ------------------------------------------------------------------------------------------- */
/* Eq. (1): numerators A_l = 1/2 sum_i sum_{j in N(i)} w_ij |U_il - U_jl|^p,  */
/* over all rows of the (local) graph.  Reading #1: the ordered double sum over a symmetric W     */
/* counts each undirected edge twice; the 1/2 of Eq. (1) undoes that.                             */
/* ------------------------------------------------------------------------------------------- */
int oracle_numerators(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w,
                      int k, const double* U, double p, double* A) {
  if (k < 1 || n_rows < 0) return OR_ERR_ARG;
  double* rowsum = (double*)calloc((size_t)(n_rows > 0 ? n_rows : 1) * k, sizeof(double));
  if (!rowsum) return OR_ERR_ARG;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n_rows; ++i) {
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t j = col[e];
      for (int l = 0; l < k; ++l)
        rowsum[i * k + l] += w[e] * pow(fabs(U[i * k + l] - U[j * k + l]), p);
    }
  }
  for (int l = 0; l < k; ++l) {
    double s = 0.0;
    for (int64_t i = 0; i < n_rows; ++i) s += rowsum[i * k + l];
    A[l] = 0.5 * s;
  }
  free(rowsum);
  return OR_OK;
}

/* p-norm to the p: B_l = ||u^l||_p^p = sum_i |U_il|^p, rows [0, n_rows). */
int oracle_pnorms(int64_t n_rows, int k, const double* U, double p, double* B) {
  if (k < 1 || n_rows < 0) return OR_ERR_ARG;
  for (int l = 0; l < k; ++l) {
    double s = 0.0;
    for (int64_t i = 0; i < n_rows; ++i) s += pow(fabs(U[i * k + l]), p);
    B[l] = s;
  }
  return OR_OK;
}

/* F_p(U) = sum_l A_l / B_l  (Eq. (1)).  Also returns A[k], B[k].  B_l = 0 -> degenerate. */
int oracle_objective(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w, int k,
                     const double* U, double p, double* A, double* B, double* F) {
  int st = oracle_numerators(n_rows, rp, col, w, k, U, p, A);
  if (st) return st;
  st = oracle_pnorms(n_rows, k, U, p, B);
  if (st) return st;
  double f = 0.0;
  for (int l = 0; l < k; ++l) {
    if (B[l] == 0.0) return OR_ERR_DEGENERATE;
    f += A[l] / B[l];
  }
  *F = f;
  return OR_OK;
}

/* p-Laplacian (Delta_p u)_i = sum_j w_ij phi_p(u_i - u_j)   (§II). */
int oracle_plaplacian(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w,
                      int k, const double* U, double p, int64_t nsel, const int64_t* rows,
                      double* L) {
  const int64_t ns = rows ? nsel : n_rows;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    for (int l = 0; l < k; ++l) {
      double acc = 0.0;
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t j = col[e];
        acc += w[e] * oracle_phi(U[i * k + l] - U[j * k + l], p);
      }
      L[s * k + l] = acc;
    }
  }
  return OR_OK;
}

/* EucGrad (closed form not printed -> reading #4):
 *   dA/du_i = p (Delta_p u)_i,  dB/du_i = p phi_p(u_i),
 *   G_il = (p / B_l) * ( (Delta_p u^l)_i - (A_l / B_l) * phi_p(U_il) ).                          */
int oracle_euc_grad(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w, int k,
                    const double* U, double p, const double* A, const double* B, int64_t nsel,
                    const int64_t* rows, double* G) {
  const int64_t ns = rows ? nsel : n_rows;
  for (int l = 0; l < k; ++l)
    if (B[l] == 0.0) return OR_ERR_DEGENERATE;
  int st = oracle_plaplacian(n_rows, rp, col, w, k, U, p, nsel, rows, G);
  if (st) return st;
#pragma omp parallel for schedule(static)
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    for (int l = 0; l < k; ++l) {
      const double Lil = G[s * k + l];
      G[s * k + l] = (p / B[l]) * (Lil - (A[l] / B[l]) * oracle_phi(U[i * k + l], p));
    }
  }
  return OR_OK;
}

/* Alg. 1 inputs, sparse mode (reading #5):
 *   w~_ij   = w_ij * cap(|u_i - u_j|)^{p-2}                     (modified weights)
 *   Hess A  = p(p-1) * Laplacian(w~);   Hess B = p(p-1) * diag(cap(|u_i|)^{p-2})
 *   H^l     = Hess A / B_l - (A_l / B_l^2) * Hess B
 *   D[l]_i  = diag(H^l)_i = p(p-1) * ( sum_j w~_ij / B_l - (A_l/B_l^2) cap(|u_i|)^{p-2} )
 *   H[l]_ij = diag(H^l) - H^l = p(p-1) * w~_ij / B_l   (off-diagonal, zero diagonal).
 * Outputs: D[nsel*k] (node-major) and Hval[nnz_sel*k], where the selected rows' edges are laid
 * out consecutively in list order (edge e of selected row s at (off_s + e - rp[i]) * k + l).     */
int oracle_hessian_parts(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w,
                         int k, const double* U, double p, double eps, const double* A,
                         const double* B, int64_t nsel, const int64_t* rows, double* D,
                         double* Hval) {
  const int64_t ns = rows ? nsel : n_rows;
  for (int l = 0; l < k; ++l)
    if (B[l] == 0.0) return OR_ERR_DEGENERATE;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ns + 1));
  if (!off) return OR_ERR_ARG;
  off[0] = 0;
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    off[s + 1] = off[s] + (rp[i + 1] - rp[i]);
  }
  const double pp1 = p * (p - 1.0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    for (int l = 0; l < k; ++l) {
      double deg_t = 0.0; /* sum_j w~_ij */
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t j = col[e];
        const double wt = w[e] * pow(cap(fabs(U[i * k + l] - U[j * k + l]), eps), p - 2.0);
        deg_t += wt;
        Hval[(off[s] + (e - rp[i])) * k + l] = pp1 * wt / B[l];
      }
      const double hb = pow(cap(fabs(U[i * k + l]), eps), p - 2.0);
      D[s * k + l] = pp1 * (deg_t / B[l] - (A[l] / (B[l] * B[l])) * hb);
    }
  }
  free(off);
  return OR_OK;
}

/* Alg. 1 EucHessianEta, per column l:
 *   line 6: v = 0;  line 7: v = vxm(eta^l, H[l]) under plus-times (H[l] symmetric, so
 *   v_i = sum_j H[l]_ij eta_j; reading #10);  line 8: w = eta^l (.) D[l];  line 9: r^l = w - v.  */
int oracle_euc_hessian_eta(int64_t n_rows, const int64_t* rp, const int32_t* col, int k,
                           const double* D, const double* Hval, const double* eta, int64_t nsel,
                           const int64_t* rows, double* r) {
  const int64_t ns = rows ? nsel : n_rows;
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ns + 1));
  if (!off) return OR_ERR_ARG;
  off[0] = 0;
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    off[s + 1] = off[s] + (rp[i + 1] - rp[i]);
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    for (int l = 0; l < k; ++l) {
      double v = 0.0;                                        /* grb::set(v, 0)     */
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e)            /* grb::vxm           */
        v += Hval[(off[s] + (e - rp[i])) * k + l] * eta[(int64_t)col[e] * k + l];
      const double wv = eta[i * k + l] * D[s * k + l];       /* grb::eWiseApply mul */
      r[s * k + l] = wv - v;                                 /* grb::eWiseApply sub */
    }
  }
  free(off);
  return OR_OK;
}

/* Full-mode rank-two correction (reading #5): the exact Hessian of A/B adds
 *   -(gA (gB.eta) + gB (gA.eta)) / B^2 + 2 A gB (gB.eta) / B^3,   gA = p Delta_p u, gB = p phi_p(u).
 * alpha_l = sum_i gB_il eta_il and beta_l = sum_i gA_il eta_il are GLOBAL dots (caller supplies
 * them for sharded use; oracle_dots_full computes them over all rows).                            */
int oracle_dots_full(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w, int k,
                     const double* U, const double* eta, double p, double* alpha, double* beta) {
  double* L = (double*)malloc(sizeof(double) * (size_t)(n_rows > 0 ? n_rows : 1) * k);
  if (!L) return OR_ERR_ARG;
  oracle_plaplacian(n_rows, rp, col, w, k, U, p, 0, NULL, L);
  for (int l = 0; l < k; ++l) {
    double a = 0.0, b = 0.0;
    for (int64_t i = 0; i < n_rows; ++i) {
      a += p * oracle_phi(U[i * k + l], p) * eta[i * k + l];
      b += p * L[i * k + l] * eta[i * k + l];
    }
    alpha[l] = a;
    beta[l] = b;
  }
  free(L);
  return OR_OK;
}

int oracle_rank_two(int64_t n_rows, const int64_t* rp, const int32_t* col, const double* w, int k,
                    const double* U, double p, const double* A, const double* B,
                    const double* alpha, const double* beta, int64_t nsel, const int64_t* rows,
                    double* r) {
  const int64_t ns = rows ? nsel : n_rows;
  double* L = (double*)malloc(sizeof(double) * (size_t)(ns > 0 ? ns : 1) * k);
  if (!L) return OR_ERR_ARG;
  oracle_plaplacian(n_rows, rp, col, w, k, U, p, nsel, rows, L);
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t i = row_of(rows, s);
    for (int l = 0; l < k; ++l) {
      const double gA = p * L[s * k + l];
      const double gB = p * oracle_phi(U[i * k + l], p);
      const double B2 = B[l] * B[l];
      r[s * k + l] += -(gA * alpha[l] + gB * beta[l]) / B2 + 2.0 * A[l] * gB * alpha[l] / (B2 * B[l]);
    }
  }
  free(L);
  return OR_OK;
}

/* ------------------------------------------------------------------------------------------- */
/* k-means discretisation (algorithm per reading #13 / SURVEY.md §8(c) item 6).      */
/* ------------------------------------------------------------------------------------------- */
/* squared distance, summed over coordinates in ascending order, no FMA contraction. */
static double dist2(const double* x, const double* c, int dim) {
  double s = 0.0;
  for (int d = 0; d < dim; ++d) {
    const double t = x[d] - c[d];
    s += t * t;
  }
  return s;
}

/* assign each point to its nearest centroid (ties -> lowest index); returns SSE (ascending i). */
static double km_assign(int64_t n, int dim, int K, const double* X, const double* C, int32_t* lab,
                        double* best_d) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int bc = 0;
    double bd = dist2(X + i * dim, C, dim);
    for (int c = 1; c < K; ++c) {
      const double d = dist2(X + i * dim, C + (int64_t)c * dim, dim);
      if (d < bd) { bd = d; bc = c; }
    }
    lab[i] = bc;
    best_d[i] = bd;
  }
  double sse = 0.0;
  for (int64_t i = 0; i < n; ++i) sse += best_d[i];
  return sse;
}

/* centroid update: mean of assigned points (sums in ascending i).  An empty cluster is reseeded
 * at the point farthest from its own current centroid (best_d; lowest index on ties); clusters
 * are repaired in ascending order and a chosen point is not chosen again.                      */
static void km_update(int64_t n, int dim, int K, const double* X, const int32_t* lab,
                      double* best_d, double* C) {
  double* sum = (double*)calloc((size_t)K * dim, sizeof(double));
  int64_t* cnt = (int64_t*)calloc((size_t)K, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    const int c = lab[i];
    cnt[c] += 1;
    for (int d = 0; d < dim; ++d) sum[(int64_t)c * dim + d] += X[i * dim + d];
  }
  for (int c = 0; c < K; ++c) {
    if (cnt[c] > 0) {
      for (int d = 0; d < dim; ++d) C[(int64_t)c * dim + d] = sum[(int64_t)c * dim + d] / (double)cnt[c];
    } else {
      int64_t far = 0;
      for (int64_t i = 1; i < n; ++i)
        if (best_d[i] > best_d[far]) far = i;
      for (int d = 0; d < dim; ++d) C[(int64_t)c * dim + d] = X[far * dim + d];
      best_d[far] = -1.0;
    }
  }
  free(sum);
  free(cnt);
}

/* k-means++ seeding with caller-supplied uniforms u[0..K): first centre floor(u0 * n); centre m is
 * the smallest i with cumsum(D^2)_i > u_m * sum(D^2) (cumsum over ascending i); if sum(D^2) = 0
 * (all points coincide with chosen centres) centre m is floor(u_m * n).                        */
static void km_seed(int64_t n, int dim, int K, const double* X, const double* u, double* C,
                    double* D2) {
  int64_t c0 = (int64_t)floor(u[0] * (double)n);
  if (c0 >= n) c0 = n - 1;
  for (int d = 0; d < dim; ++d) C[d] = X[c0 * dim + d];
  for (int64_t i = 0; i < n; ++i) D2[i] = dist2(X + i * dim, C, dim);
  for (int m = 1; m < K; ++m) {
    double S = 0.0;
    for (int64_t i = 0; i < n; ++i) S += D2[i];
    int64_t pick;
    if (S > 0.0) {
      const double target = u[m] * S;
      double cs = 0.0;
      pick = n - 1;
      for (int64_t i = 0; i < n; ++i) {
        cs += D2[i];
        if (cs > target) { pick = i; break; }
      }
    } else {
      pick = (int64_t)floor(u[m] * (double)n);
      if (pick >= n) pick = n - 1;
    }
    for (int d = 0; d < dim; ++d) C[(int64_t)m * dim + d] = X[pick * dim + d];
    for (int64_t i = 0; i < n; ++i) {
      const double dd = dist2(X + i * dim, C + (int64_t)m * dim, dim);
      if (dd < D2[i]) D2[i] = dd;
    }
  }
}

/* Lloyd with restarts.  Each restart: seed -> assign -> repeat {update; assign} until
 * sse == 0 or |sse_prev - sse| < rel_tol * sse_prev, or max_iters updates.  The returned labels
 * are the nearest-centroid assignment to the returned centroids, and sse is measured against
 * them.  Best restart = lowest sse (lowest restart index on ties).                               */
int oracle_kmeans(int64_t n, int dim, int K, const double* X, const double* uniforms, int restarts,
                  int max_iters, double rel_tol, int32_t* labels, double* centroids, double* sse_out,
                  int* iters_out) {
  if (n < K || K < 1 || dim < 1 || restarts < 1) return OR_ERR_ARG;
  double* C = (double*)malloc(sizeof(double) * (size_t)K * dim);
  double* bd = (double*)malloc(sizeof(double) * (size_t)n);
  int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  double best = INFINITY;
  for (int r = 0; r < restarts; ++r) {
    km_seed(n, dim, K, X, uniforms + (int64_t)r * K, C, bd);
    double sse = km_assign(n, dim, K, X, C, lab, bd);
    int it = 0;
    while (it < max_iters) {
      km_update(n, dim, K, X, lab, bd, C);
      const double sse_new = km_assign(n, dim, K, X, C, lab, bd);
      ++it;
      const int conv = (sse == 0.0) || (fabs(sse - sse_new) < rel_tol * sse);
      sse = sse_new;
      if (conv) break;
    }
    if (sse < best) {
      best = sse;
      memcpy(labels, lab, sizeof(int32_t) * (size_t)n);
      memcpy(centroids, C, sizeof(double) * (size_t)K * dim);
      if (iters_out) *iters_out = it;
    }
  }
  *sse_out = best;
  free(C);
  free(bd);
  free(lab);
  return OR_OK;
}

/* Balanced cut (§III-A): RCut = sum_c cut(C_c, ~C_c) / |C_c|, with
 * cut(C, ~C) = sum_{i in C} sum_{j in N(i), j not in C} w_ij (each cut edge once per side).      */
int oracle_rcut(int64_t n, const int64_t* rp, const int32_t* col, const double* w, int K,
                const int32_t* labels, double* cut, int64_t* sizes, double* rcut) {
  for (int c = 0; c < K; ++c) { cut[c] = 0.0; sizes[c] = 0; }
  for (int64_t i = 0; i < n; ++i) {
    const int c = labels[i];
    if (c < 0 || c >= K) return OR_ERR_ARG;
    sizes[c] += 1;
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e)
      if (labels[col[e]] != c) cut[c] += w[e];
  }
  double s = 0.0;
  for (int c = 0; c < K; ++c) {
    if (sizes[c] == 0) return OR_ERR_EMPTY;
    s += cut[c] / (double)sizes[c];
  }
  *rcut = s;
  return OR_OK;
}
