// Device-resident truncated CG (Steihaug-Toint; Absil-Baker-Gallivan 2007, Alg. 2) for the
// trust-region subproblem of the Grassmann Newton solver (SURVEY.md §8(f) NEXT-1,
// "CUDA-Graph the tCG iteration").  The same recurrences as solver.py's host loop, with every
// scalar kept on the device: one iteration is a fixed launch sequence (Hessian-vector product,
// projection, curvature term, dots, scalar updates, axpbys with device coefficients), so the host
// can launch many iterations without reading anything back and the sequence can be captured in a
// CUDA graph.  The scalar kernels use explicitly rounded fp64 operations in the host code's order
// (no FMA contraction), so the device recurrence is bitwise that of solver.py's loop; after the
// exit condition every further iteration is a no-op for eta, Heta, r and delta.
#include <cmath>

#include "plp_internal.h"

namespace plp {

// scalar slots (double sc[16]) and status (int st[2] = {status, iterations})
enum {
  kZr = 0, kStopTol = 1, kDelta = 2, kEPe = 3, kEPd = 4, kDPd = 5, kDHd = 6, kAlpha = 7,
  kZnew = 9, kCEta = 10, kCR = 11, kCA = 12, kCB = 13
};

__global__ void tcg_init_kernel(double* sc, int* st, double delta, double kappa, double theta) {
  const double zr = sc[kZr];
  const double r0 = sqrt(zr);
  const double rt = pow(r0, theta);
  sc[kStopTol] = __dmul_rn(r0, rt < kappa ? rt : kappa);
  sc[kDelta] = delta;
  sc[kEPe] = 0.0;
  sc[kEPd] = 0.0;
  sc[kDPd] = zr;
  st[0] = r0 == 0.0 ? PLP_TCG_INTERIOR : PLP_TCG_RUNNING;
  st[1] = 0;
}

// after <delta, H delta>: step length, trust-boundary / negative-curvature exit
__global__ void tcg_scalar_a_kernel(double* sc, int* st) {
  if (st[0] != PLP_TCG_RUNNING) {
    sc[kCEta] = 0.0;
    sc[kCR] = 0.0;
    return;
  }
  st[1] += 1;
  const double zr = sc[kZr], dHd = sc[kDHd], ePe = sc[kEPe], ePd = sc[kEPd], dPd = sc[kDPd];
  const double delta = sc[kDelta];
  const double alpha = dHd != 0.0 ? zr / dHd : INFINITY;
  // e_Pe + 2 alpha e_Pd + alpha alpha d_Pd, left to right as in solver.py
  const double ePe_new =
      __dadd_rn(__dadd_rn(ePe, __dmul_rn(__dmul_rn(2.0, alpha), ePd)), __dmul_rn(__dmul_rn(alpha, alpha), dPd));
  const double dd = __dmul_rn(delta, delta);
  if (dHd <= 0.0 || ePe_new >= dd) {
    const double disc = __dadd_rn(__dmul_rn(ePd, ePd), __dmul_rn(dPd, __dsub_rn(dd, ePe)));
    const double tau = __ddiv_rn(__dadd_rn(-ePd, sqrt(disc)), dPd);
    sc[kCEta] = tau;
    sc[kCR] = 0.0;
    st[0] = dHd <= 0.0 ? PLP_TCG_NEGATIVE_CURVATURE : PLP_TCG_BOUNDARY;
    return;
  }
  sc[kEPe] = ePe_new;
  sc[kAlpha] = alpha;
  sc[kCEta] = alpha;
  sc[kCR] = alpha;
}

// after <r, r>: convergence test, conjugation
__global__ void tcg_scalar_b_kernel(double* sc, int* st, int max_iters) {
  if (st[0] != PLP_TCG_RUNNING) {
    sc[kCA] = 0.0;
    sc[kCB] = 1.0;
    return;
  }
  const double znew = sc[kZnew];
  if (sqrt(znew) <= sc[kStopTol]) {
    st[0] = PLP_TCG_CONVERGED;
    sc[kCA] = 0.0;
    sc[kCB] = 1.0;
    return;
  }
  const double zr = sc[kZr], alpha = sc[kAlpha], ePd = sc[kEPd], dPd = sc[kDPd];
  const double beta = __ddiv_rn(znew, zr);
  sc[kZr] = znew;
  sc[kCA] = -1.0;
  sc[kCB] = beta;
  sc[kEPd] = __dmul_rn(beta, __dadd_rn(ePd, __dmul_rn(alpha, dPd)));
  sc[kDPd] = __dadd_rn(znew, __dmul_rn(__dmul_rn(beta, beta), dPd));
  if (st[1] >= max_iters) st[0] = PLP_TCG_MAXITER;
}

// y = a x + b y with a, b read from the device (the host axpby's formula: fma(a, x, b * y))
__global__ void axpby_dev_kernel(int64_t total, const double* __restrict__ a, const double* __restrict__ x,
                                 const double* __restrict__ b, double* __restrict__ y) {
  const double av = *a, bv = b ? *b : 1.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = fma(av, x[i], bv * y[i]);
}

static int axpby_grid(plp_ctx* ctx, int64_t total) {
  int64_t g = (total + 1023) / 1024;
  if (g > ctx->max_ctas) g = ctx->max_ctas;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace plp

using namespace plp;

extern "C" plp_status plp_tcg_init(plp_ctx* ctx, int64_t n, int k, const double* grad, double delta,
                                   double kappa, double theta, double* eta, double* Heta, double* r,
                                   double* dlt, double* scal, int* status) {
  if (!ctx || !grad || !eta || !Heta || !r || !dlt || !scal || !status || n < 0)
    return set_error(PLP_ERR_ARG, "null argument");
  plp_status st = check_k(k);
  if (st) return st;
  if (!(delta > 0.0)) return set_error(PLP_ERR_DOMAIN, "trust radius must be positive");
  const size_t bytes = sizeof(double) * (size_t)n * k;
  PLP_CUDA(cudaMemcpyAsync(r, grad, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
  PLP_CUDA(cudaMemsetAsync(eta, 0, bytes, ctx->stream));
  PLP_CUDA(cudaMemsetAsync(Heta, 0, bytes, ctx->stream));
  PLP_CUDA(cudaMemsetAsync(dlt, 0, bytes, ctx->stream));
  if ((st = plp_axpby(ctx, n, k, -1.0, r, 0.0, dlt))) return st;  // delta = -r
  if ((st = plp_dot(ctx, n, k, r, r, scal + kZr))) return st;
  tcg_init_kernel<<<1, 1, 0, ctx->stream>>>(scal, status, delta, kappa, theta);
  PLP_LAUNCH_CHECK("tcg_init_kernel");
  return PLP_OK;
}

extern "C" plp_status plp_tcg_run(plp_ctx* ctx, const plp_graph* g, int k, const double* U,
                                  const double* AB, const double* G_in, const double* S, double p,
                                  double eps, int mode, double* eta, double* Heta, double* r,
                                  double* dlt, double* Hd, double* scal, int* status, int max_iters,
                                  int iters) {
  if (!ctx || !g || !U || !AB || !S || !eta || !Heta || !r || !dlt || !Hd || !scal || !status)
    return set_error(PLP_ERR_ARG, "null argument");
  if (iters < 0 || max_iters < 1) return set_error(PLP_ERR_ARG, "iters >= 0, max_iters >= 1");
  const int64_t n = g->n_rows;
  const int64_t total = n * k;
  const int grid = axpby_grid(ctx, total);
  plp_status st;
  for (int it = 0; it < iters; ++it) {
    // H(delta) = P(EucHess[delta]) - delta S
    if ((st = plp_hessvec(ctx, g, k, U, dlt, p, AB, mode, eps, G_in, Hd))) return st;
    if ((st = plp_project(ctx, n, k, U, Hd, Hd))) return st;
    if ((st = plp_apply_sub(ctx, n, k, dlt, S, Hd, Hd))) return st;
    if ((st = plp_dot(ctx, n, k, dlt, Hd, scal + kDHd))) return st;
    tcg_scalar_a_kernel<<<1, 1, 0, ctx->stream>>>(scal, status);
    PLP_LAUNCH_CHECK("tcg_scalar_a_kernel");
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCEta, dlt, nullptr, eta);
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCEta, Hd, nullptr, Heta);
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCR, Hd, nullptr, r);
    PLP_LAUNCH_CHECK("axpby_dev_kernel");
    if ((st = plp_project(ctx, n, k, U, r, r))) return st;  // keep the residual horizontal
    if ((st = plp_dot(ctx, n, k, r, r, scal + kZnew))) return st;
    tcg_scalar_b_kernel<<<1, 1, 0, ctx->stream>>>(scal, status, max_iters);
    PLP_LAUNCH_CHECK("tcg_scalar_b_kernel");
    axpby_dev_kernel<<<grid, 256, 0, ctx->stream>>>(total, scal + kCA, r, scal + kCB, dlt);
    PLP_LAUNCH_CHECK("axpby_dev_kernel");
  }
  return PLP_OK;
}
