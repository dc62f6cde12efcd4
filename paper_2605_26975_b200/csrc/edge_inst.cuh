// Per-power-policy launchers.  Each policy is instantiated in its own translation unit
// (edge_<NAME>.cu, generated from PLP_POW_LIST) so the kernel shapes compile in parallel; the
// overloads below let the dispatcher in edge.cu pick the launcher from the policy's type.
#pragma once
#include "plp_internal.h"
#include "pow64.cuh"

namespace plp {

struct EpiArgs {
  int64_t n;
  int k;
  const double* U;
  double p;
  const double* AB;
  const double* dots;
  const double* G;
  double* Hv;
};

#define PLP_DECL_POLICY(NAME, TYPE)                                                          \
  plp_status launch_edge_pol(plp_ctx*, const EdgeArgs&, const TYPE&, int*);                 \
  plp_status launch_epi_pol(plp_ctx*, const EpiArgs&, const TYPE&);                          \
  plp_status launch_dbg_pol(plp_ctx*, int64_t, const double*, double*, double*, const TYPE&);
PLP_POW_LIST(PLP_DECL_POLICY)
#undef PLP_DECL_POLICY

template <class POW>
__global__ void __launch_bounds__(256) debug_pow_kernel(int64_t n, const double* a, double* s,
                                                        double* t, POW pw) {
  extern __shared__ double4 smem_raw[];
  if constexpr (POW::kNeedsTables) {
    pw.init_smem(smem_raw);
    __syncthreads();
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double si, ti;
    pw.eval(a[i], si, ti);
    s[i] = si;
    t[i] = ti;
  }
}

template <class POW>
plp_status launch_dbg(plp_ctx* ctx, int64_t n, const double* a, double* s, double* t, const POW& pw) {
  const size_t smem = POW::kNeedsTables ? sizeof(PowTables) : 0;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)ctx->num_sms * 8) blocks = (int64_t)ctx->num_sms * 8;
  if (blocks < 1) blocks = 1;
  debug_pow_kernel<POW><<<(int)blocks, 256, smem, ctx->stream>>>(n, a, s, t, pw);
  PLP_LAUNCH_CHECK("debug_pow_kernel");
  return PLP_OK;
}

// Full-mode rank-two epilogue (reading #5): elementwise over n x k.
template <class POW>
__global__ void __launch_bounds__(256) full_epilogue_kernel(EpiArgs a, POW pw) {
  extern __shared__ double4 smem_raw[];
  if constexpr (POW::kNeedsTables) {
    pw.init_smem(smem_raw);
    __syncthreads();
  }
  const int64_t total = a.n * a.k;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int l = (int)(idx % a.k);
    const double A = a.AB[l], B = a.AB[a.k + l];
    const double al = a.dots[l], ga = a.dots[a.k + l];
    const double u = a.U[idx];
    const double au = fabs(u);
    double sn, tn;
    pw.eval(au, sn, tn);
    const double gB = a.p * copysign(tn, u);
    const double AoB = A / B;
    const double gA = B * a.G[idx] + AoB * gB;  // p Delta_p u, recovered from G (plp.h)
    const double be = B * ga + AoB * al;        // gA . eta
    const double B2 = B * B;
    a.Hv[idx] += -(gA * al + gB * be) / B2 + 2.0 * A * gB * al / (B2 * B);
  }
}

template <class POW>
plp_status launch_epi(plp_ctx* ctx, const EpiArgs& a, const POW& pw) {
  const size_t smem = POW::kNeedsTables ? sizeof(PowTables) : 0;
  int64_t blocks = (a.n * a.k + 255) / 256;
  const int64_t cap = (int64_t)ctx->num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  full_epilogue_kernel<POW><<<(int)blocks, 256, smem, ctx->stream>>>(a, pw);
  PLP_LAUNCH_CHECK("full_epilogue_kernel");
  return PLP_OK;
}

}  // namespace plp
