// Instantiation unit of the fused edge kernel, full-mode epilogue and power diagnostic for the
// power policy PowR5M4 (see pow64.cuh, edge_kernel.cuh, edge_inst.cuh).
#include "edge_inst.cuh"
#include "edge_dispatch.cuh"

namespace plp {
plp_status launch_edge_pol(plp_ctx* ctx, const EdgeArgs& a, const PowR5M4& pw, int* grid) {
  return launch_edge_any(ctx, a, pw, grid);
}
plp_status launch_epi_pol(plp_ctx* ctx, const EpiArgs& a, const PowR5M4& pw) {
  return launch_epi(ctx, a, pw);
}
plp_status launch_dbg_pol(plp_ctx* ctx, int64_t n, const double* a, double* s, double* t,
                          const PowR5M4& pw) {
  return launch_dbg(ctx, n, a, s, t, pw);
}
}  // namespace plp

#ifdef PLP_HALO_TRACE
extern "C" int plp_debug_halo_trace(long long* host, long long n) {
  return (int)cudaMemcpyFromSymbol(host, plp::g_halo_trace, sizeof(long long) * n);
}
#endif
