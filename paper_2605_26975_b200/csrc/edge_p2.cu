// Instantiation unit of the fused edge kernel for the power policy PowP2 (see edge_kernel.cuh).
#include "edge_inst.cuh"
#include "edge_kernel.cuh"

namespace plp {
plp_status launch_edge_p2(plp_ctx* ctx, const EdgeArgs& a, const PowP2& pw, int* grid) {
  return launch_edge_pow(ctx, a, pw, grid);
}
plp_status launch_epi_p2(plp_ctx* ctx, const EpiArgs& a, const PowP2& pw) {
  return launch_epi(ctx, a, pw);
}
}  // namespace plp
namespace plp {
plp_status launch_dbg_p2(plp_ctx* ctx, int64_t n, const double* a, double* s, double* t,
                            const PowP2& pw) {
  return launch_dbg(ctx, n, a, s, t, pw);
}
}  // namespace plp
