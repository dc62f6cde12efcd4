// Edge-pass dispatcher per power policy (included by the edge_pol_<NAME>.cu instantiation units).
#pragma once
#include "edge_halo.cuh"

namespace plp {

// Edge-pass entry for one power policy: the halo-tile kernel where it applies, else
// the staged row kernel; PLP_EDGE_STAGED=1 forces the staged kernel, PLP_EDGE_ROWS=1 the unstaged
// row kernel (kept for comparison measurements and parity tests).
template <class POW>
plp_status launch_edge_any(plp_ctx* ctx, const EdgeArgs& a, const POW& pw, int* grid) {
#ifdef PLP_TUNE_ONLY  // tuning builds (tools/tune_edge.py): k = 8 halo or staged shapes only
  if (a.k != 8) return set_error(PLP_ERR_ARG, "tuning build: k = 8 only");
  bool used_h = false;
  if (a.tile_list) {
    plp_status sh = try_launch_halo(ctx, a, pw, grid, &used_h);
    return sh ? sh : used_h ? PLP_OK : set_error(PLP_ERR_SHAPE, "tile list needs the halo kernel");
  }
  if (getenv("PLP_EDGE_STAGED") == nullptr) {
    plp_status sh = try_launch_halo(ctx, a, pw, grid, &used_h);
    if (sh || used_h) return sh;
  }
  return launch_staged_pow(ctx, a, pw, grid);
#else
  bool used = false;
  plp_status st = PLP_OK;
  if (a.tile_list) {  // a tile work list: the halo kernel or nothing (the caller falls back)
    st = try_launch_halo(ctx, a, pw, grid, &used);
    if (st) return st;
    return used ? PLP_OK : set_error(PLP_ERR_SHAPE, "tile list needs the halo kernel");
  }
  static const bool rows = getenv("PLP_EDGE_ROWS") != nullptr;
  if (rows) return launch_edge_pow(ctx, a, pw, grid);
  static const bool staged = getenv("PLP_EDGE_STAGED") != nullptr;
  if (!staged) {
    st = try_launch_halo(ctx, a, pw, grid, &used);
    if (st || used) return st;
    // wide rows without a halo tiling (C4: k = 20 on a 10-D kNN graph): latency-bound L2 gathers;
    // the row kernel (10 lanes x 2 columns at k = 20) keeps the most warps resident (a per-warp
    // shared-memory ring of cp.async-gathered rows measured slower: 2.3-3.8 against 1.63 ms)
    if (a.k > 16) return launch_edge_pow(ctx, a, pw, grid);
  }
  return launch_staged_pow(ctx, a, pw, grid);
#endif
}

}  // namespace plp
