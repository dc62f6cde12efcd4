// Host-side graph setup of libplp: validation, RCM ordering, relabelling,
// row-block partitioning and halo plans.  Plain C++ (no CUDA), callable without a GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "plp.h"

namespace plp {
plp_status set_error(plp_status st, const char* fmt, ...);
}
using plp::set_error;

extern "C" plp_status plp_validate_csr(int64_t n_rows, int64_t n_cols, const int64_t* rp,
                                       const int32_t* col, const double* w, int symmetric) {
  if (!rp) return set_error(PLP_ERR_ARG, "row_ptr is null");
  if (n_rows < 0 || n_cols < n_rows) return set_error(PLP_ERR_SHAPE, "need 0 <= n_rows <= n_cols");
  if (rp[0] != 0) return set_error(PLP_ERR_GRAPH, "row_ptr[0] != 0");
  for (int64_t i = 0; i < n_rows; ++i) {
    if (rp[i + 1] < rp[i]) return set_error(PLP_ERR_GRAPH, "row_ptr decreases at row %lld", (long long)i);
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      const int64_t j = col[e];
      if (j < 0 || j >= n_cols)
        return set_error(PLP_ERR_GRAPH, "column %lld out of range in row %lld", (long long)j, (long long)i);
      if (j == i) return set_error(PLP_ERR_GRAPH, "diagonal entry (%lld, %lld)", (long long)i, (long long)j);
      if (e > rp[i] && col[e - 1] >= j)
        return set_error(PLP_ERR_GRAPH, "row %lld: columns not strictly increasing", (long long)i);
      if (!(w[e] > 0.0) || !std::isfinite(w[e]))
        return set_error(PLP_ERR_GRAPH, "w(%lld, %lld) = %g not a positive finite weight",
                         (long long)i, (long long)j, w[e]);
    }
  }
  if (symmetric) {
    if (n_rows != n_cols) return set_error(PLP_ERR_SHAPE, "symmetry check needs a square CSR");
    for (int64_t i = 0; i < n_rows; ++i) {
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        const int64_t j = col[e];
        const int32_t* b = col + rp[j];
        const int32_t* en = col + rp[j + 1];
        const int32_t* f = std::lower_bound(b, en, (int32_t)i);
        if (f == en || *f != i)
          return set_error(PLP_ERR_GRAPH, "asymmetric: (%lld, %lld) stored but not (%lld, %lld)",
                           (long long)i, (long long)j, (long long)j, (long long)i);
        if (w[rp[j] + (f - b)] != w[e])
          return set_error(PLP_ERR_GRAPH, "asymmetric weight at (%lld, %lld)", (long long)i, (long long)j);
      }
    }
  }
  return PLP_OK;
}

// BFS from root over unvisited nodes; neighbours enqueued in (degree, id) order.  Returns the
// level of the last node and appends the visit order to `order`.
static int bfs_levels(int64_t root, const int64_t* rp, const int32_t* col,
                      const std::vector<int64_t>& deg, std::vector<int32_t>& level,
                      std::vector<int64_t>& order, bool sorted_nbrs) {
  const size_t start = order.size();
  order.push_back(root);
  level[root] = 0;
  std::vector<int64_t> nb;
  for (size_t h = start; h < order.size(); ++h) {
    const int64_t v = order[h];
    nb.clear();
    for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
      const int64_t j = col[e];
      if (level[j] < 0) {
        level[j] = level[v] + 1;
        nb.push_back(j);
      }
    }
    if (sorted_nbrs)
      std::sort(nb.begin(), nb.end(), [&](int64_t a, int64_t b) {
        return deg[a] != deg[b] ? deg[a] < deg[b] : a < b;
      });
    order.insert(order.end(), nb.begin(), nb.end());
  }
  return level[order.back()];
}

extern "C" plp_status plp_rcm_order(int64_t n, const int64_t* rp, const int32_t* col, int64_t* perm) {
  if (!rp || !perm || n < 0) return set_error(PLP_ERR_ARG, "bad argument");
  std::vector<int64_t> deg(n);
  for (int64_t i = 0; i < n; ++i) deg[i] = rp[i + 1] - rp[i];
  // candidate start nodes in (degree, id) order
  std::vector<int64_t> cand(n);
  std::iota(cand.begin(), cand.end(), 0);
  std::stable_sort(cand.begin(), cand.end(), [&](int64_t a, int64_t b) { return deg[a] < deg[b]; });
  std::vector<int32_t> level(n, -1), scratch_level(n, -1);
  std::vector<int64_t> order;
  order.reserve(n);
  std::vector<int64_t> tmp;
  size_t ci = 0;
  while ((int64_t)order.size() < n) {
    while (level[cand[ci]] >= 0) ++ci;
    int64_t root = cand[ci];
    // George-Liu pseudo-peripheral node: BFS, pick a min-degree node of the last level, repeat
    // while the eccentricity grows (at most 8 rounds).
    int ecc = -1;
    for (int it = 0; it < 8; ++it) {
      tmp.clear();
      const int e = bfs_levels(root, rp, col, deg, scratch_level, tmp, false);
      int64_t best = -1;
      for (size_t h = tmp.size(); h-- > 0;) {
        const int64_t v = tmp[h];
        if (scratch_level[v] != e) break;
        if (best < 0 || deg[v] < deg[best] || (deg[v] == deg[best] && v < best)) best = v;
      }
      for (int64_t v : tmp) scratch_level[v] = -1;
      if (e <= ecc) break;
      ecc = e;
      root = best;
    }
    bfs_levels(root, rp, col, deg, level, order, true);
  }
  for (int64_t a = 0; a < n; ++a) perm[a] = order[n - 1 - a];
  return PLP_OK;
}

// Tile ordering: RCM sweep, then tiles of T nodes grown by BFS from the first unassigned node of
// the sweep (restarting from the next unassigned sweep node when a BFS runs dry), nodes of a tile
// sorted by decreasing degree (the halo kernel deals the tile's 8-row slices to its warps in
// snake order, so every warp gets heavy and light rows while the rows of a slice stay alike).  Consecutive T-row ranges of the relabelled graph are then compact
// graph regions: most edges have both ends in one tile (C5: ~91% at T = 256), so the tiled edge
// kernel reads them from shared memory and evaluates each such undirected edge once.
extern "C" plp_status plp_tile_order(int64_t n, const int64_t* rp, const int32_t* col, int tile,
                                     int64_t* perm) {
  if (!rp || !perm || n < 0 || tile < 1) return set_error(PLP_ERR_ARG, "bad argument");
  std::vector<int64_t> rcm(n);
  plp_status st = plp_rcm_order(n, rp, col, rcm.data());
  if (st) return st;
  std::vector<char> used(n, 0);
  std::vector<int64_t> queue;
  queue.reserve(tile);
  int64_t out = 0, oi = 0;
  while (out < n) {
    const int64_t t0 = out;
    while (out < n && out - t0 < tile) {
      while (oi < n && used[rcm[oi]]) ++oi;
      if (oi >= n) break;
      queue.clear();
      queue.push_back(rcm[oi]);
      used[rcm[oi]] = 1;
      perm[out++] = rcm[oi];
      for (size_t h = 0; h < queue.size() && out - t0 < tile; ++h) {
        const int64_t v = queue[h];
        for (int64_t e = rp[v]; e < rp[v + 1] && out - t0 < tile; ++e) {
          const int64_t j = col[e];
          if (!used[j]) {
            used[j] = 1;
            queue.push_back(j);
            perm[out++] = j;
          }
        }
      }
    }
    std::stable_sort(perm + t0, perm + out, [&](int64_t a, int64_t b) {
      return (rp[a + 1] - rp[a]) > (rp[b + 1] - rp[b]);
    });
  }
  return PLP_OK;
}

extern "C" plp_status plp_permute_csr(int64_t n, const int64_t* rp, const int32_t* col,
                                      const double* w, const int64_t* perm, int64_t* rp_out,
                                      int32_t* col_out, double* w_out) {
  if (!rp || !perm || !rp_out) return set_error(PLP_ERR_ARG, "null argument");
  std::vector<int64_t> inv(n, -1);
  for (int64_t a = 0; a < n; ++a) {
    const int64_t o = perm[a];
    if (o < 0 || o >= n || inv[o] >= 0) return set_error(PLP_ERR_ARG, "perm is not a permutation");
    inv[o] = a;
  }
  rp_out[0] = 0;
  for (int64_t a = 0; a < n; ++a) rp_out[a + 1] = rp_out[a] + (rp[perm[a] + 1] - rp[perm[a]]);
  std::vector<std::pair<int32_t, double>> row;
  for (int64_t a = 0; a < n; ++a) {
    const int64_t o = perm[a];
    row.clear();
    for (int64_t e = rp[o]; e < rp[o + 1]; ++e) row.emplace_back((int32_t)inv[col[e]], w[e]);
    std::sort(row.begin(), row.end(),
              [](const std::pair<int32_t, double>& x, const std::pair<int32_t, double>& y) {
                return x.first < y.first;
              });
    int64_t d = rp_out[a];
    for (auto& pr : row) {
      col_out[d] = pr.first;
      w_out[d] = pr.second;
      ++d;
    }
  }
  return PLP_OK;
}

extern "C" plp_status plp_partition_rows(int64_t n, const int64_t* rp, int parts, double cost_row,
                                         double cost_nnz, int64_t* bounds) {
  if (!rp || !bounds || parts < 1 || n < 0) return set_error(PLP_ERR_ARG, "bad argument");
  const double total = cost_row * (double)n + cost_nnz * (double)rp[n];
  bounds[0] = 0;
  int64_t i = 0;
  double acc = 0.0;
  for (int q = 1; q < parts; ++q) {
    const double target = total * q / parts;
    while (i < n && acc + 0.5 * (cost_row + cost_nnz * (double)(rp[i + 1] - rp[i])) <= target) {
      acc += cost_row + cost_nnz * (double)(rp[i + 1] - rp[i]);
      ++i;
    }
    bounds[q] = i;
  }
  bounds[parts] = n;
  return PLP_OK;
}

extern "C" plp_status plp_halo_plan(const int64_t* rp, const int32_t* col, int64_t r0, int64_t r1,
                                    int64_t* n_halo, int64_t* halo, int32_t* col_local) {
  if (!rp || !n_halo || r1 < r0) return set_error(PLP_ERR_ARG, "bad argument");
  std::vector<int32_t> h;
  for (int64_t e = rp[r0]; e < rp[r1]; ++e) {
    const int64_t j = col[e];
    if (j < r0 || j >= r1) h.push_back((int32_t)j);
  }
  std::sort(h.begin(), h.end());
  h.erase(std::unique(h.begin(), h.end()), h.end());
  if (halo) {
    if (*n_halo < (int64_t)h.size()) return set_error(PLP_ERR_SHAPE, "halo array too small");
    for (size_t t = 0; t < h.size(); ++t) halo[t] = h[t];
  }
  *n_halo = (int64_t)h.size();
  if (col_local) {
    const int64_t own = r1 - r0;
    for (int64_t e = rp[r0]; e < rp[r1]; ++e) {
      const int64_t j = col[e];
      int64_t l;
      if (j >= r0 && j < r1) l = j - r0;
      else l = own + (std::lower_bound(h.begin(), h.end(), (int32_t)j) - h.begin());
      col_local[e - rp[r0]] = (int32_t)l;
    }
  }
  return PLP_OK;
}
