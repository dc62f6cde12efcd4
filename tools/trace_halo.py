"""Pipeline trace of the halo kernel (build variant `trace`: -DPLP_HALO_TRACE, tools/tune_edge.py).

  PLP_LIB=paper_2605_26975_b200/variants/trace/libplp.so python tools/trace_halo.py [--config C5]
Runs the fused pass once and reads the per-tile clock64 stamps: producer past the "empty" wait /
done issuing, each consumer warp past the "full" wait / releasing the buffer.  Prints where the
consumer warps' time goes (compute, waiting for a tile) and how long a tile takes from issue to
ready, in SM cycles (medians over CTAs and tiles)."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import get_graph, CONFIG_KP  # noqa: E402
from paper_2605_26975_b200 import plp  # noqa: E402
from plp_inputs import draw_U, draw_eta  # noqa: E402

TT, SL = 320, 36


def main():
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C5"
    k, p = CONFIG_KP[cfg]
    g = get_graph(cfg, "tile")
    ctx = plp.Context(0)
    G = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=0)
    U = torch.from_numpy(draw_U(g.n, k, 0)).cuda()
    eta = torch.from_numpy(draw_eta(g.n, k, 0)).cuda()
    F, AB, _ = plp.fgrad(ctx, G, U, p, want_grad=False)
    for _ in range(3):
        plp.fgrad_hessvec(ctx, G, U, eta, p, AB_in=AB)
    torch.cuda.synchronize()
    n = 160 * TT * SL
    buf = np.zeros(n, dtype=np.int64)
    lib = plp._lib
    rc = lib.plp_debug_halo_trace(ctypes.c_void_p(buf.ctypes.data), ctypes.c_longlong(n))
    assert rc == 0, rc
    T = buf.reshape(160, TT, SL)
    HT = plp.HALO_TILE
    NC = 2 * HT // 32
    ncta = 148
    ntile = int(np.ceil(((g.n + HT - 1) // HT) / ncta))
    T = T[:ncta, :min(ntile - 1, TT)]
    P0, P1 = T[:, :, 0], T[:, :, 1]
    C = T[:, :, 2:2 + NC]          # past full wait
    R = T[:, :, 16:16 + NC]        # released
    comp = R - C                   # per warp compute per tile
    wait = C[:, 1:] - R[:, :-1]    # per warp wait before tile it
    ready = C.min(axis=2)
    rel_last = R.max(axis=2)
    rel_first = R.min(axis=2)
    issue_to_ready = ready[:, 2:] - P1[:, 2:]
    react = P0[:, 2:] - rel_last[:, :-2]   # producer past empty(it) vs last release of it - 2
    skew = rel_last - rel_first
    out = {
        "tile_period_cycles": float(np.median(np.diff(rel_last, axis=1))),
        "warp_compute_per_tile": float(np.median(comp)),
        "warp_wait_per_tile_median": float(np.median(wait)),
        "warp_wait_per_tile_mean": float(np.mean(wait)),
        "wait_fraction_of_warp_time": float(np.sum(wait) / (np.sum(wait) + np.sum(comp[:, 1:]))),
        "release_skew_median": float(np.median(skew)),
        "issue_to_ready_median": float(np.median(issue_to_ready)),
        "issue_to_ready_p90": float(np.percentile(issue_to_ready, 90)),
        "producer_reaction_median": float(np.median(react)),
        "producer_issue_cycles_median": float(np.median(P1 - P0)),
        "producer_list_wait_median": float(np.median(T[:, :, 32] - P0)),
        "producer_tma_issue_median": float(np.median(T[:, :, 33] - T[:, :, 32])),
        "producer_halo_gather_issue_median": float(np.median(T[:, :, 34] - T[:, :, 33])),
        "warp_compute_by_warp": [float(np.median(comp[:, :, w])) for w in range(NC)],
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
