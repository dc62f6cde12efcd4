"""Layout experiment: U and eta interleaved per node (UE = [U_i | eta_i], row stride 2k) vs separate
arrays, same graph and values.  Run with PLP_INTERLEAVE=1 for the interleaved arm."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import get_graph, CONFIG_KP  # noqa: E402
from paper_2605_26975_b200 import plp  # noqa: E402
from plp_inputs import draw_U, draw_eta  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
k, p = CONFIG_KP[cfg]
g = get_graph(cfg, "tile")
ctx = plp.Context(0)
G = plp.Graph(ctx, g.row_ptr, g.col, g.w, flags=0)
U = torch.from_numpy(draw_U(g.n, k, 0)).cuda()
E = torch.from_numpy(draw_eta(g.n, k, 0)).cuda()
F, AB, _ = plp.fgrad(ctx, G, U, p, want_grad=False)
inter = os.environ.pop("PLP_INTERLEAVE", "") == "1"
ref = plp.fgrad_hessvec(ctx, G, U, E, p, AB_in=AB)
torch.cuda.synchronize()
if inter:
    os.environ["PLP_DEBUG_LDX"] = str(2 * k)  # read by plp_edge_pass on every call
if inter:
    UE = torch.cat([U, E], dim=1).contiguous()
    up, ep = UE.data_ptr(), UE.data_ptr() + 8 * k
else:
    up, ep = U.data_ptr(), E.data_ptr()
Gr = torch.empty(g.n, k, dtype=torch.float64, device="cuda")
Hv = torch.empty_like(Gr)
lib = plp._lib
VP = ctypes.c_void_p


def call():
    st = lib.plp_edge_pass(ctx.h, G.h, k, VP(up), VP(ep), ctypes.c_double(p), ctypes.c_double(1e-9),
                           VP(AB.data_ptr()), None, None, VP(Gr.data_ptr()), VP(Hv.data_ptr()))
    assert st == 0, st


for _ in range(3):
    call()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
ev[0].record()
for i in range(20):
    call()
    ev[i + 1].record()
torch.cuda.synchronize()
ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
err_g = ((Gr - ref[2]).abs().max() / ref[2].abs().max()).item()
err_h = ((Hv - ref[3]).abs().max() / ref[3].abs().max()).item()
print(json.dumps({"cfg": cfg, "interleaved": inter, "ms": ts[10], "err_G": err_g, "err_Hv": err_h}))
