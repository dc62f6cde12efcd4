"""Gather microbenchmark driver (tools/micro/gather_bench.cu) on the bench graph (C5, tile order)."""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "gather_bench.so")
NAMES = ["l4v16u1", "l4v16u2", "l4v16u4", "l4v16u8", "l2v32u1", "l2v32u4", "l4v16u4b4", "l4v16u8b4",
         "l4v16u4_noeta", "l4v16u8b4_noeta", "l2v32u4b4", "l4v16u2b8"]

if __name__ == "__main__":
    if sys.argv[1:] == ["build"]:
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", SO, os.path.join(HERE, "gather_bench.cu")])
        sys.exit(0)
    import torch
    from bench import get_graph
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    order = sys.argv[2] if len(sys.argv) > 2 else "tile"
    g = get_graph(cfg, order)
    lib = ctypes.CDLL(SO)
    rp = torch.from_numpy(g.row_ptr.astype("int32")).cuda()
    col = torch.from_numpy(g.col).cuda()
    U = torch.randn(g.n, 8, dtype=torch.float64, device="cuda")
    E = torch.randn(g.n, 8, dtype=torch.float64, device="cuda")
    out = torch.empty(g.n * 4, dtype=torch.float64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    for v, name in enumerate(NAMES):
        for _ in range(2):
            lib.gather_run(v, g.n, P(rp), P(col), P(U), P(E), P(out), sms)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
        ev[0].record()
        for i in range(10):
            occ = lib.gather_run(v, g.n, P(rp), P(col), P(U), P(E), P(out), sms)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ts = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(10))
        print(json.dumps({"variant": name, "occ": occ, "ms": round(ts[5], 4)}), flush=True)
