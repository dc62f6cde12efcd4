"""Build / time variants of the edge kernel (unroll, register cap, lanes per row).

  python tools/tune_edge.py build            # here (CPU): cross-compile every variant
  python tools/tune_edge.py run [--config C5] # on the GPU box: time each variant (CUDA events)
Variants land in paper_2605_26975_b200/variants/<name>/libplp.so (git-ignored, travel with gpurun).
"""
import json
import shutil
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VDIR = os.path.join(ROOT, "paper_2605_26975_b200", "variants")

VARIANTS = {
    "trace": ["-DPLP_HALO_TRACE"],
    "nb3": ["-DPLP_HALO_NBUF=3"],
    "nb3trace": ["-DPLP_HALO_NBUF=3", "-DPLP_HALO_TRACE"],
    "checked": ["FULL", "-DPLP_DEBUG_CHECKS"],
    "sleep0": ["-DPLP_HALO_SLEEP_NS=0"],
    "sleep256": ["-DPLP_HALO_SLEEP_NS=256"],
    "cpl4": ["-DPLP_HALO_CPL8=4"],
    # epilogue coefficients in shared memory (16 registers freed); with 256-row tiles, 16 consumer
    # warps + 1 producer (17 warps per SM, <= 120 registers), halo stage cap 352 rows
    "coef": ["-DPLP_HALO_COEF_SMEM=1"],
    "t256coef": ["-DPLP_HALO_COEF_SMEM=1", "-DPLP_HALO_TILE_ROWS=256", "-DPLP_HALO_CAP8=352"],
    # 240-row tiles: 15 consumer warps + 1 producer = 16 warps, 4 per SM sub-partition (each
    # sub-partition's register file holds 4 warps x 128 registers); 16-row degree-sorting windows
    "t224": ["FULL", "-DPLP_HALO_TILE_ROWS=224", "-DPLP_SCHED_WINDOW=32", "-DPLP_HALO_CAP8=400", "-DPLP_HALO_CAP16=96"],  # the earlier default
    "w8": ["FULL", "-DPLP_SCHED_WINDOW=8"],  # degree sort within 8-row windows (row kernel: C4)
    # full builds (all k): staged-kernel occupancy for the random-graph configs (C4, k = 20)
    "full_minb3": ["FULL", "-DPLP_EDGE_MINB=3"],
}


def build(names):
    from paper_2605_26975_b200.build import build as b
    for name in names:
        d = os.path.join(VDIR, name)
        shutil.rmtree(d, ignore_errors=True)
        os.makedirs(d, exist_ok=True)
        try:
            flags = [f for f in VARIANTS[name] if f != "FULL"]
            if "FULL" not in VARIANTS[name]:
                flags.append("-DPLP_TUNE_ONLY")
            b(obj_dir=os.path.join(d, "obj"), lib=os.path.join(d, "libplp.so"), extra=flags)
        except RuntimeError as e:
            print("FAILED", name, str(e)[-600:], flush=True)
        shutil.rmtree(os.path.join(d, "obj"), ignore_errors=True)
        print("built", name, flush=True)


def run(names, config, reps):
    res = {}
    for name in names:
        env = dict(os.environ, PLP_LIB=os.path.join(VDIR, name, "libplp.so"))
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "prof_edge.py"), "--config", config,
                              "--reps", str(reps), "--events"], env=env, capture_output=True, text=True)
        line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
        res[name] = json.loads(line[-1]) if line else {"error": out.stderr[-2000:]}
        print(name, res[name], flush=True)
    return res


if __name__ == "__main__":
    cmd = sys.argv[1]
    names = [a for a in sys.argv[2:] if not a.startswith("--")] or list(VARIANTS)
    config = "C5"
    if "--config" in sys.argv:
        config = sys.argv[sys.argv.index("--config") + 1]
        names = [n for n in names if n != config]
    if cmd == "build":
        build(names)
    else:
        r = run(names, config, 20)
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        json.dump(r, open(os.path.join(ROOT, "gpurun_out", f"tune_{config}.json"), "w"), indent=1)
