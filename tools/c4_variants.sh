#!/bin/bash
# C4 (k = 20) row-kernel variants: the default build, then each variant of tools/tune_edge.py, kernel
# time by CUDA events (tools/prof_edge.py --events).  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
python tools/prof_edge.py --config C4 --reps 20 --events > gpurun_out/c4_base.log 2>&1
python tools/tune_edge.py run "$@" --config C4 > gpurun_out/c4_variants.log 2>&1
python tools/prof_edge.py --config C4 --reps 20 --events > gpurun_out/c4_base2.log 2>&1
