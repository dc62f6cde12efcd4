#!/bin/bash
# Time the edge kernels (staged default / row / tiled, and any PLP_LIB variants given as args) on
# C5 and C3 with CUDA events (tools/prof_edge.py --events).
#   gpurun -- 'bash tools/cmp_edge.sh [variant ...]'
set -u
OUT=gpurun_out; mkdir -p $OUT
for cfg in C5 C3; do
  python tools/prof_edge.py --config $cfg --reps 20 --events > $OUT/cmp_default_$cfg.log 2>&1
  PLP_EDGE_STAGED=1 python tools/prof_edge.py --config $cfg --reps 20 --events > $OUT/cmp_staged_$cfg.log 2>&1
  PLP_EDGE_ROWS=1 python tools/prof_edge.py --config $cfg --reps 20 --events > $OUT/cmp_row_$cfg.log 2>&1
  for v in "$@"; do
    PLP_LIB=paper_2605_26975_b200/variants/$v/libplp.so python tools/prof_edge.py --config $cfg --reps 20 --events > $OUT/cmp_${v}_$cfg.log 2>&1
  done
done
grep -H kernel_ms $OUT/cmp_*.log | sed 's/"F".*//'
