#!/bin/bash
# A/B of the fused tCG iteration: this build against a tools/tune_edge.py variant (default
# tcg_r_every: every pass C writes r), alternating, tools/prof_tcg.py with CUDA events.
set -u
VAR=${1:-tcg_r_every}
OUT=gpurun_out/tcg_ab_$VAR.txt
mkdir -p gpurun_out
for rep in 1 2; do
  for c in C5 D23; do
    echo "$c this-build $(python tools/prof_tcg.py --config $c --iters 10 --time 20 2>&1 | tail -1)" >> $OUT
    echo "$c $VAR $(PLP_LIB=paper_2605_26975_b200/variants/$VAR/libplp.so python tools/prof_tcg.py --config $c --iters 10 --time 20 2>&1 | tail -1)" >> $OUT
  done
done
