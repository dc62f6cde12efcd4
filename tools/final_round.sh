#!/bin/bash
# End-of-round evidence: tools/gpu_round.sh (tests, smoke, bench, reference arm, launch list, ncu of
# the edge kernel, per-row table, solver times, tCG launch list / ncu), the per-config bench lines,
# and the pass-B grid sweep of the fused tCG (PLP_TCG_GRID_B CTAs per SM).
set -u
TAG=${1:-r02n}
mkdir -p gpurun_out
bash tools/gpu_round.sh $TAG
for c in C3 C4 D23; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu >> gpurun_out/bench_configs_$TAG.jsonl 2>> gpurun_out/bench_configs_$TAG.err
done
for gb in 2 3 4 6; do
  echo "PLP_TCG_GRID_B=$gb $(PLP_TCG_GRID_B=$gb python tools/prof_tcg.py --config C5 --iters 10 --time 20 2>&1 | tail -1)" >> gpurun_out/tcg_gridb_$TAG.txt
done
echo DONE > gpurun_out/final_done_$TAG.txt
