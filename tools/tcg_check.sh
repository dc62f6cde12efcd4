#!/bin/bash
# tCG checks and timing after a change to the fused passes: the tCG GPU tests, then the steady-state
# fused iteration at C5 and D23 (tools/prof_tcg.py, CUDA events).  Outputs in gpurun_out/.
set -u
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_collective.py -m gpu -q -p no:cacheprovider \
    > gpurun_out/tcg_tests_$TAG.log 2>&1
echo "TESTS_RC=$?" >> gpurun_out/tcg_tests_$TAG.log
for c in C5 D23; do
  for it in 2 10; do
    echo "$c iters=$it $(python tools/prof_tcg.py --config $c --iters $it --time 20 2>&1 | tail -1)" >> gpurun_out/tcg_time_$TAG.txt
  done
done
