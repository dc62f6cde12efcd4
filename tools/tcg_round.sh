#!/bin/bash
# After a change to the fused tCG passes: the tCG / solver / collective GPU tests, the A/B of the
# fused iteration against a variant library (tools/tcg_ab.sh), and one ncu capture of pass B.
set -u
TAG=${1:-x}; VAR=${2:-tcg_old}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_collective.py -m gpu -q -p no:cacheprovider \
    > gpurun_out/tcg_tests_$TAG.log 2>&1
echo "TESTS_RC=$?" >> gpurun_out/tcg_tests_$TAG.log
bash tools/tcg_ab.sh $VAR
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tcg_update_kernel" -s 1 -c 1 \
    -o gpurun_out/prof_tcg_update_$TAG python tools/prof_tcg.py --iters 2 > gpurun_out/ncu_tcg_$TAG.log 2>&1
