#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tiny invocations of every kernel family
# (tools/sanitize_cases.py); summaries land in gpurun_out/sanitize_<tool>_<case>.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for c in halo staged rows tcg dense kmeans; do
    env=""
    [ "$c" = staged ] && env="PLP_EDGE_STAGED=1"
    [ "$c" = rows ] && env="PLP_EDGE_ROWS=1"
    extra=""
    [ "$tool" = racecheck ] && extra="--racecheck-report all"
    timeout 900 env $env $CS --tool $tool $extra --print-limit 20 --error-exitcode 99 \
        python tools/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    echo "RC=$?" >> gpurun_out/sanitize_${tool}_${c}.log
  done
done
