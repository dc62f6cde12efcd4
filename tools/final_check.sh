#!/bin/bash
# Final check of a build on one box: k-means A/B against variant libraries (PLP_LIB), the whole GPU
# suite, smoke, the bench line, and the ncu capture of km_d2_kernel.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/final_check.sh TAG [variant.so ...]'
set -u
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
: > $OUT/kmeans_ab_$TAG.txt
for rep in 1 2; do
  echo "default $(python tools/prof_kmeans.py --time 9 2>&1 | tail -1)" >> $OUT/kmeans_ab_$TAG.txt
  for lib in "$@"; do
    echo "$lib $(PLP_LIB=$PWD/paper_2605_26975_b200/$lib python tools/prof_kmeans.py --time 9 2>&1 | tail -1)" >> $OUT/kmeans_ab_$TAG.txt
  done
done
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests_$TAG.log 2>&1
echo "TESTS_RC=$?" >> $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "SMOKE_RC=$?" >> $OUT/smoke_$TAG.log
python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "BENCH_RC=$?" >> $OUT/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/kmeans_launches_$TAG.csv python tools/prof_kmeans.py --iters 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:km_d2_kernel" -s 1 -c 1 \
    -o $OUT/prof_km_d2_$TAG python tools/prof_kmeans.py --iters 0 > $OUT/ncu_km_d2_$TAG.log 2>&1
echo DONE > $OUT/final_check_done_$TAG.txt
