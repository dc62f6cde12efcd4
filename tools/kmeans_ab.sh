#!/bin/bash
# k-means assign kernel A/B on one box: the built library against variant libraries (PLP_LIB), then
# the k-means GPU tests and the ncu capture of the default build.
#   /usr/local/graft/bin/gpurun --timeout 1200 -- 'bash tools/kmeans_ab.sh TAG lib1.so lib2.so ...'
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
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "kmeans or cluster or end_to_end or smoke" > $OUT/kmeans_tests_$TAG.log 2>&1
echo "TESTS_RC=$?" >> $OUT/kmeans_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" >> $OUT/kmeans_tests_$TAG.log 2>&1
echo "SMOKE_RC=$?" >> $OUT/kmeans_tests_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/kmeans_launches_$TAG.csv python tools/prof_kmeans.py --iters 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:km_assign_mma_kernel" -s 1 -c 1 \
    -o $OUT/prof_km_assign_$TAG python tools/prof_kmeans.py --iters 3 > $OUT/ncu_km_assign_$TAG.log 2>&1
echo DONE > $OUT/kmeans_ab_done_$TAG.txt
