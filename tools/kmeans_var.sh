#!/bin/bash
# k-means variants on one box: Lloyd / seeding times of the built library and of variant libraries
# (PLP_LIB), then the k-means, clustering and end-to-end GPU tests under each variant.
#   /usr/local/graft/bin/gpurun --timeout 1500 -- 'bash tools/kmeans_var.sh TAG variant.so ...'
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
for lib in "$@"; do
  PLP_LIB=$PWD/paper_2605_26975_b200/$lib timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "kmeans or cluster or end_to_end" > $OUT/kmeans_tests_${TAG}_$lib.log 2>&1
  echo "TESTS_RC=$?" >> $OUT/kmeans_tests_${TAG}_$lib.log
done
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "kmeans or cluster or end_to_end" > $OUT/kmeans_tests_${TAG}_default.log 2>&1
echo "TESTS_RC=$?" >> $OUT/kmeans_tests_${TAG}_default.log
echo DONE > $OUT/kmeans_var_done_$TAG.txt
