#!/bin/bash
# k-means (a11) evidence on one GPU: Lloyd iteration / seeding times, the ncu launch list with DRAM
# bytes, and one full capture each of km_assign_mma_kernel and km_d2_kernel at C5's n x k.
#   /usr/local/graft/bin/gpurun --timeout 900 -- 'bash tools/kmeans_round.sh [TAG]'
set -u
TAG=${1:-r02q}
OUT=gpurun_out
mkdir -p $OUT
python tools/prof_kmeans.py --time 7 > $OUT/kmeans_time_$TAG.json 2> $OUT/kmeans_time_$TAG.err
echo "RC=$?" >> $OUT/kmeans_time_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/kmeans_launches_$TAG.csv python tools/prof_kmeans.py --iters 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:km_assign_mma_kernel" -s 1 -c 1 \
    -o $OUT/prof_km_assign_$TAG python tools/prof_kmeans.py --iters 3 > $OUT/ncu_km_assign_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:km_d2_kernel" -s 1 -c 1 \
    -o $OUT/prof_km_d2_$TAG python tools/prof_kmeans.py --iters 0 > $OUT/ncu_km_d2_$TAG.log 2>&1
echo DONE > $OUT/kmeans_done_$TAG.txt
