#!/bin/bash
# ncu --set full of one edge-kernel launch on the bench workload: default library (staged) and the
# unstaged row kernel, plus any PLP_LIB variants given as args.  Reports in gpurun_out/.
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-x}
python tools/prof_edge.py --reps 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:edge_(staged_)?kernel" -s 1 -c 1 \
    -o $OUT/prof_${TAG}_staged python tools/prof_edge.py --reps 2 > $OUT/ncu_${TAG}_staged.log 2>&1
PLP_EDGE_ROWS=1 ncu --set full --clock-control none --import-source on -k "regex:edge_(staged_)?kernel" -s 1 -c 1 \
    -o $OUT/prof_${TAG}_row python tools/prof_edge.py --reps 2 > $OUT/ncu_${TAG}_row.log 2>&1
for v in "$@"; do
  PLP_LIB=paper_2605_26975_b200/variants/$v/libplp.so ncu --set full --clock-control none --import-source on \
    -k "regex:edge_(staged_)?kernel" -s 1 -c 1 -o $OUT/prof_${TAG}_$v python tools/prof_edge.py --reps 2 \
    > $OUT/ncu_${TAG}_$v.log 2>&1
done
