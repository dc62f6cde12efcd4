#!/bin/bash
# NEXT-4 on one GPU (the gpurun boxes have one): per-component runtime breakdown of the whole
# continuation solve + clustering on Delaunay stand-ins of growing size (r = 20..23, the paper's
# weak-scaling sizes), and the NEXT-3 quality study; plus the halo pipeline trace.
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/next4_round.sh TAG'
TAG=${1:-r02}
mkdir -p gpurun_out
for r in 20 21 22 23; do
  timeout 900 python tools/solver_breakdown.py D$r --k 4 --sched 2.0,1.6,1.2 --graphs > gpurun_out/breakdown_${TAG}_D$r.json 2> gpurun_out/breakdown_${TAG}_D$r.err
done
timeout 1800 python tools/quality_study.py D16 D20 D21 D22 D23 > gpurun_out/quality_$TAG.jsonl 2> gpurun_out/quality_$TAG.err
PLP_LIB=paper_2605_26975_b200/variants/trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_$TAG.json 2>&1
echo DONE > gpurun_out/next4_done_$TAG.txt
for c in C5 C3 C4 D23; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-variants > gpurun_out/bench_${TAG}_$c.json 2>/dev/null; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py -q -x -p no:cacheprovider > gpurun_out/par_$TAG.log 2>&1
