#!/bin/bash
# One GPU box session: tests, smoke, bench (plain), then the ncu launch list of the same bench
# command and one full ncu capture of the edge kernel.  Outputs land in gpurun_out/.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [TAG]'
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/gpu_tests_$TAG.log 2>&1
echo "TESTS_RC=$?" >> $OUT/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "SMOKE_RC=$?" >> $OUT/smoke_$TAG.log
python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
echo "BENCH_RC=$?" >> $OUT/bench_$TAG.err
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
# launch list of the bench command (cold, serialised: compare shares, not absolutes)
python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/bench_small_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $OUT/launches_$TAG.csv python bench.py --steps 3 --warmup 3 --no-cpu \
    > $OUT/ncu_launches_$TAG.log 2>&1
echo "NCU_LAUNCHES_RC=$?" >> $OUT/ncu_launches_$TAG.log
# full capture of the dominant kernel (edge pass) on the bench workload
python tools/prof_edge.py --reps 3 > $OUT/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:edge_(halo_|staged_|tiled_)?kernel" -s 1 -c 1 \
    -o $OUT/prof_edge_$TAG python tools/prof_edge.py --reps 3 > $OUT/ncu_full_$TAG.log 2>&1
echo "NCU_FULL_RC=$?" >> $OUT/ncu_full_$TAG.log
# per-row table (every §8 row + the tCG iteration variants) and solver wall times
timeout 1200 python tools/bench_kernels.py --config C5 --oracle > $OUT/kernel_table_$TAG.jsonl 2>&1
timeout 900 python tools/solver_time.py C1 C2:20000 D16:8192 D20 > $OUT/solver_time_$TAG.jsonl 2>&1
# launch list + one full capture of the fused tCG passes (NEXT-2)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/tcg_launches_$TAG.csv python tools/prof_tcg.py --iters 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:tcg_update_kernel" -s 1 -c 1 \
    -o $OUT/prof_tcg_update_$TAG python tools/prof_tcg.py --iters 2 > $OUT/ncu_tcg_$TAG.log 2>&1
# optional (QUALITY=1): the NEXT-3 quality study up to D23 and the D23 per-component breakdown
if [ "${QUALITY:-0}" = "1" ]; then
  timeout 1800 python tools/quality_study.py D16 D20 D21 D22 D23 > $OUT/quality_$TAG.jsonl 2> $OUT/quality_$TAG.err
  timeout 900 python tools/solver_breakdown.py D23 --k 4 --sched 2.0,1.6,1.2 --graphs > $OUT/breakdown_d23_$TAG.json 2>/dev/null
fi
echo "DONE" > $OUT/round_done_$TAG.txt
