set -u
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi_r02n.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > $OUT/gpu_tests_r02n.log 2>&1
echo "TESTS_RC=$?" >> $OUT/gpu_tests_r02n.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_r02n.log 2>&1; echo "SMOKE_RC=$?" >> $OUT/smoke_r02n.log
python bench.py --steps 20 --warmup 5 > $OUT/bench_r02n.json 2> $OUT/bench_r02n.err; echo "BENCH_RC=$?" >> $OUT/bench_r02n.err
