mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gpu_tests_r02s.log 2>&1; echo RC=$? >> gpurun_out/gpu_tests_r02s.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02s.json 2> gpurun_out/bench_r02s.err
python bench.py --sharded --steps 10 --warmup 3 --no-cpu --no-variants > gpurun_out/bench_sharded_r02s.json 2> gpurun_out/bench_sharded_r02s.err
for c in C3 C4 D23; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e --no-variants > gpurun_out/bench_r02s_$c.json 2>/dev/null; done
