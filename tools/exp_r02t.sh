mkdir -p gpurun_out
for i in 1 2; do python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02t_$i.log 2>&1; done
PLP_LIB=paper_2605_26975_b200/variants/trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02t.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py tests/test_gpu_collective.py -q -x -p no:cacheprovider > gpurun_out/par_r02t.log 2>&1
