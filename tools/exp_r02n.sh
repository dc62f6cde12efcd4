mkdir -p gpurun_out
python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02n.log 2>&1
python tools/tune_edge.py run nogather > gpurun_out/tune_r02n.log 2>&1
PLP_LIB=paper_2605_26975_b200/variants/trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02n.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py tests/test_gpu_collective.py -q -x -p no:cacheprovider > gpurun_out/par_r02n.log 2>&1
