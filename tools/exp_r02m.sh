mkdir -p gpurun_out
python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02m.log 2>&1
PLP_LIB=paper_2605_26975_b200/variants/trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02m.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py tests/test_gpu_collective.py -q -x -p no:cacheprovider > gpurun_out/par_r02m.log 2>&1
python tools/prof_edge.py --reps 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:edge_halo_kernel" -s 1 -c 1 -o gpurun_out/prof_edge_r02m python tools/prof_edge.py --reps 3 > gpurun_out/ncu_full_r02m.log 2>&1
