mkdir -p gpurun_out
python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02o.log 2>&1
python tools/tune_edge.py run prod2 > gpurun_out/tune_r02o.log 2>&1
PLP_LIB=paper_2605_26975_b200/variants/prod2trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02o_prod2.json 2>&1
PLP_LIB=paper_2605_26975_b200/variants/prod2/libplp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py -q -x -p no:cacheprovider -k "not alternative and not agree" > gpurun_out/par_r02o_prod2.log 2>&1
