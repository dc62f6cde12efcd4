mkdir -p gpurun_out
python tools/tune_edge.py run t192 t128c2 > gpurun_out/tune_r02l.log 2>&1
PLP_LIB=paper_2605_26975_b200/variants/t192trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02l_t192.json 2>&1
PLP_LIB=paper_2605_26975_b200/variants/checked/libplp.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py -q -x -p no:cacheprovider -k "not alternative and not agree" > gpurun_out/checked_r02l.log 2>&1
