mkdir -p gpurun_out
python tools/tune_edge.py run t256 > gpurun_out/tune_r02p.log 2>&1
PLP_LIB=paper_2605_26975_b200/variants/t256trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02p_t256.json 2>&1
PLP_LIB=paper_2605_26975_b200/variants/trace/libplp.so python tools/trace_halo.py > gpurun_out/trace_r02p.json 2>&1
