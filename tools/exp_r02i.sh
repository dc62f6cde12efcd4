mkdir -p gpurun_out
for T in 120 224; do
  PLP_ORDER_TILE=$T python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02i_T$T.log 2>&1
  PLP_ORDER_TILE=$T python tools/tune_edge.py run t224b3 t160b3 sleep0 > gpurun_out/tune_r02i_T$T.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py tests/test_gpu_collective.py -q -p no:cacheprovider > gpurun_out/par_r02i.log 2>&1
