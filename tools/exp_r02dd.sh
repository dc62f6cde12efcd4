mkdir -p gpurun_out
for T in 120 224; do
  PLP_ORDER_TILE=$T python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02dd_T$T.log 2>&1
  PLP_ORDER_TILE=$T python tools/tune_edge.py run pfl2 gfirst gfirstpf > gpurun_out/tune_r02dd_T$T.log 2>&1
done
