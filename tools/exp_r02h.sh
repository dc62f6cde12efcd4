mkdir -p gpurun_out
for T in 224 120; do
  PLP_ORDER_TILE=$T python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02h_T$T.log 2>&1
  PLP_ORDER_TILE=$T python tools/tune_edge.py run t224b3 > gpurun_out/tune_r02h_T$T.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py tests/test_gpu_collective.py -q -p no:cacheprovider -k "C5t or D16t or hessvec or collective" > gpurun_out/par_r02h.log 2>&1
python tools/prof_edge.py --reps 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:edge_halo_kernel" -s 1 -c 1 -o gpurun_out/prof_edge_r02h python tools/prof_edge.py --reps 3 > gpurun_out/ncu_full_r02h.log 2>&1
