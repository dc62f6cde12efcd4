mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02f.log 2>&1
timeout 600 python -m pytest tests/test_gpu_collective.py -q -x -p no:cacheprovider > gpurun_out/coll_r02f.log 2>&1
for T in 224 120; do PLP_ORDER_TILE=$T python tools/prof_edge.py --reps 20 --events > gpurun_out/prof_r02f_T$T.log 2>&1; done
python tools/prof_edge.py --reps 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:edge_halo_kernel" -s 1 -c 1 -o gpurun_out/prof_edge_r02f python tools/prof_edge.py --reps 3 > gpurun_out/ncu_full_r02f.log 2>&1
