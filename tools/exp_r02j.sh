mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err
python tools/prof_edge.py --reps 3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k "regex:edge_halo_kernel" -s 1 -c 1 -o gpurun_out/prof_edge_r02j python tools/prof_edge.py --reps 3 > gpurun_out/ncu_full_r02j.log 2>&1
bash tools/sanitize.sh
