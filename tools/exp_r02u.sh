mkdir -p gpurun_out
python tools/prof_edge.py --config C4 --reps 10 --events > gpurun_out/prof_r02u_C4.log 2>&1
python tools/tune_edge.py run k20u4 k20u12 --config C4 > gpurun_out/tune_r02u.log 2>&1
python tools/prof_edge.py --config C5 --reps 20 --events > gpurun_out/prof_r02u_C5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "C4s or k20 or 20" > gpurun_out/par_r02u.log 2>&1
