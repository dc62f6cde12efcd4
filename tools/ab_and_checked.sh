#!/bin/bash
# A/B of the fused tCG iteration against the tcg_r_every variant (tools/tcg_ab.sh), then the ncu
# launch list of the fused passes (per-pass time and DRAM bytes) of this build.
set -u
mkdir -p gpurun_out
bash tools/tcg_ab.sh tcg_r_every
python tools/prof_tcg.py --iters 4 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/tcg_launches_r02n.csv python tools/prof_tcg.py --iters 4 > /dev/null 2>&1
echo "NCU_RC=$?" > gpurun_out/tcg_launches_r02n.rc
