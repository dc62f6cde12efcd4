mkdir -p gpurun_out
for c in C5 C3; do python tools/prof_edge.py --config $c --reps 20 --events > gpurun_out/prof_r02r_$c.log 2>&1; done
python -c "
import sys; sys.path.insert(0,'.')
from paper_2605_26975_b200 import plp
import tools.prof_edge" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hessvec.py tests/test_gpu_collective.py -q -x -p no:cacheprovider > gpurun_out/par_r02r.log 2>&1
