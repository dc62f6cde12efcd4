#!/bin/bash
# The deferred re-projection's own GPU tests, the tile-ordered end-to-end checks, then the fused
# tCG A/B against the pre-change library (variants/tcg_old).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_solver.py -m gpu -q -p no:cacheprovider \
    -k "deferred_reprojection or tile_ordered or graph_replay" > gpurun_out/tcg_tests_r02p.log 2>&1
echo "TESTS_RC=$?" >> gpurun_out/tcg_tests_r02p.log
bash tools/tcg_ab.sh tcg_old
