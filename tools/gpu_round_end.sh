#!/bin/bash
# Final evidence of a round: gpu_final.sh (tests, smoke, bench lines, ncu
# summaries, sha-stamped C5 traffic, launch list) + the fuzz suite at
# FUZZ_SCALE x its default case counts.
set -u
T=${1:-r02z}
bash tools/gpu_final.sh $T
B64_FUZZ_SCALE=${FUZZ_SCALE:-10} B64_FUZZ_SEED=7 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/${T}_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/${T}_fuzz.log
