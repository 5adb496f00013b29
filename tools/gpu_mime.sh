#!/bin/bash
# MIME kernels: build, ws / wrap / fuzz / >4 GiB tests, A/B of variants on the mime workload.
set -u
T=${1:-mm}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_ws.py tests/test_gpu_wrap.py tests/test_gpu_fuzz.py tests/test_gpu_mime_large.py -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
if [ -n "${VARIANTS:-}" ]; then
  python tools/sweep.py run --workload mime --steps 10 --reps ${REPS:-2} $VARIANTS > gpurun_out/${T}_sweep.log 2>&1; cat gpurun_out/${T}_sweep.log | cut -c1-220
fi
