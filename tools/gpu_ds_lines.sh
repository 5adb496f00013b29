#!/bin/bash
# Despace line fast path: build, the despace / ws / fuzz tests, bench lines
# (fast path and the general path), and (NCU=1) one ncu --set full capture of
# decode_lines_kernel on NCU_W (default: despace).
set -u
T=${1:-dl}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_despace.py tests/test_gpu_ws.py tests/test_gpu_fuzz.py ${EXTRA_TESTS:-} -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
for w in despace despace_irregular mime mime_irregular; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo "bench $w rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/${T}_bench_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['ms_per_step'],4), d['roofline']['frac'])" 2>/dev/null
done
if [ "${NCU:-0}" = "1" ]; then
  NCUF="ncu --set full --clock-control none --import-source on"
  timeout 600 $NCUF -k regex:"${NCU_K:-decode_lines}" -s ${NCU_S:-1} -c 1 -o gpurun_out/${T}_ncu_${NCU_W:-despace} -f python bench.py --workload ${NCU_W:-despace} --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
fi
