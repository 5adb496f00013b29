#!/bin/bash
# A/B run of the one-pass compaction kernels (f3 despace, f4 general ws
# decode): build, the despace / ws / fuzz / >4 GiB MIME tests, bench lines,
# and (NCU=1) one ncu --set full capture of each one-pass kernel.
set -u
T=${1:-op}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_despace.py tests/test_gpu_ws.py tests/test_gpu_fuzz.py ${EXTRA_TESTS:-} -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
for w in despace mime_irregular; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err; echo "bench $w rc=$?"
done
if [ "${NCU:-0}" = "1" ]; then
  NCUF="ncu --set full --clock-control none --import-source on"
  timeout 600 $NCUF -k regex:"despace1" -s 3 -c 1 -o gpurun_out/${T}_ncu_ds -f python bench.py --workload despace --steps 1 --warmup 3 > gpurun_out/${T}_ncu_ds.log 2>&1; echo "ncu ds rc=$?"
  timeout 600 $NCUF -k regex:"decode_ws1" -s 3 -c 1 -o gpurun_out/${T}_ncu_ws -f python bench.py --workload mime_irregular --steps 1 --warmup 3 > gpurun_out/${T}_ncu_ws.log 2>&1; echo "ncu ws rc=$?"
fi
