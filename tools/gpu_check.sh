#!/bin/bash
# GPU box: build, gpu tests, smoke, bench lines for every workload.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${1:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { echo build failed; tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
for w in ${WORKLOADS:-despace c2 c4 c1}; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err; echo "bench $w rc=$?"
done
if [ "${DEFAULT:-1}" = "1" ]; then
  timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench default rc=$?"
fi
echo check-done
