#!/bin/bash
# Batched kernels: build, batched / variants / fuzz / graph tests, C2 bench lines.
set -u
T=${1:-bt}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_batch_shard.py tests/test_gpu_graph.py tests/test_gpu_fuzz.py tests/test_gpu_configs.py -x -q -k "batch or c2 or graph or fuzz" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
for r in 1 2 3; do
  timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 > gpurun_out/${T}_bench_c2_$r.json 2> gpurun_out/${T}_bench_c2_$r.err
  python -c "import json;d=json.load(open('gpurun_out/${T}_bench_c2_$r.json'));print('c2', d['detail']['encode_ms'], d['detail']['decode_ms'], d['detail']['graph_replay_ms'], d['roofline']['frac'])"
done
if [ -n "${VARIANTS:-}" ]; then
  python tools/sweep.py run --workload c2 --steps 20 --reps ${REPS:-3} $VARIANTS > gpurun_out/${T}_sweep.log 2>&1; cut -c1-230 gpurun_out/${T}_sweep.log
fi
