#!/bin/bash
# Plain bench lines + ncu --set full of the compaction kernels (despace, mime workloads).
set -u
T=${1:-cp}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || exit 1
for w in despace mime; do
  B="python bench.py --workload $w --steps 5 --warmup 3"
  $B > gpurun_out/${T}_${w}.json 2>&1 || { echo $w failed; tail gpurun_out/${T}_${w}.json; continue; }
  tail -1 gpurun_out/${T}_${w}.json | cut -c1-600
  ncu --set full --clock-control none --import-source on -k regex:"despace|cp_count|decode_ws" -s 4 -c 2 -o gpurun_out/${T}_${w} -f $B > gpurun_out/${T}_ncu_${w}.log 2>&1
  echo ncu $w rc=$?
done
