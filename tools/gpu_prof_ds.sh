#!/bin/bash
# ncu --set full of the two despace kernels (bench --workload despace) + launch times.
set -u
T=${1:-ds}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || exit 1
B="python bench.py --workload despace --steps 2 --warmup 3"
$B > gpurun_out/${T}_plain.json 2>&1 || { echo plain failed; tail gpurun_out/${T}_plain.json; exit 1; }
cat gpurun_out/${T}_plain.json
ncu --set full --clock-control none --import-source on -k regex:despace -s 6 -c 2 -o gpurun_out/${T}_ds -f $B > gpurun_out/${T}_ncu.log 2>&1
echo ncu rc=$?
