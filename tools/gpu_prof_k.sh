#!/bin/bash
# ncu --set full of kernels matching $2 in `bench.py --workload $1` (one capture), plus the plain line.
set -u
W=$1; K=$2; T=${3:-pk}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || exit 1
B="python bench.py --workload $W --steps 3 --warmup 3"
$B > gpurun_out/${T}_${W}.json 2>&1 || { echo $W failed; tail gpurun_out/${T}_${W}.json; exit 1; }
tail -1 gpurun_out/${T}_${W}.json | cut -c1-300
ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${SKIP:-3} -c ${COUNT:-1} -o gpurun_out/${T}_${W} -f $B > gpurun_out/${T}_ncu_${W}.log 2>&1
echo ncu rc=$?
