#!/bin/bash
# One ncu --set full capture of the kernels matching REGEX in one bench workload.
#   tools/gpu_ncu1.sh TAG WORKLOAD REGEX [SKIP] [COUNT]
set -u
T=$1; W=$2; K=$3; SK=${4:-3}; C=${5:-1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --workload $W --steps 2 --warmup 3 > gpurun_out/${T}_plain.json 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${T}_plain.json; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SK -c $C -o gpurun_out/${T} -f \
  python bench.py --workload $W --steps 1 --warmup 3 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
