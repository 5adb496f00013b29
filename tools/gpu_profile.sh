#!/bin/bash
# Run on the GPU box (via gpurun): plain bench on C3, then one ncu --set full
# capture of each codec kernel on the same command, plus the launch list of
# the default bench command.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${1:-prof}
B="python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/${TAG}_c3plain.json 2>&1 || { echo "plain c3 run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:encode_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_enc_c3 -f $B > gpurun_out/${TAG}_ncu_enc.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_dec_c3 -f $B > gpurun_out/${TAG}_ncu_dec.log 2>&1
if [ "${LAUNCHES:-1}" = "1" ]; then
  D="python bench.py --steps 10"
  $D > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/${TAG}_launches.csv $D > gpurun_out/${TAG}_ncu_launch.log 2>&1
fi
echo profile-done
