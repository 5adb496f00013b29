#!/bin/bash
# Round-end evidence in one call, small enough to come back through gpurun:
# tests + smoke + every bench line (gpu_check.sh), the ncu captures of
# gpu_profile_all.sh reduced to their JSON summaries (the .ncu-rep files
# are deleted on the box), the C5 traffic and launch-list CSVs.
set -u
T=${1:-final}
WORKLOADS="c1 c2 c3 c4 despace despace_irregular mime mime_irregular" bash tools/gpu_check.sh $T
bash tools/gpu_profile_all.sh $T
for r in gpurun_out/${T}_*.ncu-rep; do
  [ -f "$r" ] || continue
  b=$(basename $r .ncu-rep)
  python tools/ncu_summary.py $r > gpurun_out/${b}.summary.json 2> /dev/null
  rm -f $r
done
du -sh gpurun_out
echo final-done
