#!/bin/bash
# Round-end evidence on the GPU box: plain runs first (must exit 0), then
#  * DRAM bytes of the C5 launches (single-pass metrics, no replay of 80 GB)
#    -> profiles/ncu_traffic.json stamped with the source sha (tools/traffic_json.py),
#    BEFORE the default bench, so its roofline.traffic comes from this build
#  * the default bench line and the launch list (gpu__time_duration) of the same command
#  * ncu --set full of encode_kernel / decode_kernel on C3 (one launch each)
#  * ncu --set full of the batched kernels on C2, the f3/f4 kernels (despace fast / general path, mime workloads)
set -u
T=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { echo build failed; exit 1; }
B5="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu"
$B5 > gpurun_out/${T}_c5plain.json 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"(en|de)code_kernel" -s 6 -c 2 --csv --log-file gpurun_out/${T}_c5_traffic.csv $B5 > /dev/null 2>&1
python tools/traffic_json.py gpurun_out/${T}_c5_traffic.csv $T > gpurun_out/${T}_traffic.log 2>&1; echo "traffic rc=$?"
cp profiles/ncu_traffic.json gpurun_out/${T}_ncu_traffic.json
D="python bench.py"
$D > gpurun_out/${T}_bench_plain.json 2> gpurun_out/${T}_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${T}_launches.csv $D > gpurun_out/${T}_ncu_launch.log 2>&1
NCU="ncu --set full --clock-control none --import-source on"
B3="python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu"
$B3 > gpurun_out/${T}_c3plain.json 2>&1 || { echo "c3 plain failed"; exit 1; }
$NCU -k regex:encode_kernel -s 3 -c 1 -o gpurun_out/${T}_enc_c3 -f $B3 > gpurun_out/${T}_ncu_enc.log 2>&1
$NCU -k regex:decode_kernel -s 3 -c 1 -o gpurun_out/${T}_dec_c3 -f $B3 > gpurun_out/${T}_ncu_dec.log 2>&1
B2="python bench.py --workload c2 --steps 1 --warmup 3"
$B2 > gpurun_out/${T}_c2plain.json 2>&1 && \
$NCU -k regex:batch_kernel -s 4 -c 2 -o gpurun_out/${T}_batch_c2 -f $B2 > gpurun_out/${T}_ncu_c2.log 2>&1
BD="python bench.py --workload despace --steps 1 --warmup 3"
$BD > gpurun_out/${T}_dsplain.json 2>&1 && \
$NCU -k regex:"decode_lines" -s 3 -c 1 -o gpurun_out/${T}_despace -f $BD > gpurun_out/${T}_ncu_ds.log 2>&1
BDI="python bench.py --workload despace_irregular --steps 1 --warmup 3"
$BDI > gpurun_out/${T}_dsirrplain.json 2>&1 && \
$NCU -k regex:"cp_mask|despace_kernel" -s 4 -c 2 -o gpurun_out/${T}_despaceirr -f $BDI > gpurun_out/${T}_ncu_dsirr.log 2>&1
BM="python bench.py --workload mime --steps 1 --warmup 3"
$BM > gpurun_out/${T}_mimeplain.json 2>&1 && \
$NCU -k regex:"decode_lines" -s 3 -c 1 -o gpurun_out/${T}_mime -f $BM > gpurun_out/${T}_ncu_mime.log 2>&1
$NCU -k regex:"encode_(wrap|lines)" -s 3 -c 1 -o gpurun_out/${T}_mimeenc -f $BM > gpurun_out/${T}_ncu_mimeenc.log 2>&1
BI="python bench.py --workload mime_irregular --steps 1 --warmup 3"
$BI > gpurun_out/${T}_mimeirrplain.json 2>&1 && \
$NCU -k regex:"cp_mask|decode_ws" -s 6 -c 2 -o gpurun_out/${T}_mimeirr -f $BI > gpurun_out/${T}_ncu_mimeirr.log 2>&1
for w in c1 c2 c4 despace despace_irregular mime mime_irregular sweep; do
  python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/${T}_bench_$w.json 2> gpurun_out/${T}_bench_$w.err
done
echo profile-all-done
