set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCUF="ncu --set full --clock-control none --import-source on"
B2="python bench.py --workload c2 --steps 1 --warmup 3"
$B2 > /dev/null 2>&1
timeout 600 $NCUF -k regex:"batch_kernel" -s 4 -c 1 -o gpurun_out/encd0 -f $B2 > /dev/null 2>&1; echo "ncu0 rc=$?"
B64GPU_LIB=build/variants/libb64gpu_b_encd1.so timeout 600 $NCUF -k regex:"batch_kernel" -s 4 -c 1 -o gpurun_out/encd1 -f $B2 > /dev/null 2>&1; echo "ncu1 rc=$?"
