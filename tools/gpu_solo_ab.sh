set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/so_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_graph.py -x -q > gpurun_out/so_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/so_pytest.log
python tools/sweep.py run --workload sweep --steps 20 --reps 2 old base_ref > gpurun_out/so_sweep.log 2>&1
python - <<'PY'
import json
rows=json.load(open('gpurun_out/sweep_sweep.json'))
for r in rows:
    c=r['detail']['sweep']
    print(r['variant'], r['rep'], ' '.join(f"{x['n']}:{x['decode_us']:.2f}" for x in c[:12]))
PY
for w in c1 c4; do python tools/sweep.py run --workload $w --steps 20 --reps 2 old base_ref 2>&1 | cut -c1-200; done
