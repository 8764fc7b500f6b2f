# GPU tests + a short cfg2 bench line
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/q_tests.log
timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/q_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('q/s', round(d['value']), 'ms', round(d['ms_per_step'],3), 'filter', round(r['filter_ms_per_step'],3), 'select', round(r['select_ms_per_step'],3), r['scan_stats'], 'e2e', round(d['e2e']['value']), 'api', round(d['e2e_reference_api']['value']), d['parity_spot_check'])"
