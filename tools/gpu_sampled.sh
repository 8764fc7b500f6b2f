# sampled estimate: tests, cfg2 bench at several sample sizes, cfg1, cfg4 lines
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/s_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s_tests.log
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('q/s', round(d['value']), 'ms', round(d['ms_per_step'],3), 'filter', round(r['filter_ms_per_step'],3), 'select', round(r['select_ms_per_step'],3), r['scan_stats'], 'e2e', round(d['e2e']['value']), d['parity_spot_check'])"; }
for P in 32768 65536 16384; do
  env QA_B200_EST_ROWS=$P timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/s_bench.log 2>&1; echo "P=$P bench rc=$?"; summ gpurun_out/s_bench.log
done
env QA_B200_TRACE=0 timeout -s KILL 300 python tools/diag_times.py 2 1000000 1024 2>&1 | grep -v "^  \|Warn" | tail -8
timeout -s KILL 300 python bench.py --config 1 --no-cpu-baseline --steps 5 > gpurun_out/s_bench1.log 2>&1; echo "cfg1 rc=$?"; summ gpurun_out/s_bench1.log
timeout -s KILL 600 python tools/bench_configs.py --config 4 > gpurun_out/s_cfg4.log 2>&1; echo "cfg4 rc=$?"
grep '^{' gpurun_out/s_cfg4.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['metric'], d['k'], d['batch'], round(d['p50_ms'],4), d.get('graph_result_equals_sync_search'))"
