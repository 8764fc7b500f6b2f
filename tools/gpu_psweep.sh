export PYTHONUNBUFFERED=1
summ() { tail -1 $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('q/s', round(d['value']), 'ms', round(d['ms_per_step'],3), 'filter', round(r['filter_ms_per_step'],3), 'select', round(r['select_ms_per_step'],3), 'e2e', round(d['e2e']['value']), d['parity_spot_check']['ids_equal'])"; }
for P in 32768 65536 131072; do
  echo "=== P=$P"
  env QA_B200_EST_ROWS=$P timeout -s KILL 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/p.log 2>&1; echo -n "cfg2 "; summ gpurun_out/p.log
  env QA_B200_EST_ROWS=$P timeout -s KILL 300 python bench.py --config 1 --no-cpu-baseline --steps 5 > gpurun_out/p.log 2>&1; echo -n "cfg1 "; summ gpurun_out/p.log
  env QA_B200_EST_ROWS=$P timeout -s KILL 600 python tools/bench_configs.py --config 4 > gpurun_out/p4.log 2>&1
  grep '^{' gpurun_out/p4.log | python -c "
import json,sys
print(' '.join(f\"{d['metric']}/k{d['k']}/b{d['batch']}:{d['p50_ms']:.3f}\" for d in map(json.loads, sys.stdin)))"
done
