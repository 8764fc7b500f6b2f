export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python tools/bench_configs.py --config 4 --iters 50 --parity-rows 0 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"; python -c "
import json
for l in open('gpurun_out/cfg4.jsonl'):
    j=json.loads(l); print(j['metric'], j['k'], j['batch'], round(j['p50_ms'],3), round(j['roofline']['frac'],3), j['scan_stats'])
"; tail -3 gpurun_out/cfg4.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python tools/bench_configs.py --config 4 --iters 2 --parity-rows 0 --n 10000000 > gpurun_out/small_ncu.log 2>&1; echo "ncu rc=$?"
