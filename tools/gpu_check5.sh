export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
timeout -s KILL 600 python tools/bench_configs.py --config 4 --iters 50 --parity-rows 2 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"; python -c "
import json
for l in open('gpurun_out/cfg4.jsonl'):
    j=json.loads(l); print(j['metric'], j['k'], j['batch'], round(j['p50_ms'],3), round(j['roofline']['frac'],3), j['scan_stats'], j.get('parity_spot_check'))
"; tail -3 gpurun_out/cfg4.err
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/ck_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/ck_bench.log | cut -c1-250
timeout -s KILL 600 python tools/bench_configs.py --config 2 --steps 2 > gpurun_out/cfg2.jsonl 2> gpurun_out/cfg2.err; echo "cfg2 rc=$?"; cut -c1-400 gpurun_out/cfg2.jsonl; tail -3 gpurun_out/cfg2.err
