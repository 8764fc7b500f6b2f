export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
timeout -s KILL 600 python tools/bench_configs.py --config 4 --iters 30 --parity-rows 2 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"; python -c "
import json
for l in open('gpurun_out/cfg4.jsonl'):
    j=json.loads(l); print(j['metric'], j['k'], j['batch'], round(j['p50_ms'],3), round(j['roofline']['frac'],3), j['scan_stats'], j.get('parity_spot_check',{}).get('ids_equal'))
"; tail -2 gpurun_out/cfg4.err
