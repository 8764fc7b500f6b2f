export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
AB_REPS=2 timeout -s KILL 900 python tools/ab.py base: est2off:QA_B200_EST2=0
QA_B200_TRACE=1 timeout -s KILL 300 python tools/diag_l2.py 1 1000000 10000 2 > gpurun_out/diag1.log 2>&1; grep -v qa_trace gpurun_out/diag1.log | cut -c1-300; grep qa_trace gpurun_out/diag1.log | tail -4
timeout -s KILL 600 python tools/bench_configs.py --config 2 --steps 2 > gpurun_out/cfg2.jsonl 2> gpurun_out/cfg2.err; echo "cfg2 rc=$?"; cut -c1-300 gpurun_out/cfg2.jsonl
timeout -s KILL 600 python tools/bench_configs.py --config 4 --iters 30 --parity-rows 1 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"; python -c "
import json
for l in open('gpurun_out/cfg4.jsonl'):
    j=json.loads(l); print(j['metric'], j['k'], j['batch'], round(j['p50_ms'],3), round(j['roofline']['frac'],3), j['scan_stats'], j.get('parity_spot_check',{}).get('ids_equal'))
"
