# round-2 re-entry evidence at HEAD: GPU tests, cfg2 bench (both arms), cfg1, cfg4, launch list
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${TAG:-c}
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${T}_bench.log | head -c 2500; echo
timeout -s KILL 300 python bench.py --impl reference --steps 3 > gpurun_out/${T}_ref.log 2>&1; echo "ref rc=$?"
timeout -s KILL 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/${T}_cfg1.log 2>&1; echo "cfg1 rc=$?"
timeout -s KILL 900 python tools/bench_configs.py --config 4 > gpurun_out/${T}_cfg4.log 2>&1; echo "cfg4 rc=$?"
grep '^{' gpurun_out/${T}_cfg4.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['metric'], d['k'], d['batch'], round(d['p50_ms'],4), d.get('graph_result_equals_sync_search'))"
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg2.csv python tools/diag_l2.py 2 1000000 1024 1 > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_list.py gpurun_out/${T}_launches_cfg2.csv
