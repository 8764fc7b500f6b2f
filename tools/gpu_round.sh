# Round evidence on one B200 box: GPU tests, the driver's bench lines (both
# arms), the other BASELINE configs, encode throughput, the cfg2 launch list
# and ncu captures of the final filter pass and of the encode.
#   TAG=r02 bash tools/gpu_round.sh        (outputs under gpurun_out/${TAG}_*)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${TAG:-r}
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${T}_bench.log | head -c 1200; echo
timeout -s KILL 300 python bench.py --impl reference --steps 3 > gpurun_out/${T}_ref.log 2>&1; echo "ref rc=$?"
timeout -s KILL 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/${T}_cfg1.log 2>&1; echo "cfg1 rc=$?"
timeout -s KILL 600 python bench.py --config 0 --no-cpu-baseline > gpurun_out/${T}_cfg0.log 2>&1; echo "cfg0 rc=$?"
timeout -s KILL 900 python tools/bench_configs.py --config 4 > gpurun_out/${T}_cfg4.log 2>&1; echo "cfg4 rc=$?"
grep '^{' gpurun_out/${T}_cfg4.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['metric'], d['k'], d['batch'], round(d['p50_ms'],4), d.get('graph_result_equals_sync_search'))"
timeout -s KILL 1500 python tools/bench_configs.py --config 3 > gpurun_out/${T}_cfg3.log 2>&1; echo "cfg3 rc=$?"
grep '^{' gpurun_out/${T}_cfg3.log | tail -1 | head -c 900; echo
python tools/bench_encode.py 100 128 256 > gpurun_out/${T}_encode.jsonl 2>&1; cat gpurun_out/${T}_encode.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_cfg2.csv python tools/diag_l2.py 2 1000000 1024 1 > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_list.py gpurun_out/${T}_launches_cfg2.csv | tee gpurun_out/${T}_launch_summary.txt
TAG=${T}_cfg2_final SKIP=3 bash tools/gpu_ncu.sh
timeout -s KILL 600 ncu --set full --import-source on --clock-control none -k regex:encode_staged --launch-skip 3 --launch-count 1 -o gpurun_out/${T}_encode256 -f python tools/bench_encode.py 256 > gpurun_out/${T}_encode_ncu.log 2>&1; echo "ncu encode rc=$?"
timeout -s KILL 200 python tools/stress_encode.py 60 21 2>&1 | tail -1
timeout -s KILL 300 python tools/stress.py 120 21 2>&1 | tail -1
