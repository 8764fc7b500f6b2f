export PYTHONUNBUFFERED=1
for v in QA_B200_UNIT_TABLE=0 QA_B200_UNIT_TABLE=1; do
echo "== $v"
env $v timeout -s KILL 600 python tools/bench_configs.py --config 4 > gpurun_out/s_cfg4.log 2>&1; echo "cfg4 rc=$?"
grep '^{' gpurun_out/s_cfg4.log | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['metric'], d['k'], d['batch'], round(d['p50_ms'],4))" | grep l2
done
