export PYTHONUNBUFFERED=1
for P in 32768 131072 262144; do
QA_B200_EST_ROWS=$P timeout -s KILL 300 python tools/bench_configs.py --config 4 --iters 30 --parity-rows 1 > gpurun_out/p$P.jsonl 2>&1; echo "P=$P rc=$?"; python -c "
import json
for l in open('gpurun_out/p$P.jsonl'):
    if not l.startswith('{'): continue
    j=json.loads(l)
    if j['batch'] in (1,64): print(j['metric'], j['k'], j['batch'], round(j['p50_ms'],3), round(j['roofline']['frac'],3), j['scan_stats'], j.get('parity_spot_check',{}).get('ids_equal'))
"
done
