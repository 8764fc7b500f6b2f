export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for pf in 0 8 16 32 64; do
QA_B200_L2PF=$pf timeout -s KILL 300 python tools/bench_configs.py --config 4 --iters 30 --parity-rows 1 > gpurun_out/pf$pf.jsonl 2>gpurun_out/pf$pf.err; echo "pf=$pf rc=$?"; python -c "
import json
for l in open('gpurun_out/pf$pf.jsonl'):
    j=json.loads(l)
    if j['batch'] in (1,64): print(j['metric'], j['k'], j['batch'], round(j['p50_ms'],3), round(j['roofline']['frac'],3), round(j['scan_stats']['filter_ms'],3), round(j['scan_stats']['select_ms'],3), j.get('parity_spot_check',{}).get('ids_equal'))
"
done
