export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/stageC.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/stageC.log
for R in 2 4; do
QA_B200_RATIO=$R timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r$R.log 2>&1; echo "bench ratio $R rc=$?"
tail -1 gpurun_out/bench_r$R.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), round(r['achieved'],1), round(r['filter_ms_per_step'],3), round(r['select_ms_per_step'],3), r['scan_stats'], d['parity_spot_check'])"
done
