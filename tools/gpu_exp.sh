export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/stageC.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/stageC.log
for R0 in 256 1024 2048 4096; do
QA_B200_R0=$R0 timeout -s KILL 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_r0$R0.log 2>&1; echo "r0 $R0 rc=$?"
tail -1 gpurun_out/bench_r0$R0.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value']), round(d['ms_per_step'],3), round(r['achieved'],1), round(r['filter_ms_per_step'],3), round(r['select_ms_per_step'],3), r['scan_stats'], d['parity_spot_check'])"
done
