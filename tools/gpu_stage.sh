export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/stageC.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/stageC.log
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline']))"
