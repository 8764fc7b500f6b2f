# round-2 evidence for the non-headline configs
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/r02_cfg1.log 2>&1; echo "cfg1 rc=$?"
timeout -s KILL 1500 python tools/bench_configs.py --config 3 > gpurun_out/r02_cfg3.log 2>&1; echo "cfg3 rc=$?"
tail -c 400 gpurun_out/r02_cfg1.log
tail -c 600 gpurun_out/r02_cfg3.log
