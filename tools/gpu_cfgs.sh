# Extra-config measurements: cfg2 batched, cfg4 small batch, cfg3 60M IP.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python tools/bench_configs.py --config 2 > gpurun_out/cfg2.jsonl 2> gpurun_out/cfg2.err; echo "cfg2 rc=$?"; cut -c1-600 gpurun_out/cfg2.jsonl; tail -3 gpurun_out/cfg2.err
timeout -s KILL 900 python tools/bench_configs.py --config 4 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"; cut -c1-400 gpurun_out/cfg4.jsonl; tail -3 gpurun_out/cfg4.err
timeout -s KILL 900 python tools/bench_configs.py --config 3 --parity-rows 1 > gpurun_out/cfg3.jsonl 2> gpurun_out/cfg3.err; echo "cfg3 rc=$?"; cut -c1-900 gpurun_out/cfg3.jsonl; tail -3 gpurun_out/cfg3.err
