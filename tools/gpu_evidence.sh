# Round evidence: bench line (+cpu baseline), reference arm, extra configs, launch list, ncu captures.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -q > gpurun_out/ev_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ev_tests.log)"
timeout -s KILL 600 python bench.py > gpurun_out/ev_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/ev_bench.log | cut -c1-300
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/ev_ref.log | cut -c1-300
timeout -s KILL 600 python tools/bench_configs.py --config 2 --steps 3 > gpurun_out/ev_cfg2.jsonl 2> gpurun_out/ev_cfg2.err; echo "cfg2 rc=$?"
timeout -s KILL 900 python tools/bench_configs.py --config 3 --parity-rows 1 > gpurun_out/ev_cfg3.jsonl 2> gpurun_out/ev_cfg3.err; echo "cfg3 rc=$?"
timeout -s KILL 900 python tools/bench_configs.py --config 4 --iters 200 --parity-rows 2 > gpurun_out/ev_cfg4.jsonl 2> gpurun_out/ev_cfg4.err; echo "cfg4 rc=$?"
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 300 $B > gpurun_out/ev_b1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $B > gpurun_out/ev_ncu1.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 11 -c 1 -o gpurun_out/ev_filter $B > gpurun_out/ev_ncu2.log 2>&1; echo "ncu filter rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select -s 11 -c 1 -o gpurun_out/ev_select $B > gpurun_out/ev_ncu3.log 2>&1; echo "ncu select rc=$?"
