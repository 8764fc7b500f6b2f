export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
QA_B200_TRACE=1 timeout -s KILL 300 python tools/diag_l2.py 2 1000000 1024 1 > gpurun_out/diag2.log 2>&1; echo "diag2 rc=$?"; grep -v "^qa_trace" gpurun_out/diag2.log | cut -c1-400; grep qa_trace gpurun_out/diag2.log | tail -9
timeout -s KILL 300 python tools/diag_l2.py 1 1000000 10000 2 > gpurun_out/diag1.log 2>&1; echo "diag1 rc=$?"; cut -c1-400 gpurun_out/diag1.log
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/ck_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/ck_bench.log | cut -c1-300
timeout -s KILL 600 python tools/bench_configs.py --config 2 --steps 2 > gpurun_out/cfg2.jsonl 2> gpurun_out/cfg2.err; echo "cfg2 rc=$?"; cut -c1-700 gpurun_out/cfg2.jsonl; tail -3 gpurun_out/cfg2.err
timeout -s KILL 600 python tools/bench_configs.py --config 4 --iters 100 > gpurun_out/cfg4.jsonl 2> gpurun_out/cfg4.err; echo "cfg4 rc=$?"; cut -c1-330 gpurun_out/cfg4.jsonl; tail -3 gpurun_out/cfg4.err
