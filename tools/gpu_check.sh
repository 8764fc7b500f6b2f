# Quick health check: GPU parity tests + a default bench line.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"
timeout -s KILL 600 python bench.py > gpurun_out/ck_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/ck_bench.log
