export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_stats.py -x -q > gpurun_out/stats_tests.log 2>&1; echo "stats tests rc=$? $(tail -1 gpurun_out/stats_tests.log)"; grep -E "Error|assert|Mismatch|x:|y:|name" gpurun_out/stats_tests.log | head -30
timeout -s KILL 600 python -m pytest tests -m gpu -q > gpurun_out/ck_tests.log 2>&1; echo "all gpu tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"
