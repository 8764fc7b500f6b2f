export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
AB_REPS=2 timeout -s KILL 900 python tools/ab.py base:
QA_B200_TRACE=1 timeout -s KILL 300 python tools/diag_l2.py 1 1000000 10000 2 > gpurun_out/diag1.log 2>&1; grep -v qa_trace gpurun_out/diag1.log | cut -c1-300; grep qa_trace gpurun_out/diag1.log | tail -3
