export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 300 python tools/diag_l2.py 0 100000 1000 1,0 > gpurun_out/diag0.log 2>&1; echo "diag0 rc=$?"; cat gpurun_out/diag0.log | cut -c1-400
QA_B200_TRACE=1 timeout -s KILL 300 python tools/diag_l2.py 2 1000000 1024 1,0 > gpurun_out/diag2.log 2>&1; echo "diag2 rc=$?"; grep -v "^qa_trace" gpurun_out/diag2.log | cut -c1-400; grep qa_trace gpurun_out/diag2.log | tail -12
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
