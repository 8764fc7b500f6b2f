export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests -m gpu -x -q > gpurun_out/ck_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/ck_tests.log)"; grep -E "FAIL|Error|assert" gpurun_out/ck_tests.log | head -20
AB_REPS=3 timeout -s KILL 900 python tools/ab.py old:QA_B200_LIB=abtest/old/libqa_b200.so new:
