export PYTHONUNBUFFERED=1
for v in QA_B200_UNIT_TABLE=1 QA_B200_UNIT_TABLE=0 QA_B200_FINAL_TPU=8; do
  echo "== $v"; env $v timeout -s KILL 300 python tools/diag_times.py 2 1000000 1024 2>&1 | grep "qa_time\|Error" | head -4
done
echo "== cfg1 angular 10k"; timeout -s KILL 300 python tools/diag_times.py 1 1000000 10000 2>&1 | grep "qa_time\|Error" | head -4
echo "== cfg1 angular 10k no table"; QA_B200_UNIT_TABLE=0 timeout -s KILL 300 python tools/diag_times.py 1 1000000 10000 2>&1 | grep "qa_time\|Error" | head -4
