export PYTHONUNBUFFERED=1
for P in 32768 65536; do
  echo "== cfg1 P=$P"; QA_B200_EST_ROWS=$P timeout -s KILL 300 python tools/diag_times.py 1 1000000 10000 2>&1 | grep "qa_time\|rounds\|Error" | head -4
  echo "== cfg2 P=$P"; QA_B200_EST_ROWS=$P timeout -s KILL 300 python tools/diag_times.py 2 1000000 1024 2>&1 | grep "qa_time\|rounds\|Error" | head -4
done
