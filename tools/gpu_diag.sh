export PYTHONUNBUFFERED=1
for v in QA_B200_EST_SAMPLED=1 QA_B200_EST_SAMPLED=0; do
  echo "== $v"; env $v QA_B200_TRACE=0 timeout -s KILL 300 python tools/diag_times.py ${CFG:-2} ${N:-1000000} ${NQ:-1024} 2>&1 | grep -v "^  \|Warn" | tail -16
done
