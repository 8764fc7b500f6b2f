# Round-2 decomposition of the cfg2 (L2, 1M x 128, 1024 queries) filter pass.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/diag_l2.py 2 1000000 1024 1"
QA_B200_TRACE=1 timeout -s KILL 300 $C > gpurun_out/d2_trace.log 2>&1; echo "trace rc=$?"
QA_B200_LIB=abtest/wst/libqa_b200.so timeout -s KILL 300 $C > gpurun_out/d2_wst.log 2>&1; echo "wst rc=$?"
for e in 0 2 8; do
  QA_B200_EXPERIMENT=$e timeout -s KILL 300 $C > gpurun_out/d2_e$e.log 2>&1 && \
  QA_B200_EXPERIMENT=$e timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d2_launch_e$e.csv $C > gpurun_out/d2_ncu_e$e.log 2>&1; echo "e$e rc=$?"
done
