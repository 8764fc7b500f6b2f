export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/diag_l2.py 2 1000000 1024 1"
timeout -s KILL 300 $C > gpurun_out/c2_plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c2_launches.csv $C > gpurun_out/c2_ncu.log 2>&1; echo "rc=$?"; cat gpurun_out/c2_plain.log | cut -c1-300
