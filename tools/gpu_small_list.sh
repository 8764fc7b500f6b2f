export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/small_one.py 0 10 1"
timeout -s KILL 300 $C > gpurun_out/sl_plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv $C > gpurun_out/sl_ncu.log 2>&1; echo "rc=$?"
