export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout -s KILL 600 $B > gpurun_out/bl.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncul.log 2>&1; echo "rc=$?"
