export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/bench.log
timeout -s KILL 600 $B > gpurun_out/b2.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo "ncu-list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 27 -c 1 -o gpurun_out/prof_filter $B > gpurun_out/ncu2.log 2>&1; echo "ncu-full rc=$?"
tail -3 gpurun_out/ncu2.log
