export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 600 $B > gpurun_out/b2.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 27 -c 1 -o gpurun_out/prof_filter2 $B > gpurun_out/ncu2.log 2>&1; echo "ncu-full rc=$?"
tail -2 gpurun_out/ncu2.log
