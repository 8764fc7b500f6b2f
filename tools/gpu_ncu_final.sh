# ncu --set full of the final filter pass and the final select of the timed search
export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 300 $B > gpurun_out/rt_b1.log 2>&1; echo "bench rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 27 -c 1 -o gpurun_out/rt_filter $B > gpurun_out/rt_ncu2.log 2>&1; echo "ncu filter rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select -s 27 -c 1 -o gpurun_out/rt_select $B > gpurun_out/rt_ncu3.log 2>&1; echo "ncu select rc=$?"
