export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 300 $B > gpurun_out/ev_b1.log 2>&1; echo "plain rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 11 -c 1 -o gpurun_out/ev_filter $B > gpurun_out/ev_ncu2.log 2>&1; echo "ncu filter rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select -s 11 -c 1 -o gpurun_out/ev_select $B > gpurun_out/ev_ncu3.log 2>&1; echo "ncu select rc=$?"
