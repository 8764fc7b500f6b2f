export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 300 $B > gpurun_out/s0_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select_reg -s 9 -c 1 -o gpurun_out/prof_sel0 $B > gpurun_out/s0_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/s0_ncu.log
