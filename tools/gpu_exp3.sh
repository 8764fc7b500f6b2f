export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
QA_B200_EXPERIMENT=2 timeout -s KILL 600 $B > gpurun_out/bx2.log 2>&1 && \
QA_B200_EXPERIMENT=2 timeout -s KILL 900 ncu --set full --clock-control none -k regex:filter_tc -s 25 -c 1 -o gpurun_out/prof_exp2 $B > gpurun_out/ncu_e2.log 2>&1; echo "rc=$?"
