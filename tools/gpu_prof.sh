export PYTHONUNBUFFERED=1
export QA_B200_RATIO=${QA_B200_RATIO:-2}
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 600 $B > gpurun_out/b2.log 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo "ncu-list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s ${FSKIP:-51} -c 1 -o gpurun_out/prof_filter4 $B > gpurun_out/ncu2.log 2>&1; echo "ncu-full rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select -s ${SSKIP:-50} -c 1 -o gpurun_out/prof_select4 $B > gpurun_out/ncu3.log 2>&1; echo "ncu-sel rc=$?"
