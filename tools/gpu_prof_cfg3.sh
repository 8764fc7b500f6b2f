export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/bench_configs.py --config 3 --n 20000000 --nq 2048 --parity-rows 0"
timeout -s KILL 300 $C > gpurun_out/c3_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 5 -c 1 -o gpurun_out/prof_cfg3 $C > gpurun_out/c3_ncu.log 2>&1; echo "rc=$?"; cut -c1-400 gpurun_out/c3_plain.log
