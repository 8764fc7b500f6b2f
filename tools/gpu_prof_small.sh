export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/small_one.py 0 10 1"
timeout -s KILL 300 $C > gpurun_out/small_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 9 -c 3 -o gpurun_out/prof_small $C > gpurun_out/small_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/small_ncu.log
