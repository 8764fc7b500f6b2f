export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/small_one.py 0 10 1"
timeout -s KILL 300 $C > gpurun_out/ss_plain.log 2>&1 && \
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:select_reg -s 9 -c 3 -o gpurun_out/prof_ssel $C > gpurun_out/ss_ncu.log 2>&1; echo "rc=$?"
