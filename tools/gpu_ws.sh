export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
QA_B200_LIB=abtest/ws/libqa_b200.so timeout -s KILL 300 python tools/small_one.py 0 10 1 > gpurun_out/ws_small.log 2>&1; echo "rc=$?"; grep wst gpurun_out/ws_small.log | tail -6
QA_B200_LIB=abtest/ws/libqa_b200.so QA_B200_MAXSTAGES=6 timeout -s KILL 300 python tools/small_one.py 0 10 1 > gpurun_out/ws_small6.log 2>&1; echo "rc=$?"; grep wst gpurun_out/ws_small6.log | tail -2
