export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
for ex in 0 4 6; do
QA_B200_EXPERIMENT=$ex QA_B200_LIB=abtest/ws/libqa_b200.so timeout -s KILL 200 python tools/small_one.py 0 10 1 > gpurun_out/ws_ex$ex.log 2>&1; echo "ex=$ex rc=$?"; grep wst gpurun_out/ws_ex$ex.log | awk '{print $2, $3, $4, $5, $6, $7, $8, $9, $10}' | sort -t= -k3 -n | tail -2
done
