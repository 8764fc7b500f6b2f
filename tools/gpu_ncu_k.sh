# ncu --set full capture of one launch of kernel regex $K in a cfg search:
#   K=select_reg SKIP=0 TAG=x CFG=2 N=1000000 NQ=1024 METRIC=1 bash tools/gpu_ncu_k.sh
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/diag_l2.py ${CFG:-2} ${N:-1000000} ${NQ:-1024} ${METRIC:-1}"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:${K} \
  --launch-skip ${SKIP:-0} --launch-count 1 -o gpurun_out/${TAG:-k} -f $C > gpurun_out/${TAG:-k}_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG:-k}_ncu.log
