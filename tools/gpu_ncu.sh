# ncu --set full capture of one filter launch (the final pass of a search):
#   CFG=2 N=1000000 NQ=1024 METRIC=1 SKIP=2 TAG=x bash tools/gpu_ncu.sh
# (SKIP = filter launches to skip; diag_l2 runs the search twice)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
C="python tools/diag_l2.py ${CFG:-2} ${N:-1000000} ${NQ:-1024} ${METRIC:-1}"
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:filter_tc \
  --launch-skip ${SKIP:-2} --launch-count 1 -o gpurun_out/${TAG:-filter} -f $C \
  > gpurun_out/${TAG:-filter}_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG:-filter}_ncu.log
