# usage: bash tools/gpu_list2.sh TAG VAR=VAL ...  -> gpurun_out/launches_TAG.csv
export PYTHONUNBUFFERED=1
tag=$1; shift
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
env "$@" timeout -s KILL 300 $B > gpurun_out/bx_$tag.log 2>&1 && \
env "$@" timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $B > gpurun_out/ncux_$tag.log 2>&1; echo "$tag rc=$?"
