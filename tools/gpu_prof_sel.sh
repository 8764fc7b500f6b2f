# usage: bash tools/gpu_prof_sel.sh TAG SKIP  -> gpurun_out/prof_TAG.ncu-rep (select kernel #SKIP)
export PYTHONUNBUFFERED=1
tag=$1; skip=$2; shift; shift
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
env "$@" timeout -s KILL 300 $B > gpurun_out/bp_$tag.log 2>&1 && \
env "$@" timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select -s $skip -c 1 -o gpurun_out/prof_$tag $B > gpurun_out/ncup_$tag.log 2>&1; echo "prof $tag rc=$?"
