export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout -s KILL 300 $B > gpurun_out/bx_$tag.log 2>&1 && \
  env "$@" timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $B > gpurun_out/ncux_$tag.log 2>&1; echo "$tag rc=$?"
}
run e5 QA_B200_EXPERIMENT=5
run e6 QA_B200_EXPERIMENT=6
run e0c2k QA_B200_EXPERIMENT=0 QA_B200_STAGECAP=2048
