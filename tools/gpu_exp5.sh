export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/stageC.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/stageC.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout -s KILL 300 $B > gpurun_out/bx_$tag.log 2>&1 && \
  env "$@" timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv $B > gpurun_out/ncux_$tag.log 2>&1; echo "$tag rc=$?"
  python tools/launch_list.py gpurun_out/launches_$tag.csv | head -2
}
run e0 QA_B200_EXPERIMENT=0
run e2 QA_B200_EXPERIMENT=2
run e0s1 QA_B200_EXPERIMENT=0 QA_B200_SCHED=1
run e2s1 QA_B200_EXPERIMENT=2 QA_B200_SCHED=1
