export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/stageC.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/stageC.log
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
for E in 0 2 3 4; do
QA_B200_EXPERIMENT=$E timeout -s KILL 600 $B > gpurun_out/bx$E.log 2>&1 && \
QA_B200_EXPERIMENT=$E timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_e$E.csv $B > gpurun_out/ncux$E.log 2>&1; echo "exp $E rc=$?"
done
