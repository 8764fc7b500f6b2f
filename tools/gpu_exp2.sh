export PYTHONUNBUFFERED=1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
for E in 0 2; do
QA_B200_EXPERIMENT=$E timeout -s KILL 600 $B > gpurun_out/bx$E.log 2>&1 && \
QA_B200_EXPERIMENT=$E timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_e$E.csv $B > gpurun_out/ncux$E.log 2>&1; echo "exp $E rc=$?"
done
