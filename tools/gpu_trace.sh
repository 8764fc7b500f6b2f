export PYTHONUNBUFFERED=1
for R in 2 4; do
QA_B200_RATIO=$R QA_B200_TRACE=1 timeout -s KILL 600 python tools/trace.py > gpurun_out/trace_r$R.log 2>&1; echo "trace ratio $R rc=$?"
sed -n '/traced search/,$p' gpurun_out/trace_r$R.log
done
