# GPU tests + the driver's bench lines (both arms) on one box.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
T=${TAG:-r}
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"
timeout -s KILL 600 python bench.py > gpurun_out/${T}_bench.log 2>&1; echo "bench rc=$?"
timeout -s KILL 300 python bench.py --impl reference --steps 3 > gpurun_out/${T}_ref.log 2>&1; echo "ref rc=$?"
tail -3 gpurun_out/${T}_tests.log; tail -c 3000 gpurun_out/${T}_bench.log; tail -c 1500 gpurun_out/${T}_ref.log
