set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
export PYTHONUNBUFFERED=1
QA_B200_FILTER=simt timeout -s KILL 400 python -m pytest tests/test_gpu_parity.py -x -q -k "encode or minmax or norms or scan_golden or gate2 or hand" > gpurun_out/stageA.log 2>&1; echo "stageA rc=$?"
tail -5 gpurun_out/stageA.log
timeout -s KILL 200 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core_dots" > gpurun_out/stageB.log 2>&1; echo "stageB rc=$?"
tail -30 gpurun_out/stageB.log
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/stageC.log 2>&1; echo "stageC rc=$?"
tail -40 gpurun_out/stageC.log
