export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
bash tools/gpu_wst.sh
grep "^wst cta\|filter\|select" gpurun_out/wst.log | grep -v wstc | tail -30
