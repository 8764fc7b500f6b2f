# Round-end evidence: full bench line, reference arm, launch list, ncu captures.
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout -s KILL 240 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/rt_tests.log 2>&1; echo "tests rc=$? $(tail -1 gpurun_out/rt_tests.log)"
timeout -s KILL 600 python bench.py > gpurun_out/rt_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/rt_bench.log
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rt_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/rt_ref.log | cut -c1-400
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout -s KILL 300 $B > gpurun_out/rt_b1.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rt_launches.csv $B > gpurun_out/rt_ncu1.log 2>&1; echo "list rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:filter_tc -s 27 -c 1 -o gpurun_out/rt_filter $B > gpurun_out/rt_ncu2.log 2>&1; echo "ncu filter rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:select -s 27 -c 1 -o gpurun_out/rt_select $B > gpurun_out/rt_ncu3.log 2>&1; echo "ncu select rc=$?"
