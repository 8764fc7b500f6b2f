# per-launch times for a config/metric under env variants: CFG N NQ METRIC then variants
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
cfg=$1; n=$2; nq=$3; m=$4; shift 4
i=0
for v in "$@"; do
  i=$((i+1))
  env $v timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l3_$i.csv python tools/diag_l2.py $cfg $n $nq $m > /dev/null 2>&1
  echo "== cfg$cfg $v"; python tools/launch_list.py gpurun_out/l3_$i.csv
done
