# A/B of env settings on one cfg2 1024-query search: "NAME=VAL ..." per arg
export PYTHONUNBUFFERED=1
for v in "$@"; do
  for r in 1 2; do
    env $v timeout -s KILL 300 python tools/diag_l2.py 2 1000000 1024 ${METRICS:-1} 2>&1 | grep '"cfg"' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'filter_ms', round(d['filter_ms'],3), 'select_ms', round(d['select_ms'],3), 'cands', d['candidates'], 'retries', d['retries'])"
  done
done
