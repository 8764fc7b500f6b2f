# per-CTA cycle totals of each filter launch (-DQA_WAIT_STATS build)
export PYTHONUNBUFFERED=1
QA_B200_LIB=gpurun_libs/libqa_ws.so QA_B200_TIMES=1 timeout -s KILL 300 python tools/diag_times.py ${CFG:-2} ${N:-1000000} ${NQ:-1024} > gpurun_out/wst.log 2>&1
python - <<'PY'
import re
L=[l for l in open('gpurun_out/wst.log') if l.startswith('wstc')]
print(len(L), 'wstc lines')
i=0; li=0
while i < len(L):
    grp=L[i:i+148]; i+=148
    tot=sorted(int(re.search(r'total=(\d+)',l).group(1)) for l in grp)
    sv=sorted(int(re.search(r'surv=(\d+)',l).group(1)) for l in grp)
    print(f'launch {li}: total min {tot[0]} p50 {tot[len(tot)//2]} p90 {tot[int(len(tot)*.9)]} max {tot[-1]}  surv min {sv[0]} p50 {sv[len(sv)//2]} max {sv[-1]}')
    li+=1
PY
