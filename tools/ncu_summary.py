"""Summarise an ncu report: headline metrics + top SASS lines by stall samples."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def run(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = ("Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Executed Instructions", "Avg. Active Threads Per Warp",
        "No Eligible", "Warp Cycles Per Issued Instruction")
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>20s} {d['Metric Unit']}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
names, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
for n, v in zip(names, vals):
    if n in ("dram__bytes_read.sum", "dram__bytes_write.sum",
             "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
             "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
             "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active"):
        print(f"{n:70s} {v}")
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
stall = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
agg = {c: sum(int(d[c] or 0) for d in data) for c in stall}
print("stall totals:", ", ".join(f"{c[6:]}={v*100//max(tot,1)}%" for c, v in
                                 sorted(agg.items(), key=lambda x: -x[1])[:8]))
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:ntop]
for d in top:
    st = sorted(((c[6:], int(d[c] or 0)) for c in stall), key=lambda x: -x[1])[:2]
    print(f"{d['Address'][-5:]} {d['Source'][:58]:58s} {d['Warp Stall Sampling (All Samples)']:>7s}"
          f" ex={d['Instructions Executed']:>10s} {st}")
