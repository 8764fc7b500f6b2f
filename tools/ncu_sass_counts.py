"""Group SASS instructions of an ncu report by execution count (per-tile vs per-chunk loops)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot = sum(int(d["Instructions Executed"] or 0) for d in data)
print("total warp-instructions", tot)
buckets = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for d in data:
    ex = int(d["Instructions Executed"] or 0)
    if ex == 0:
        continue
    key = ex  # group identical counts
    b = buckets[key]
    b[0] += 1
    b[1] += ex
    b[2][d["Source"].split()[0] if not d["Source"].startswith("@") else d["Source"].split()[1]] += 1
for key, (n, s, ops) in sorted(buckets.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"exec={key:>10d} x{n:4d} instr -> {s/tot*100:5.1f}%  {dict(ops.most_common(8))}")
