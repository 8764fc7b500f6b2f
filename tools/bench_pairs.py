"""Throughput of the listed-pair distance service (qa_gather_scores_i8): random
candidate lists over a resident int8 database, as a graph traversal's hop
would issue them.  Bytes per pair: ld (the gathered row) + 4 (id) + 8 (score)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08919_b200 import device as dev

n, d = 10_000_000, 128
g = torch.Generator(device="cuda"); g.manual_seed(0)
db = dev.DeviceCodes.empty(n, d)
db.codes.copy_(torch.randint(-128, 128, (n, d), device="cuda", generator=g, dtype=torch.int8))
dev.norms_(db)
for nq, m in [(64, 32), (1024, 32), (8192, 64)]:
    qs = dev.DeviceCodes.empty(nq, d)
    qs.codes.copy_(torch.randint(-128, 128, (nq, d), device="cuda", generator=g, dtype=torch.int8))
    dev.norms_(qs)
    cand = torch.randint(0, n, (nq, m), device="cuda", generator=g, dtype=torch.int32)
    for metric in (1, 0):
        for _ in range(3):
            dev.gather_scores(db, qs, cand, metric)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ts = []
        for _ in range(20):
            ev[0].record(); dev.gather_scores(db, qs, cand, metric); ev[1].record()
            torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
        ms = sorted(ts)[len(ts) // 2]
        by = nq * m * (db.ld + 12)
        print(json.dumps({"n": n, "d": d, "nq": nq, "m": m, "metric": ["ip", "l2"][metric], "ms": ms,
                          "pairs_per_s": nq * m / ms * 1e3, "GBps": by / ms / 1e6}), flush=True)
