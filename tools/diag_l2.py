"""Diagnostics: per-round trace and scan stats of one search (L2/IP on the
sift-like law, angular on the glove-like law)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2110_08919_b200 as qa
import synth
from paper_2110_08919_b200 import _lib

cfg = int(sys.argv[1]); n = int(sys.argv[2]); nq = int(sys.argv[3])
metrics = [int(m) for m in sys.argv[4].split(",")] if len(sys.argv) > 4 else [synth.CONFIGS[cfg]["metric"]]
X, Q = synth.generate(cfg, n=n, nq=nq)
x = torch.from_numpy(X).cuda()
for m in metrics:
    idx = qa.Int8Index.build(x, qa.Metric(m), synth.CONFIGS[cfg]["calibration"])
    qc = idx.encode_queries(torch.from_numpy(Q).cuda())
    idx.search_codes(qc, 100); torch.cuda.synchronize()
    _lib.set_profiling(True)
    t0 = time.time(); idx.search_codes(qc, 100); torch.cuda.synchronize(); dt = time.time() - t0
    st = _lib.last_scan_stats(); _lib.set_profiling(False)
    print(json.dumps({"cfg": cfg, "n": n, "nq": nq, "metric": m, "wall_ms": dt * 1e3, **st}), flush=True)
    sq = idx.codes.sqnorm.cpu().numpy()
    print("  sqnorm min/median/max", sq.min(), np.median(sq), sq.max(), " q sqnorm", qc.sqnorm.cpu().numpy()[:4], flush=True)
