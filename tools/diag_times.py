"""Diagnostics: per-launch filter/select times and per-pass survivors of one
synchronous search (env QA_B200_TIMES / QA_B200_TRACE print them).
usage: diag_times.py CFG N NQ [METRIC] [K]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("QA_B200_TIMES", "1")
import torch
import paper_2110_08919_b200 as qa
import synth
from paper_2110_08919_b200 import _lib

cfg, n, nq = (int(v) for v in sys.argv[1:4])
metric = int(sys.argv[4]) if len(sys.argv) > 4 else synth.CONFIGS[cfg]["metric"]
k = int(sys.argv[5]) if len(sys.argv) > 5 else 100
X, Q = synth.generate(cfg, n=n, nq=nq)
idx = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric(metric), synth.CONFIGS[cfg]["calibration"])
qc = idx.encode_queries(torch.from_numpy(Q).cuda())
idx.search_codes(qc, k, sync=True)
torch.cuda.synchronize()
print("---- timed search", flush=True)
_lib.set_profiling(True)
idx.search_codes(qc, k, sync=True)
print(_lib.last_scan_stats(), flush=True)
_lib.set_profiling(False)
os.environ["QA_B200_TRACE"] = "1"
print("---- traced search", flush=True)
idx.search_codes(qc, k, sync=True)
