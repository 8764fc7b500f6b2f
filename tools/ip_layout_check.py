"""IP small batches: scan statistics with and without the norm-sorted layout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_08919_b200 as qa
import synth
from paper_2110_08919_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
X, Q = synth.sift_like(n, 64, 128, 4)
x = torch.from_numpy(X).cuda()
fr = qa.fit_minmax(qa.minmax_stats(x))
for sort in (False, True):
    idx = qa.Int8Index.from_params(x, fr.params, qa.Metric.INNER_PRODUCT, sort_rows=sort)  # sort: the shuffled layout
    for B in (1, 8, 64):
        qc = idx.encode_queries(torch.from_numpy(Q[:B]).cuda())
        _lib.set_profiling(True)
        idx.search_codes(qc, 10, sync=True)
        st = _lib.last_scan_stats()
        _lib.set_profiling(False)
        print("sorted" if sort else "caller", B, {k: st[k] for k in ("rounds", "retries", "candidates", "filter_ms", "select_ms")}, flush=True)
    del idx
    torch.cuda.empty_cache()
