"""One small-batch configuration (cfg4 law) searched a few times: the
target of the small-batch ncu captures.  python tools/small_one.py METRIC K BATCH"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2110_08919_b200 as qa
import synth

metric, k, B = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 10_000_000
X, Q = synth.sift_like(n, 64, 128, 4)
x = torch.from_numpy(X).cuda()
del X
index = qa.Int8Index.build(x, qa.Metric(metric), "minmax")
del x
qc = index.encode_queries(torch.from_numpy(Q[:B]).cuda())
for _ in range(4):
    index.search_codes(qc, k)
torch.cuda.synchronize()
print("ok")
