"""Randomised parity stress: the GPU scan (plain and norm-banded index
layouts, every metric) against the C oracle on random shapes, value ranges
(tie-heavy included), k and batch sizes.  python tools/stress.py SECONDS SEED"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import qa_oracle as o
from paper_2110_08919_b200 import device as dev

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0, cases, fails = time.time(), 0, 0
while time.time() - t0 < budget:
    n = int(rng.choice([1, 7, 129, 1000, 5000, 40_000, 140_000, 300_000]))
    d = int(rng.choice([1, 3, 8, 31, 64, 100, 128, 200, 256]))
    nq = int(rng.choice([1, 3, 64, 65, 129, 256, 257, 1000, 3000]))
    if n * d > 40_000_000 or n * nq * d > 4e10:
        continue
    k = int(rng.choice([1, 5, 10, 32, 33, 64, 100, 128, 129, 500, 2048]))
    lim = int(rng.choice([2, 4, 30, 128]))
    metric = int(rng.integers(0, 3))
    skew = rng.random() < 0.3   # SIFT-like: values near -128 (large dots)
    def draw(m):
        if skew:
            x = np.clip(-128 + np.abs(rng.normal(0, 40, size=(m, d))), -128, 127)
        else:
            x = rng.integers(-lim, lim, size=(m, d))
        x = x.astype(np.int8)
        x[~x.any(axis=1), 0] = 1
        return x
    X, Q = draw(n), draw(nq)
    layout = int(rng.integers(0, 3))  # 0 plain, 1 banded, 2 banded + stratified
    db = dev.DeviceCodes.from_host(X)
    if layout:
        db = db.sorted_by_norm(stratify=layout == 2)
    qs = dev.DeviceCodes.from_host(Q)
    try:
        sc, ids = dev.scan_topk(db, qs, k, metric, id_offset=0)
        sc, ids = sc.cpu().numpy(), ids.cpu().numpy()
    except Exception as e:  # noqa: BLE001
        print("ERROR", n, d, nq, k, lim, metric, skew, layout, repr(e)[:200], flush=True)
        fails += 1
        cases += 1
        continue
    osc, oids = o.scan_topk_i8(X, Q, k, metric, o.norms_i8(X), o.norms_i8(Q))
    ok = np.array_equal(ids, oids) and np.array_equal(sc, osc)
    cases += 1
    if not ok:
        fails += 1
        print("MISMATCH", n, d, nq, k, lim, metric, skew, layout, flush=True)
print(f"stress: {cases} cases, {fails} failures, {time.time() - t0:.0f}s", flush=True)
