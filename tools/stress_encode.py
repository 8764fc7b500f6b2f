"""Randomised encode parity (GPU encode kernels vs the C oracle's Eq. 1):
random shapes (d <= 256 takes the multi-row kernel), scales, windows, bits,
NaN/inf/denormal sprinkles.  python tools/stress_encode.py SECONDS SEED"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import qa_oracle as o
from paper_2110_08919_b200 import device as dev

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0, cases, fails = time.time(), 0, 0
while time.time() - t0 < budget:
    n = int(rng.choice([1, 2, 3, 5, 33, 1000, 20_000]))
    d = int(rng.choice([1, 4, 8, 100, 124, 128, 132, 200, 256, 260, 300]))
    bits = int(rng.integers(1, 9))
    sc = 10 ** rng.uniform(-4, 4)
    X = (rng.normal(size=(n, d)) * sc).astype(np.float32)
    m = rng.random((n, d))
    X[m < 0.01] = np.nan
    X[(m > 0.01) & (m < 0.015)] = np.inf
    X[(m > 0.015) & (m < 0.02)] = np.float32(1e-41)
    c = rng.normal(size=d).astype(np.float32) * np.float32(sc)
    h = (np.abs(rng.normal(size=d)) * sc + 1e-6).astype(np.float32)
    k = c
    sb = (c - h).astype(np.float32)
    se = (c + h).astype(np.float32)
    bad = ~(sb < se)
    se[bad] = np.nextafter(sb[bad], np.float32(np.inf))
    got = dev.encode(torch.from_numpy(X).cuda(), torch.from_numpy(k).cuda(),
                     torch.from_numpy(sb).cuda(), torch.from_numpy(se).cuda(), bits).to_host()
    want = o.encode(X, k, sb, se, bits)
    cases += 1
    if not np.array_equal(got, want):
        fails += 1
        print("MISMATCH", n, d, bits, sc, flush=True)
print(f"stress_encode: {cases} cases, {fails} failures, {time.time() - t0:.0f}s", flush=True)
