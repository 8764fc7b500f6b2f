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
    # adversarial columns for the fast division (zero / off-centre k, extreme
    # window widths) and elements on code boundaries, equal or next to k
    mode = int(rng.integers(0, 6))
    cols = rng.random(d)
    if mode >= 1:
        k = np.where(cols < 0.3, np.float32(0), k).astype(np.float32)
        k = np.where((cols > 0.3) & (cols < 0.4), (c + 3 * h).astype(np.float32), k).astype(np.float32)
    if mode == 2:
        wexp = rng.choice([-44.0, -38.0, -30.0, -20.0, 20.0, 30.0, 37.0], size=d)
        h = np.where(cols > 0.6, (10.0 ** wexp), h).astype(np.float32)
        sb = (c - h).astype(np.float32)
        se = (c + h).astype(np.float32)
    bad = ~(sb < se)
    se[bad] = np.nextafter(sb[bad], np.float32(np.inf))
    if mode >= 3:
        w = (se - sb).astype(np.float32)
        j = rng.integers(-140, 141, size=(n, d)).astype(np.float32)
        edge = (k[None, :] + w[None, :] * (j / np.float32(2 ** bits))).astype(np.float32)
        pick = rng.random((n, d))
        X = np.where(pick < 0.3, edge, X).astype(np.float32)
        X = np.where((pick > 0.3) & (pick < 0.35), np.nextafter(edge, np.float32(np.inf)), X).astype(np.float32)
        X = np.where((pick > 0.35) & (pick < 0.4), np.nextafter(edge, np.float32(-np.inf)), X).astype(np.float32)
        X = np.where((pick > 0.4) & (pick < 0.45), k[None, :], X).astype(np.float32)
        tinyv = np.float32(10.0) ** rng.integers(-45, -20, size=(n, d)).astype(np.float32)
        X = np.where((pick > 0.45) & (pick < 0.5), (k[None, :] + tinyv).astype(np.float32), X).astype(np.float32)
        X = np.where((pick > 0.5) & (pick < 0.53), -tinyv.astype(np.float32), X).astype(np.float32)
    if mode == 5:  # integer-valued data under a min/max window
        X = np.clip(np.round(np.abs(rng.normal(size=(n, d)) * 40)), 0, 255).astype(np.float32)
        sb = X.min(axis=0).astype(np.float32)
        se = X.max(axis=0).astype(np.float32)
        flat = ~(sb < se)
        se[flat] = sb[flat] + np.float32(1)
        k = ((sb.astype(np.float64) + se.astype(np.float64)) / 2).astype(np.float32)
    got = dev.encode(torch.from_numpy(X).cuda(), torch.from_numpy(k).cuda(),
                     torch.from_numpy(sb).cuda(), torch.from_numpy(se).cuda(), bits).to_host()
    want = o.encode(X, k, sb, se, bits)
    cases += 1
    if not np.array_equal(got, want):
        fails += 1
        print("MISMATCH", n, d, bits, sc, flush=True)
print(f"stress_encode: {cases} cases, {fails} failures, {time.time() - t0:.0f}s", flush=True)
