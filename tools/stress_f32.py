"""Randomised parity stress of the float32 exact scan (vs the C oracle's
_scan_f32 restatement) and of estimate_stats (vs the numpy evaluation the
reference's quantizer.py:176-222 performs, restated here as the checker).
python tools/stress_f32.py SECONDS SEED"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import qa_oracle as o
import paper_2110_08919_b200 as qa
from paper_2110_08919_b200 import device as dev


def np_stats(x):
    n, d = x.shape
    out = {k: np.empty(d) for k in ("mu", "sigma", "min", "max", "tam")}
    for lo in range(0, d, 64):
        hi = min(lo + 64, d)
        b = x[:, lo:hi].astype(np.float64)
        m = b.mean(axis=0)
        c = b - m
        out["mu"][lo:hi] = m
        out["sigma"][lo:hi] = np.sqrt(np.mean(c * c, axis=0))
        out["min"][lo:hi] = b.min(axis=0)
        out["max"][lo:hi] = b.max(axis=0)
        ql = np.quantile(b, 0.001, axis=0, method="lower")
        qh = np.quantile(b, 0.999, axis=0, method="higher")
        kept = (b >= ql) & (b <= qh)
        out["tam"][lo:hi] = np.where(kept, np.abs(c), -np.inf).max(axis=0)
    fs = 0.0
    for lo in range(0, d, 64):
        fs += float(np.sum(x[:, lo:lo + 64].astype(np.float64)))
    fm = fs / (n * d)
    pv = 0.0
    for lo in range(0, d, 64):
        b = x[:, lo:lo + 64].astype(np.float64) - fm
        pv += float(np.sum(b * b))
    return out, fm, math.sqrt(pv / (n * d))


budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
t0, cases, fails = time.time(), 0, 0
while time.time() - t0 < budget:
    n = int(rng.choice([2, 3, 9, 130, 1000, 20_000, 70_000]))
    d = int(rng.choice([1, 2, 17, 64, 65, 100, 129, 200]))
    scale = 10 ** rng.uniform(-3, 3)
    X = (rng.normal(size=(n, d)) * scale).astype(np.float32)
    if rng.random() < 0.3:
        X = np.round(X).astype(np.float32)  # ties
    # estimate_stats
    st = qa.estimate_stats(torch.from_numpy(X).cuda())
    ref, fm, ps = np_stats(X)
    ok = (np.array_equal(st.mu, ref["mu"]) and np.array_equal(st.sigma, ref["sigma"])
          and np.array_equal(st.min, ref["min"]) and np.array_equal(st.max, ref["max"])
          and np.array_equal(st.trimmed_absmax, ref["tam"]) and st.pooled_mu == fm
          and st.pooled_sigma == ps)
    cases += 1
    if not ok:
        fails += 1
        print("STATS MISMATCH", n, d, scale, flush=True)
    # float32 scan
    if n * d <= 2_000_000:
        nq = int(rng.choice([1, 5, 70, 1100]))
        k = int(rng.choice([1, 10, 100, 2048, 3000]))
        metric = int(rng.integers(0, 3))
        Q = (rng.normal(size=(nq, d)) * scale).astype(np.float32)
        X2 = X.copy()
        X2[~X2.any(axis=1), 0] = 1
        Q[~Q.any(axis=1), 0] = 1
        xn, qn = o.norms_f32(X2), o.norms_f32(Q)
        sc, ids = dev.scan_topk_f32(torch.from_numpy(X2).cuda(), torch.from_numpy(Q).cuda(), k,
                                    metric, torch.from_numpy(xn).cuda(), torch.from_numpy(qn).cuda())
        osc, oids = o.scan_topk_f32(X2, Q, k, metric, xn, qn)
        cases += 1
        if not (np.array_equal(ids.cpu().numpy(), oids) and np.array_equal(sc.cpu().numpy(), osc)):
            fails += 1
            print("F32 MISMATCH", n, d, nq, k, metric, flush=True)
print(f"stress_f32: {cases} cases, {fails} failures, {time.time() - t0:.0f}s", flush=True)
