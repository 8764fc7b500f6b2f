"""Seeded synthetic stand-ins for the BASELINE.json workloads.

The paper measures on SIFT, GloVe-100 and the proprietary PRODUCT60M; none
are available offline, so each BASELINE config is generated with its
shape, metric and value distribution.  Every generator is a
pure function of its arguments (numpy default_rng, fixed call order:
database first, then queries).
"""

from __future__ import annotations

import numpy as np


def sift_like(n: int, nq: int, d: int = 128, seed: int = 0, chunk: int = 1 << 18):
    """Configs 0/2/4: round(|N(0, 40^2)|) clipped to [0, 255], 10% of the
    entries forced to 0; queries from the same law."""
    rng = np.random.default_rng(seed)

    def draw(m):
        out = np.empty((m, d), dtype=np.float32)
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            v = np.clip(np.round(np.abs(rng.normal(0.0, 40.0, size=(hi - lo, d)))), 0, 255)
            v[rng.random((hi - lo, d)) < 0.1] = 0.0
            out[lo:hi] = v
        return out

    return draw(n), draw(nq)


def glove_like(n: int, nq: int, d: int = 100, seed: int = 1, chunk: int = 1 << 18):
    """Config 1: per-dimension mean_j ~ N(0, 0.1^2), std_j ~ U(0.2, 1.0),
    x_ij ~ N(mean_j, std_j^2), every row L2-normalised (float64 norm, stored
    float32); queries drawn the same way."""
    rng = np.random.default_rng(seed)
    mean = rng.normal(0.0, 0.1, size=d)
    std = rng.uniform(0.2, 1.0, size=d)

    def draw(m):
        out = np.empty((m, d), dtype=np.float32)
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            v = rng.normal(size=(hi - lo, d)) * std + mean
            v /= np.linalg.norm(v, axis=1, keepdims=True)
            out[lo:hi] = v
        return out

    return draw(n), draw(nq)


def mixture_like(n: int, nq: int, d: int = 256, clusters: int = 1024, seed: int = 3,
                 chunk: int = 1 << 18):
    """Config 3: Gaussian mixture, centres ~ N(0, I), weights ~ Dirichlet(1),
    within-cluster std 0.3.  Returns (db, queries); use ``mixture_chunks``
    for databases too large to materialise."""
    rng = np.random.default_rng(seed)
    centres = rng.normal(size=(clusters, d))
    weights = rng.dirichlet(np.ones(clusters))

    def draw(m):
        out = np.empty((m, d), dtype=np.float32)
        for lo in range(0, m, chunk):
            hi = min(m, lo + chunk)
            z = rng.choice(clusters, size=hi - lo, p=weights)
            out[lo:hi] = centres[z] + 0.3 * rng.normal(size=(hi - lo, d))
        return out

    return draw(n), draw(nq)


CONFIGS = {
    0: dict(name="cfg0-l2-100k", gen="sift", n=100_000, nq=1_000, d=128, metric=1,
            calibration="minmax", k=100, seed=0),
    1: dict(name="cfg1-angular-1m", gen="glove", n=1_000_000, nq=10_000, d=100, metric=2,
            calibration="symmetric", k=100, seed=1),
    2: dict(name="cfg2-l2-1m", gen="sift", n=1_000_000, nq=10_000, d=128, metric=1,
            calibration="minmax", k=100, seed=2),
    3: dict(name="cfg3-ip-60m", gen="mixture", n=60_000_000, nq=10_000, d=256, metric=0,
            calibration="minmax", k=100, seed=3),
    4: dict(name="cfg4-small-batch-10m", gen="sift", n=10_000_000, nq=64, d=128, metric=1,
            calibration="minmax", k=100, seed=4),
}


def generate(cfg: int, n: int | None = None, nq: int | None = None):
    c = CONFIGS[cfg]
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    if c["gen"] == "sift":
        return sift_like(n, nq, c["d"], c["seed"])
    if c["gen"] == "glove":
        return glove_like(n, nq, c["d"], c["seed"])
    return mixture_like(n, nq, c["d"], seed=c["seed"])
