"""Seeded synthetic stand-ins for the BASELINE.json workloads (measurement
and test infrastructure; not part of the product package).

The paper measures on SIFT, GloVe-100 and the proprietary PRODUCT60M; none
are available offline, so each BASELINE config is generated with its
shape, metric and value distribution.

Rows are generated in fixed chunks of ``CHUNK`` rows, each chunk from its
own ``SeedSequence((seed, stream, chunk))`` (stream 0 = database, 1 =
queries, 2 = shared law parameters).  Any row range ``[lo, hi)`` is
therefore reproducible on its own -- one rank of a row-sharded run
generates only its shard -- and chunks can be drawn in parallel.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

CHUNK = 1 << 16
_DB, _Q, _LAW = 0, 1, 2


def _rng(seed: int, stream: int, chunk: int = 0) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence((seed, stream, chunk)))


def _sift_chunk(rng, m, d):
    """round(|N(0, 40^2)|) clipped to [0, 255], 10 % of the entries forced to 0."""
    v = np.clip(np.round(np.abs(rng.normal(0.0, 40.0, size=(m, d)))), 0, 255)
    v[rng.random((m, d)) < 0.1] = 0.0
    return v


def _glove_law(seed, d):
    rng = _rng(seed, _LAW)
    return rng.normal(0.0, 0.1, size=d), rng.uniform(0.2, 1.0, size=d)


def _glove_chunk(rng, m, d, law):
    """x_ij ~ N(mean_j, std_j^2), every row L2-normalised (float64 norm)."""
    mean, std = law
    v = rng.normal(size=(m, d)) * std + mean
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v


def _mixture_law(seed, d, clusters=1024):
    rng = _rng(seed, _LAW)
    return rng.normal(size=(clusters, d)), rng.dirichlet(np.ones(clusters))


def _mixture_chunk(rng, m, d, law):
    """Gaussian mixture: centre ~ N(0, I), weights ~ Dirichlet(1), within-cluster std 0.3."""
    centres, weights = law
    z = rng.choice(centres.shape[0], size=m, p=weights)
    return centres[z] + 0.3 * rng.normal(size=(m, d))


CONFIGS = {
    0: dict(name="cfg0-l2-100k", gen="sift", n=100_000, nq=1_000, d=128, metric=1,
            calibration="minmax", k=100, seed=0, batch=1_000),
    1: dict(name="cfg1-angular-1m", gen="glove", n=1_000_000, nq=10_000, d=100, metric=2,
            calibration="symmetric", k=100, seed=1, batch=10_000),  # unbatched in BASELINE
    2: dict(name="cfg2-l2-1m", gen="sift", n=1_000_000, nq=10_000, d=128, metric=1,
            calibration="minmax", k=100, seed=2, batch=1_024),
    3: dict(name="cfg3-ip-60m", gen="mixture", n=60_000_000, nq=10_000, d=256, metric=0,
            calibration="minmax", k=100, seed=3, batch=1_024),
    4: dict(name="cfg4-small-batch-10m", gen="sift", n=10_000_000, nq=64, d=128, metric=1,
            calibration="minmax", k=100, seed=4, batch=64),
}


def _law(c):
    if c["gen"] == "glove":
        return _glove_law(c["seed"], c["d"])
    if c["gen"] == "mixture":
        return _mixture_law(c["seed"], c["d"])
    return None


def _fill(c, law, stream, lo, hi, out, threads):
    d, seed = c["d"], c["seed"]

    def one(ci):
        a, b = max(lo, ci * CHUNK), min(hi, (ci + 1) * CHUNK)
        rng = _rng(seed, stream, ci)
        m = CHUNK  # whole chunks: a row's value never depends on the range asked for
        if c["gen"] == "sift":
            v = _sift_chunk(rng, m, d)
        elif c["gen"] == "glove":
            v = _glove_chunk(rng, m, d, law)
        else:
            v = _mixture_chunk(rng, m, d, law)
        out[a - lo:b - lo] = v[a - ci * CHUNK:b - ci * CHUNK]

    chunks = range(lo // CHUNK, (hi + CHUNK - 1) // CHUNK)
    if threads > 1 and len(chunks) > 1:
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, chunks))
    else:
        for ci in chunks:
            one(ci)


def rows(cfg: int, lo: int, hi: int, threads: int | None = None) -> np.ndarray:
    """Database rows [lo, hi) of config ``cfg`` as float32 [hi - lo, d]."""
    c = CONFIGS[cfg]
    out = np.empty((hi - lo, c["d"]), dtype=np.float32)
    _fill(c, _law(c), _DB, lo, hi, out, threads or min(16, os.cpu_count() or 1))
    return out


def queries(cfg: int, nq: int | None = None, threads: int | None = None) -> np.ndarray:
    """The first ``nq`` queries of config ``cfg`` as float32 [nq, d]."""
    c = CONFIGS[cfg]
    nq = c["nq"] if nq is None else nq
    out = np.empty((nq, c["d"]), dtype=np.float32)
    _fill(c, _law(c), _Q, 0, nq, out, threads or min(16, os.cpu_count() or 1))
    return out


def generate(cfg: int, n: int | None = None, nq: int | None = None):
    """(database [n, d], queries [nq, d]) float32 of config ``cfg``."""
    c = CONFIGS[cfg]
    n = c["n"] if n is None else n
    return rows(cfg, 0, n), queries(cfg, nq)


def sift_like(n: int, nq: int, d: int = 128, seed: int = 0):
    """Configs 0/2/4 law at any shape (tests)."""
    c = dict(CONFIGS[0], d=d, seed=seed)
    X = np.empty((n, d), dtype=np.float32)
    Q = np.empty((nq, d), dtype=np.float32)
    _fill(c, None, _DB, 0, n, X, 1)
    _fill(c, None, _Q, 0, nq, Q, 1)
    return X, Q
