"""Recall and throughput bookkeeping (reference bench.py:52-145)."""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .dataset import DenseDataset, GroundTruth
from .errors import LengthMismatch


@dataclass(frozen=True)
class RecallReport:
    k: int
    per_query: np.ndarray
    expected_total: int
    hit_total: int

    def __post_init__(self):
        self.per_query.flags.writeable = False

    @property
    def mean(self) -> float:
        return float(self.per_query.mean())


@dataclass(frozen=True)
class ThroughputReport:
    n_queries: int
    elapsed_s: float
    threads: int = 1

    @property
    def qps(self) -> float:
        return self.n_queries / self.elapsed_s


def recall_at_k(expected, actual, k: int) -> RecallReport:
    """Mean fraction of the first k exact ids found in the first k returned
    ids (order-free set intersection, bench.py:99-124)."""
    exp = expected.ids if isinstance(expected, GroundTruth) else np.asarray(expected)
    act = actual.ids if isinstance(actual, GroundTruth) else np.asarray(actual)
    if k < 1:
        raise ValueError("k must be >= 1")
    if exp.shape[0] != act.shape[0]:
        raise LengthMismatch(f"{exp.shape[0]} expected lists vs {act.shape[0]} actual lists")
    if exp.shape[1] < k:
        raise ValueError(f"expected lists have {exp.shape[1]} entries, need >= {k}")
    per = np.empty(exp.shape[0], dtype=np.float64)
    for i in range(exp.shape[0]):
        per[i] = np.isin(act[i, :k], exp[i, :k]).sum() / k
    return RecallReport(k=k, per_query=per, expected_total=exp.shape[0] * k,
                        hit_total=int(round(per.sum() * k)))


def measure_qps(search_fn, queries: DenseDataset, warmup: int = 10):
    """One timed pass of search_fn over every query row after ``warmup``
    untimed calls (bench.py:127-145)."""
    if queries.n < 1:
        raise ValueError("need at least one query")
    rows = queries.data
    for i in range(min(warmup, queries.n)):
        search_fn(rows[i])
    results = []
    t0 = time.perf_counter()
    for i in range(queries.n):
        results.append(search_fn(rows[i]))
    return ThroughputReport(n_queries=queries.n, elapsed_s=time.perf_counter() - t0), results
