"""Row-sharded search plumbing on CPU: world_size 2 over gloo.

Each rank computes its shard's top-k (CPU oracle -- the checker stands in
for the GPU scan here), ``sharded.sharded_search`` pads, all-gathers and
merges; the merged result must equal the single-process full scan bit for
bit, including heavy ties across the shard boundary.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _merge_host(s_all: torch.Tensor, i_all: torch.Tensor, k: int):
    """(score, id) merge of [G, nq, kin] lists (test-side checker)."""
    G, nq, kin = s_all.shape
    s = s_all.permute(1, 0, 2).reshape(nq, G * kin).numpy()
    i = i_all.permute(1, 0, 2).reshape(nq, G * kin).numpy()
    out_s = np.empty((nq, k))
    out_i = np.empty((nq, k), np.int32)
    for q in range(nq):
        order = np.lexsort((i[q], s[q] + 0.0))[:k]
        out_s[q], out_i[q] = s[q][order], i[q][order]
    return torch.from_numpy(out_s), torch.from_numpy(out_i)


def _np_topk(X, Q, k, metric):
    """numpy (score, id) top-k (the forked workers avoid the OpenMP oracle:
    libgomp is not fork-safe once the parent used it)."""
    Xw, Qw = X.astype(np.int64), Q.astype(np.int64)
    dots = Qw @ Xw.T
    if metric == 0:
        sc = -dots.astype(np.float64)
    elif metric == 1:
        sc = ((Qw * Qw).sum(1)[:, None] + (Xw * Xw).sum(1)[None, :] - 2 * dots).astype(np.float64)
    else:
        xn = np.sqrt((Xw * Xw).sum(1).astype(np.float64)).astype(np.float32).astype(np.float64)
        qn = np.sqrt((Qw * Qw).sum(1).astype(np.float64)).astype(np.float32).astype(np.float64)
        sc = 1.0 - dots.astype(np.float64) / (qn[:, None] * xn[None, :])
    keff = min(k, X.shape[0])
    ids = np.arange(X.shape[0])
    out_s = np.empty((Q.shape[0], keff))
    out_i = np.empty((Q.shape[0], keff), np.int32)
    for q in range(Q.shape[0]):
        order = np.lexsort((ids, sc[q]))[:keff]
        out_s[q], out_i[q] = sc[q][order], order
    return out_s, out_i


def _worker(rank, world, port, X, Q, k, metric, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_08919_b200 import sharded

    lo, hi = sharded.shard_bounds(X.shape[0], world, rank)

    def local(id_offset):
        s, i = _np_topk(X[lo:hi], Q, k, metric)
        return torch.from_numpy(s), torch.from_numpy(i + id_offset)

    s, i = sharded.sharded_search(local, X.shape[0], k, merge=_merge_host)
    out[rank] = (s.numpy(), i.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _worker_batches(rank, world, port, X, Qs, k, metric, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2110_08919_b200 import sharded

    lo, hi = sharded.shard_bounds(X.shape[0], world, rank)

    def local_for(Q):
        def local(id_offset):
            s, i = _np_topk(X[lo:hi], Q, k, metric)
            return torch.from_numpy(s), torch.from_numpy(i + id_offset)
        return local

    res = sharded.sharded_search_batches([local_for(Q) for Q in Qs], X.shape[0], k,
                                         merge=_merge_host)
    out[rank] = [(s.numpy(), i.numpy()) for s, i in res]
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_pipelined_batches_equal_full_scan(oracle, world):
    """sharded_search_batches (the gather of batch i overlapped with the scan
    of batch i + 1): every batch equals the single-process full scan."""
    rng = np.random.default_rng(91 + world)
    n, k, metric = 700, 40, 1
    X = rng.integers(-4, 5, size=(n, 12)).astype(np.int8)
    X[~X.any(axis=1), 0] = 1
    Qs = []
    for nq in (5, 1, 8, 3):  # ragged batches
        Q = rng.integers(-4, 5, size=(nq, 12)).astype(np.int8)
        Q[~Q.any(axis=1), 0] = 1
        Qs.append(Q)
    manager = mp.Manager()
    out = manager.dict()
    mp.start_processes(_worker_batches, args=(world, _free_port(), X, Qs, k, metric, out),
                       nprocs=world, join=True, start_method="fork")
    for b, Q in enumerate(Qs):
        want_s, want_i = oracle.scan_topk_i8(X, Q, k, metric, oracle.norms_i8(X), oracle.norms_i8(Q))
        for rank in range(world):
            s, i = out[rank][b]
            np.testing.assert_array_equal(i, want_i)
            np.testing.assert_array_equal(s, want_s)


@pytest.mark.parametrize("metric", [0, 1, 2])
@pytest.mark.parametrize("world,n,k", [(2, 1001, 50), (3, 1001, 50), (3, 100, 50)])
def test_gloo_merge_equals_full_scan(oracle, metric, world, n, k):
    # world 3: uneven shards (334/334/333); n=100, k=50: every shard holds
    # fewer than k rows, so its list is padded before the exchange
    rng = np.random.default_rng(40 + metric + world)
    X = rng.integers(-4, 5, size=(n, 12)).astype(np.int8)   # many ties
    X[~X.any(axis=1), 0] = 1
    Q = rng.integers(-4, 5, size=(7, 12)).astype(np.int8)
    Q[~Q.any(axis=1), 0] = 1
    manager = mp.Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(world, _free_port(), X, Q, k, metric, out), nprocs=world,
                       join=True, start_method="fork")
    want_s, want_i = oracle.scan_topk_i8(X, Q, k, metric, oracle.norms_i8(X), oracle.norms_i8(Q))
    for rank in range(world):
        s, i = out[rank]
        np.testing.assert_array_equal(i, want_i)
        np.testing.assert_array_equal(s, want_s)


def test_shard_bounds_partition():
    from paper_2110_08919_b200.sharded import shard_bounds

    for n in (0, 1, 7, 100, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
