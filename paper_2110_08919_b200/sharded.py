"""Row-sharded multi-GPU search.

One process per GPU.  The database is split into contiguous row ranges
``shard_bounds(n, world, rank)``; queries are replicated.  Each rank runs the
tensor-core scan on its shard with ``id_offset = shard start`` (global ids),
the per-rank sorted top-k lists are exchanged with one ``all_gather`` over
NCCL (NVLink/NVSwitch on a B200 box), and the (score, id) merge runs on the
GPU (libqa_b200 ``qa_merge_topk``).  Because (score, id) is a total order
and every rank reports exactly min(k, shard rows) entries in that order,
the merge equals the single-GPU result bit for bit.

The exchange is the only collective on the data path: k candidates per
query per rank (nq * k * 12 bytes, scores and ids packed into ONE byte
buffer so a batch costs one all-gather), independent of n.
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [lo, hi) row range of ``rank``; sizes differ by at most 1."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_topk(scores: torch.Tensor, ids: torch.Tensor, group=None):
    """All-gather per-rank [nq, kin] lists into [world, nq, kin] tensors with
    one collective: float64 scores and int32 ids travel as one packed
    [nq, kin * 12] byte row per query.

    Every rank must pass the same kin (ranks whose shard has fewer rows pad
    with +inf scores / INT32_MAX ids, which sort last)."""
    world = dist.get_world_size(group)
    kin = scores.shape[1]
    packed = _pack(scores, ids)
    parts = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(parts, packed, group=group)
    return _unpack(parts, kin)


def _pack(scores: torch.Tensor, ids: torch.Tensor) -> torch.Tensor:
    nq, kin = scores.shape
    return torch.cat([scores.contiguous().view(torch.uint8).reshape(nq, kin * 8),
                      ids.contiguous().view(torch.uint8).reshape(nq, kin * 4)], dim=1)


def _unpack(parts, kin: int):
    allp = torch.stack(parts)  # [world, nq, kin * 12]
    world, nq = allp.shape[0], allp.shape[1]
    s_all = allp[:, :, : kin * 8].contiguous().view(torch.float64).reshape(world, nq, kin)
    i_all = allp[:, :, kin * 8:].contiguous().view(torch.int32).reshape(world, nq, kin)
    return s_all, i_all


def pad_topk(scores: torch.Tensor, ids: torch.Tensor, kin: int):
    """Pad [nq, keff] lists to [nq, kin] with entries that sort last."""
    nq, keff = scores.shape
    if keff == kin:
        return scores, ids
    ps = torch.full((nq, kin), float("inf"), dtype=scores.dtype, device=scores.device)
    pi = torch.full((nq, kin), 2**31 - 1, dtype=ids.dtype, device=ids.device)
    ps[:, :keff] = scores
    pi[:, :keff] = ids
    return ps, pi


def sharded_search(local_search: Callable[[int], tuple], n_total: int, k: int,
                   merge: Callable | None = None, group=None):
    """Run ``local_search(id_offset) -> (scores, ids)`` on this rank's shard,
    exchange candidates and merge.  ``merge`` defaults to the GPU merge
    kernel; every rank returns the global (scores, ids)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, _ = shard_bounds(n_total, world, rank)
    scores, ids = local_search(lo)
    kin = min(k, -(-n_total // world))  # largest shard's keff
    scores, ids = pad_topk(scores, ids, kin)
    s_all, i_all = gather_topk(scores, ids, group)
    keff = min(k, n_total)
    if merge is None:
        from .device import merge_topk as merge
    return merge(s_all, i_all, keff)


def sharded_search_batches(local_searches, n_total: int, k: int, merge: Callable | None = None,
                           group=None):
    """``sharded_search`` for a sequence of query batches, pipelined: batch
    i's all-gather is issued asynchronously and waited for only after batch
    i + 1's local search has been launched, so the exchange (NCCL's own
    stream) overlaps the next batch's scan.  ``local_searches``: one
    ``id_offset -> (scores, ids)`` callable per batch.  Returns the list of
    merged (scores, ids), equal to calling ``sharded_search`` per batch."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, _ = shard_bounds(n_total, world, rank)
    kin = min(k, -(-n_total // world))
    keff = min(k, n_total)
    if merge is None:
        from .device import merge_topk as merge
    results = []
    pending = None  # (work, parts) of the previous batch

    def finish(p):
        work, parts = p
        work.wait()
        s_all, i_all = _unpack(parts, kin)
        results.append(merge(s_all, i_all, keff))

    for local_search in local_searches:
        scores, ids = pad_topk(*local_search(lo), kin)
        packed = _pack(scores, ids)
        parts = [torch.empty_like(packed) for _ in range(world)]
        work = dist.all_gather(parts, packed, group=group, async_op=True)
        if pending is not None:
            finish(pending)
        pending = (work, parts)
    if pending is not None:
        finish(pending)
    return results
