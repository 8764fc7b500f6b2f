"""Listed-pair distances on the GPU (qa_gather_scores_i8, the batched form of
the reference's HnswCore._dq / _dist_rows, _core.pyx:472-494) against the
oracle: bit-exact float64 scores for every metric."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _case(rng, n, d, nq, m, lo=-128, hi=128):
    X = rng.integers(lo, hi, size=(n, d)).astype(np.int8)
    Q = rng.integers(lo, hi, size=(nq, d)).astype(np.int8)
    X[~X.any(axis=1), 0] = 1
    Q[~Q.any(axis=1), 0] = 1
    cand = rng.integers(-3, n + 3, size=(nq, m)).astype(np.int32)
    return X, Q, cand


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_pair_scores_match_oracle(oracle, metric):
    import torch
    from paper_2110_08919_b200 import device as dev

    rng = np.random.default_rng(100 + metric)
    for n, d, nq, m in [(1, 1, 1, 1), (7, 3, 2, 5), (500, 100, 33, 17), (4096, 128, 64, 64),
                        (3000, 256, 9, 130), (2000, 300, 5, 4), (900, 1000, 3, 33)]:
        X, Q, cand = _case(rng, n, d, nq, m)
        xn, qn = oracle.norms_i8(X), oracle.norms_i8(Q)
        want = oracle.pair_scores_i8(X, Q, cand, metric, xn, qn)
        db = dev.DeviceCodes.from_host(X)
        qs = dev.DeviceCodes.from_host(Q)
        got = dev.gather_scores(db, qs, torch.from_numpy(cand).cuda(), metric).cpu().numpy()
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_pair_scores_on_index_layouts(oracle, metric):
    """The database kept in the search's index layouts (norm bands, shuffled):
    caller ids are mapped to stored rows."""
    import torch
    from paper_2110_08919_b200 import device as dev

    rng = np.random.default_rng(7)
    X, Q, cand = _case(rng, 20_000, 128, 16, 48, lo=-20, hi=90)
    xn, qn = oracle.norms_i8(X), oracle.norms_i8(Q)
    want = oracle.pair_scores_i8(X, Q, cand, metric, xn, qn)
    base = dev.DeviceCodes.from_host(X)
    qs = dev.DeviceCodes.from_host(Q)
    for db in (base.sorted_by_norm(), base.shuffled()):
        got = dev.gather_scores(db, qs, torch.from_numpy(cand).cuda(), metric,
                                row_of_id=dev.inverse_ids(db)).cpu().numpy()
        np.testing.assert_array_equal(got, want)


def test_pair_scores_host_seam(oracle):
    """The host seam (_backend.pair_scores): frozen corpus resident, numpy in/out,
    ragged lists padded with -1, and the reference's argument errors."""
    from paper_2110_08919_b200 import _backend

    rng = np.random.default_rng(3)
    X, Q, cand = _case(rng, 1500, 96, 12, 40)
    cand[:, 30:] = -1
    X.flags.writeable = False
    xn, qn = oracle.norms_i8(X), oracle.norms_i8(Q)
    for metric in (0, 1, 2):
        got = _backend.pair_scores(X, Q, cand, metric, xn, qn)
        np.testing.assert_array_equal(got, oracle.pair_scores_i8(X, Q, cand, metric, xn, qn))
        assert np.isinf(got[:, 30:]).all()
    with pytest.raises(ValueError):
        _backend.pair_scores(X, Q[:, :10], cand, 0)
    with pytest.raises(ValueError):
        _backend.pair_scores(X, Q, cand, 2)
    with pytest.raises(ValueError):
        _backend.pair_scores(X, Q, cand[:3], 0)


def test_greedy_descent_matches_reference_formulation(oracle):
    """A host greedy descent (the reference's _greedy, _core.pyx:505-527:
    move to the (score, id)-smallest strictly better neighbour until none
    improves) over a random graph, for a batch of queries in lockstep with one
    pair-score call per hop, reaches the nodes the per-pair CPU loop reaches."""
    from paper_2110_08919_b200 import _backend

    rng = np.random.default_rng(11)
    n, d, nq, deg = 3000, 64, 32, 12
    X, Q, _ = _case(rng, n, d, nq, 1)
    X.flags.writeable = False
    nbrs = rng.integers(0, n, size=(n, deg)).astype(np.int32)

    def cpu_greedy(q):
        cur = 0
        cur_d = oracle.pair_scores_i8(X, Q[q:q + 1], np.array([[cur]], np.int32), 1)[0, 0]
        changed = True
        while changed:
            changed = False
            for u in nbrs[cur].tolist():  # the list the pass started on (_core.pyx:507)
                du = oracle.pair_scores_i8(X, Q[q:q + 1], np.array([[u]], np.int32), 1)[0, 0]
                if (du, u) < (cur_d, cur):
                    cur, cur_d, changed = u, du, True
        return cur

    cur = np.zeros(nq, dtype=np.int32)
    cur_d = _backend.pair_scores(X, Q, cur[:, None], 1)[:, 0]
    active = np.ones(nq, dtype=bool)
    while active.any():
        lists = nbrs[cur]                      # [nq, deg], one hop for every query
        du = _backend.pair_scores(X, Q, lists, 1)
        for q in np.flatnonzero(active):
            c, cd, moved = int(cur[q]), float(cur_d[q]), False
            for j in range(deg):               # the reference's sequential acceptance rule
                u = int(lists[q, j])
                if (float(du[q, j]), u) < (cd, c):
                    c, cd, moved = u, float(du[q, j]), True
            cur[q], cur_d[q], active[q] = c, cd, moved
    assert cur.tolist() == [cpu_greedy(q) for q in range(nq)]
