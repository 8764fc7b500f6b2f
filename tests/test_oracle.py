"""The CPU oracle is pinned before it is trusted: against the golden vectors
produced by the REAL reference (tests/golden/make_golden.py) and, where the
reference's compiled kernel was built here (oracle/_ref), against it on fresh
random instances."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import synth


def test_encode_matches_reference_golden(oracle, golden_encode):
    for name, c in golden_encode.items():
        got = oracle.encode(c["x"], c["k"], c["sb"], c["se"], int(c["bits"]))
        np.testing.assert_array_equal(got, c["codes"], err_msg=name)
        got_np = oracle.encode_np(c["x"], c["k"], c["sb"], c["se"], int(c["bits"]))
        np.testing.assert_array_equal(got_np, c["codes"], err_msg=name)


def test_encode_hand_values(oracle, golden_encode):
    # test_quantizer.py:133-141: 0->0, 0.05->64, -0.1->-128, 0.1->127,
    # 0.5->127, -0.2->-128, NaN->-128; +inf->127, -inf->-128
    c = golden_encode["hand"]
    got = oracle.encode(c["x"], c["k"], c["sb"], c["se"], 8)[:, 0]
    assert list(got) == [0, 64, -128, 127, 127, -128, -128, 127, -128]


def test_scan_matches_reference_golden(oracle, golden_scan):
    for name, c in golden_scan.items():
        sc, ids = oracle.scan_topk_i8(c["X"], c["Q"], int(c["k"]), int(c["metric"]), c["xn"],
                                      c["qn"])
        np.testing.assert_array_equal(ids, c["ids"], err_msg=name)
        np.testing.assert_array_equal(sc, c["scores"], err_msg=name)
        np.testing.assert_array_equal(oracle.norms_i8(c["X"]), c["xn"], err_msg=name)


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_cfg_pipeline_matches_reference_golden(oracle, golden_cfg, cfg):
    g = golden_cfg[f"cfg{cfg}"]
    X, Q = synth.generate(cfg, n=6000, nq=24)
    mn, mx = oracle.minmax(X)
    np.testing.assert_array_equal(mn, g["mn"])
    np.testing.assert_array_equal(mx, g["mx"])
    if cfg == 1:
        k, sb, se = oracle.fit_range(np.zeros_like(mn), np.maximum(np.abs(mn), np.abs(mx)))
    else:
        k, sb, se = oracle.fit_range((mn + mx) / 2.0, (mx - mn) / 2.0)
    np.testing.assert_array_equal(k, g["k"])
    np.testing.assert_array_equal(sb, g["sb"])
    np.testing.assert_array_equal(se, g["se"])
    Xc = oracle.encode(X, k, sb, se, 8)
    assert hashlib.sha256(Xc.tobytes()).digest() == g["codes_sha"].tobytes()
    Qc = oracle.encode(Q, k, sb, se, 8)
    np.testing.assert_array_equal(Qc, g["qcodes"])
    metric = synth.CONFIGS[cfg]["metric"]
    sc, ids = oracle.scan_topk_i8(Xc, Qc, 100, metric, oracle.norms_i8(Xc), oracle.norms_i8(Qc))
    np.testing.assert_array_equal(ids, g["ids"])
    np.testing.assert_array_equal(sc, g["scores"])


def test_hand_distances(oracle):
    # test_distances.py:32-44 through the scan: dot [1,2,3].[4,5,6] = 32,
    # 3*127^2 = 48387, l2(-128, 127) = 65025, [1,2] vs [4,6] -> 25
    sc, _ = oracle.scan_topk_i8(np.int8([[4, 5, 6]]), np.int8([[1, 2, 3]]), 1, 0)
    assert sc[0, 0] == -32.0
    sc, _ = oracle.scan_topk_i8(np.int8([[127, 127, 127]]), np.int8([[127, 127, 127]]), 1, 0)
    assert sc[0, 0] == -48387.0
    sc, _ = oracle.scan_topk_i8(np.int8([[-128]]), np.int8([[127]]), 1, 1)
    assert sc[0, 0] == 65025.0
    sc, _ = oracle.scan_topk_i8(np.int8([[4, 6]]), np.int8([[1, 2]]), 1, 1)
    assert sc[0, 0] == 25.0


def test_tie_order_and_full_sort(oracle):
    # test_exact.py:48-57 (int8 form): ties break by ascending id; k >= n
    # returns the full sort.
    X = np.int8([[1, 0], [1, 0], [0, 0], [1, 0]])
    _, ids = oracle.scan_topk_i8(X, np.int8([[1, 0]]), 4, 1)
    assert list(ids[0]) == [0, 1, 3, 2]
    _, ids = oracle.scan_topk_i8(np.int8([[5], [1], [3]]), np.int8([[0]]), 10, 1)
    assert list(ids[0]) == [1, 2, 0]


def test_oracle_equals_reference_kernel_on_fresh_instances(oracle):
    core = oracle.ref_core()
    if core is None:
        pytest.skip("reference _core not built here (make -C oracle ref)")
    rng = np.random.default_rng(2024)
    for i in range(30):
        n, d, nq = int(rng.integers(1, 900)), int(rng.integers(1, 40)), int(rng.integers(1, 4))
        metric = i % 3
        hi = 4 if i % 5 == 0 else 128
        X = rng.integers(-hi, hi, size=(n, d)).astype(np.int8)
        Q = rng.integers(-hi, hi, size=(nq, d)).astype(np.int8)
        X[~X.any(axis=1), 0] = 1
        Q[~Q.any(axis=1), 0] = 1
        k = int(rng.choice([1, 7, 100, n + 3]))
        xn, qn = core.norms(X), core.norms(Q)
        a = oracle.scan_topk_i8(X, Q, k, metric, xn, qn)
        b = core.scan_topk(X, Q, k, metric, xn, qn)
        np.testing.assert_array_equal(a[1], b[1])
        np.testing.assert_array_equal(a[0], b[0])


def test_pair_scores_equal_reference_scores(oracle):
    """The listed-pair scores (the batched HnswCore._dq, _core.pyx:483-494)
    against the reference: its full scan (k = n) gives every row's score per
    query, and its public dot / l2sq give the integer metrics per pair."""
    core = oracle.ref_core()
    if core is None:
        pytest.skip("reference _core not built here (make -C oracle ref)")
    rng = np.random.default_rng(77)
    for i in range(12):
        n, d, nq, m = int(rng.integers(2, 300)), int(rng.integers(1, 70)), 3, int(rng.integers(1, 20))
        metric = i % 3
        X = rng.integers(-128, 128, size=(n, d)).astype(np.int8)
        Q = rng.integers(-128, 128, size=(nq, d)).astype(np.int8)
        X[~X.any(axis=1), 0] = 1
        Q[~Q.any(axis=1), 0] = 1
        cand = rng.integers(-2, n + 2, size=(nq, m)).astype(np.int32)
        xn, qn = core.norms(X), core.norms(Q)
        got = oracle.pair_scores_i8(X, Q, cand, metric, xn, qn)
        sc, ids = core.scan_topk(X, Q, n, metric, xn, qn)
        for q in range(nq):
            by_id = dict(zip(ids[q].tolist(), sc[q].tolist()))
            for j in range(m):
                c = int(cand[q, j])
                want = by_id[c] if 0 <= c < n else np.inf
                assert got[q, j] == want
                if 0 <= c < n and metric == 0:
                    assert got[q, j] == -core.dot(Q[q], X[c])
                if 0 <= c < n and metric == 1:
                    assert got[q, j] == core.l2sq(Q[q], X[c])


# ----------------------------------------------- float32 path (_scan_f32) --

def test_scan_f32_matches_reference_golden(oracle, golden_scan_f32):
    for name, c in golden_scan_f32.items():
        np.testing.assert_array_equal(oracle.norms_f32(c["X"]), c["xn"], err_msg=name)
        sc, ids = oracle.scan_topk_f32(c["X"], c["Q"], int(c["k"]), int(c["metric"]), c["xn"],
                                       c["qn"])
        np.testing.assert_array_equal(ids, c["ids"], err_msg=name)
        np.testing.assert_array_equal(sc, c["scores"], err_msg=name)


def test_scan_f32_cfg_minis_ground_truth(oracle, golden_cfg):
    # the reference's float32 ground truth of the reduced BASELINE pipelines
    for cfg in (0, 1, 3):
        X, Q = synth.generate(cfg, n=6000, nq=24)
        metric = synth.CONFIGS[cfg]["metric"]
        _, ids = oracle.scan_topk_f32(X, Q, 100, metric, oracle.norms_f32(X), oracle.norms_f32(Q))
        np.testing.assert_array_equal(ids, golden_cfg[f"cfg{cfg}"]["gt32"])


def test_scan_f32_equals_reference_kernel_on_fresh_instances(oracle):
    core = oracle.ref_core()
    if core is None:
        pytest.skip("reference _core not built here (make -C oracle ref)")
    rng = np.random.default_rng(77)
    for i in range(24):
        n, d, nq = int(rng.integers(1, 700)), int(rng.integers(1, 90)), int(rng.integers(1, 4))
        metric = i % 3
        X = (rng.normal(size=(n, d)) * 10 ** rng.uniform(-3, 3, size=d)).astype(np.float32)
        Q = (rng.normal(size=(nq, d)) * 10 ** rng.uniform(-3, 3, size=d)).astype(np.float32)
        if i % 4 == 0:
            X = np.round(X).astype(np.float32)
            Q = np.round(Q).astype(np.float32)
        X[~X.any(axis=1), 0] = 1
        Q[~Q.any(axis=1), 0] = 1
        k = int(rng.choice([1, 7, 100, n + 3]))
        xn, qn = core.norms(X), core.norms(Q)
        np.testing.assert_array_equal(oracle.norms_f32(X), xn)
        a = oracle.scan_topk_f32(X, Q, k, metric, xn, qn)
        b = core.scan_topk(X, Q, k, metric, xn, qn)
        np.testing.assert_array_equal(a[1], b[1])
        np.testing.assert_array_equal(a[0], b[0])
