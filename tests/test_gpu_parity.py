"""Parity of the CUDA path (through the C-ABI) with the CPU oracle.

Bar: bit-exact codes, norms, int32 dots, top-k ids AND float64 scores for
every metric -- the reference's own contract (_core.pyx:8-14).  Sizes here
are ones the oracle finishes in seconds; the full BASELINE sizes are in
test_gpu_configs.py (oracle subsets + size-independent properties).
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_08919_b200 as qa  # noqa: E402
import synth  # noqa: E402
from paper_2110_08919_b200 import _backend, device as dev  # noqa: E402


def _rand_codes(rng, n, d, lo=-127, hi=128, nonzero=False):
    X = rng.integers(lo, hi, size=(n, d)).astype(np.int8)
    if nonzero:
        X[~X.any(axis=1), 0] = 1
    return X


def _scan_gpu(X, Q, k, metric, xn=None, qn=None):
    return _backend.scan_topk(X, Q, k, metric, xn, qn)


def _scan_oracle(oracle, X, Q, k, metric):
    return oracle.scan_topk_i8(X, Q, k, metric, oracle.norms_i8(X), oracle.norms_i8(Q))


# ----------------------------------------------------------------- encode --

def test_encode_golden(golden_encode):
    for name, c in golden_encode.items():
        x = torch.from_numpy(c["x"]).cuda()
        k, sb, se = (torch.from_numpy(c[f]).cuda() for f in ("k", "sb", "se"))
        codes = dev.encode(x, k, sb, se, int(c["bits"]))
        np.testing.assert_array_equal(codes.to_host(), c["codes"], err_msg=name)
        pad = codes.codes[:, codes.d:].cpu().numpy()
        assert not pad.any(), name
        w = c["codes"].astype(np.int64)
        np.testing.assert_array_equal(codes.sqnorm.cpu().numpy(), (w * w).sum(1), err_msg=name)


def test_encode_large_random_vs_oracle(oracle):
    rng = np.random.default_rng(5)
    for d in (1, 3, 100, 128, 257):
        x = (rng.normal(size=(3001, d)) * rng.uniform(0.1, 10, size=d)).astype(np.float32)
        x[::97, 0] = np.nan
        x[1::89, -1] = np.float32(1e-41)
        mn, mx = oracle.minmax(np.nan_to_num(x, nan=0.0))
        k, sb, se = oracle.fit_range((mn + mx) / 2, (mx - mn) / 2 * 0.8)
        for bits in (8, 5, 1):
            want = oracle.encode(x, k, sb, se, bits)
            got = dev.encode(torch.from_numpy(x).cuda(), *(torch.from_numpy(a).cuda()
                                                             for a in (k, sb, se)), bits)
            np.testing.assert_array_equal(got.to_host(), want, err_msg=f"d={d} bits={bits}")
            np.testing.assert_array_equal(got.norm.cpu().numpy(), oracle.norms_i8(want))


def test_minmax_exact(oracle):
    rng = np.random.default_rng(6)
    x = rng.normal(size=(50_001, 100)).astype(np.float32)
    mn, mx = dev.minmax(torch.from_numpy(x).cuda())
    omn, omx = oracle.minmax(x)
    np.testing.assert_array_equal(mn.double().cpu().numpy(), omn)
    np.testing.assert_array_equal(mx.double().cpu().numpy(), omx)


def test_norms_vs_oracle(oracle):
    rng = np.random.default_rng(7)
    X = _rand_codes(rng, 777, 200, -128, 128)
    np.testing.assert_array_equal(_backend.norms(X), oracle.norms_i8(X))


# ------------------------------------------------------------------- dots --

@pytest.mark.parametrize("d", [1, 16, 32, 33, 64, 100, 128, 200, 256, 512, 1024])
def test_tensor_core_dots_exact(d):
    rng = np.random.default_rng(d)
    n, nq = 1000 + d, 300 + (d % 7)
    X = _rand_codes(rng, n, d, -128, 128)
    Q = _rand_codes(rng, nq, d, -128, 128)
    want = Q.astype(np.int64) @ X.astype(np.int64).T
    db = dev.DeviceCodes.from_host(X)
    qs = dev.DeviceCodes.from_host(Q)
    tc = dev.debug_dots(db, qs, impl=0).cpu().numpy()
    np.testing.assert_array_equal(tc, want)
    simt = dev.debug_dots(db, qs, impl=1).cpu().numpy()
    np.testing.assert_array_equal(simt, want)


@pytest.mark.parametrize("nq", [1, 7, 64, 65, 128, 129, 256, 300])
def test_tensor_core_dots_query_tiles(nq):
    rng = np.random.default_rng(100 + nq)
    X = _rand_codes(rng, 4099, 128)
    Q = _rand_codes(rng, nq, 128)
    want = Q.astype(np.int64) @ X.astype(np.int64).T
    got = dev.debug_dots(dev.DeviceCodes.from_host(X), dev.DeviceCodes.from_host(Q)).cpu().numpy()
    np.testing.assert_array_equal(got, want)


# ------------------------------------------------------------------- scan --

def test_scan_golden(golden_scan):
    for name, c in golden_scan.items():
        sc, ids = _scan_gpu(c["X"], c["Q"], int(c["k"]), int(c["metric"]), c["xn"], c["qn"])
        np.testing.assert_array_equal(ids, c["ids"], err_msg=name)
        np.testing.assert_array_equal(sc, c["scores"], err_msg=name)


def test_gate2_random_instances(oracle):
    # test_acceptance.py:116-135 (int8 half): 200 instances, n<=1000, d<=32,
    # all metrics, bit-exact ids and scores through exact_topk
    for i in range(200):
        rng = np.random.default_rng(1000 + i)
        n, d = int(rng.integers(1, 1001)), int(rng.integers(1, 33))
        metric = qa.Metric(i % 3)
        X = _rand_codes(rng, n, d, nonzero=True)
        q = _rand_codes(rng, 1, d, nonzero=True)[0]
        k = min(int(rng.choice([1, 10, 100])), n)
        res = qa.exact_topk(qa.DenseDataset(X), q, k, metric)
        sc, ids = _scan_oracle(oracle, X, q[None], k, int(metric))
        np.testing.assert_array_equal(res.ids, ids[0])
        np.testing.assert_array_equal(res.scores, sc[0])


def test_exact_hand_cases():
    X = qa.DenseDataset(np.int8([[1], [2], [3]]))
    res = qa.exact_topk(X, np.int8([4]), 1, qa.Metric.L2_SQUARED)
    assert res.ids[0] == 2 and res.scores[0] == 1.0
    ties = qa.DenseDataset(np.int8([[1, 0], [1, 0], [0, 0], [1, 0]]))
    assert list(qa.exact_topk(ties, np.int8([1, 0]), 4, qa.Metric.L2_SQUARED).ids) == [0, 1, 3, 2]
    full = qa.exact_topk(qa.DenseDataset(np.int8([[5], [1], [3]])), np.int8([0]), 10,
                         qa.Metric.L2_SQUARED)
    assert list(full.ids) == [1, 2, 0] and len(full) == 3
    gt = qa.batch_ground_truth(qa.DenseDataset(np.int8([[1, 1]])),
                               qa.DenseDataset(np.int8([[2, 2]])), 1, qa.Metric.L2_SQUARED)
    np.testing.assert_array_equal(gt.ids, [[0]])
    # inner product of zero vector scores -0.0 exactly like the reference
    r = qa.exact_topk(qa.DenseDataset(np.int8([[0, 0], [1, 1]])), np.int8([0, 0]), 2,
                      qa.Metric.INNER_PRODUCT)
    assert np.signbit(r.scores[0]) and r.scores[0] == 0.0
    with pytest.raises(qa.ZeroNorm):
        qa.exact_topk(qa.DenseDataset(np.int8([[1, 0], [0, 0]])), np.int8([1, 0]), 1,
                      qa.Metric.ANGULAR)


def test_self_query_property():
    rng = np.random.default_rng(4)
    X = _rand_codes(rng, 3000, 24)
    X = np.unique(X, axis=0)
    gt = qa.batch_ground_truth(qa.DenseDataset(X), qa.DenseDataset(X), 1, qa.Metric.L2_SQUARED)
    np.testing.assert_array_equal(gt.ids[:, 0], np.arange(X.shape[0]))


@pytest.mark.parametrize("metric", [0, 1, 2])
@pytest.mark.parametrize("k", [1, 10, 32, 33, 64, 65, 100, 128, 129, 1000])
def test_scan_mid_size_vs_oracle(oracle, metric, k):
    rng = np.random.default_rng(10 * metric + k)
    X = _rand_codes(rng, 20_000, 96, nonzero=True)
    Q = _rand_codes(rng, 70, 96, nonzero=True)
    sc, ids = _scan_gpu(X, Q, k, metric, oracle.norms_i8(X), oracle.norms_i8(Q))
    osc, oids = _scan_oracle(oracle, X, Q, k, metric)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(sc, osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_heavy_ties_exercise_overflow_retry(oracle, metric):
    # narrow code range: thousands of rows share each score, so candidate
    # lists overflow and the capacity-retry path must restore exactness.
    rng = np.random.default_rng(77 + metric)
    X = _rand_codes(rng, 60_000, 8, -2, 3, nonzero=True)
    X[:20_000] = X[0]
    Q = np.repeat(X[:1], 3, axis=0)
    Q[1] = _rand_codes(rng, 1, 8, -2, 3, nonzero=True)[0]
    sc, ids = _scan_gpu(X, Q, 100, metric, oracle.norms_i8(X), oracle.norms_i8(Q))
    osc, oids = _scan_oracle(oracle, X, Q, 100, metric)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(sc, osc)


def test_many_queries_and_edge_shapes(oracle):
    rng = np.random.default_rng(9)
    for n, nq, d, k in ((1, 5, 3, 1), (1, 5, 3, 10), (129, 513, 16, 128), (5000, 1500, 40, 30),
                        (300, 2, 200, 300), (257, 3, 64, 2048),
                        (3000, 70, 1024, 10),    # widest tensor-core K (64-query tiles)
                        (2000, 7, 1500, 10)):    # K > 1024: the dp4a filter
        for metric in (0, 1, 2):
            X = _rand_codes(rng, n, d, nonzero=True)
            Q = _rand_codes(rng, nq, d, nonzero=True)
            sc, ids = _scan_gpu(X, Q, k, metric, oracle.norms_i8(X), oracle.norms_i8(Q))
            osc, oids = _scan_oracle(oracle, X, Q, k, metric)
            np.testing.assert_array_equal(ids, oids, err_msg=f"{n} {nq} {d} {k} {metric}")
            np.testing.assert_array_equal(sc, osc)


def test_host_c_abi_entry(oracle):
    import ctypes

    from paper_2110_08919_b200._lib import check, lib

    rng = np.random.default_rng(11)
    X = _rand_codes(rng, 3000, 50, nonzero=True)
    Q = _rand_codes(rng, 17, 50, nonzero=True)
    for metric in (0, 1, 2):
        xn, qn = oracle.norms_i8(X), oracle.norms_i8(Q)
        out_s = np.empty((17, 100), np.float64)
        out_i = np.empty((17, 100), np.int32)
        p = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        check(lib.qa_scan_topk_i8_host(p(X), 3000, 50, p(Q), 17, 100, metric, p(xn), p(qn),
                                       p(out_s), p(out_i)))
        osc, oids = _scan_oracle(oracle, X, Q, 100, metric)
        np.testing.assert_array_equal(out_i, oids)
        np.testing.assert_array_equal(out_s, osc)


# ------------------------------------------------- BASELINE configs (mini) --

@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_cfg_minis_golden(golden_cfg, cfg):
    g = golden_cfg[f"cfg{cfg}"]
    X, Q = synth.generate(cfg, n=6000, nq=24)
    c = synth.CONFIGS[cfg]
    x = torch.from_numpy(X).cuda()
    index = qa.Int8Index.build(x, qa.Metric(c["metric"]), c["calibration"])
    np.testing.assert_array_equal(index.params.k, g["k"])
    np.testing.assert_array_equal(index.params.sb, g["sb"])
    np.testing.assert_array_equal(index.params.se, g["se"])
    assert hashlib.sha256(index.codes_in_input_order().tobytes()).digest() == g["codes_sha"].tobytes()
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    np.testing.assert_array_equal(qc.to_host(), g["qcodes"])
    sc, ids = index.search_codes(qc, 100)
    np.testing.assert_array_equal(ids.cpu().numpy(), g["ids"])
    np.testing.assert_array_equal(sc.cpu().numpy(), g["scores"])
    r = qa.recall_at_k(qa.GroundTruth(g["gt32"]), ids.cpu().numpy(), 100)
    r_ref = qa.recall_at_k(qa.GroundTruth(g["gt32"]), g["ids"], 100)
    assert abs(r.mean - r_ref.mean) <= 0.001


def test_cfg0_full_parity(oracle):
    # BASELINE config 0 at full size: 100k x 128, 1000 queries, L2, min/max.
    X, Q = synth.generate(0)
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric.L2_SQUARED, "minmax")
    mn, mx = oracle.minmax(X)
    k, sb, se = oracle.fit_range((mn + mx) / 2.0, (mx - mn) / 2.0)
    np.testing.assert_array_equal(index.params.sb, sb)
    np.testing.assert_array_equal(index.params.se, se)
    Xc = oracle.encode(X, k, sb, se, 8)
    Qc = oracle.encode(Q, k, sb, se, 8)
    np.testing.assert_array_equal(index.codes_in_input_order(), Xc)
    sc, ids = index.search(torch.from_numpy(Q).cuda(), 100)
    osc, oids = _scan_oracle(oracle, Xc, Qc, 100, 1)
    np.testing.assert_array_equal(ids.cpu().numpy(), oids)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)


# ------------------------------------------- float32 exact search (8f-1) --

def test_scan_f32_golden(golden_scan_f32):
    for name, c in golden_scan_f32.items():
        np.testing.assert_array_equal(_backend.norms(c["X"]), c["xn"], err_msg=name)
        sc, ids = _backend.scan_topk(c["X"], c["Q"], int(c["k"]), int(c["metric"]), c["xn"],
                                     c["qn"])
        np.testing.assert_array_equal(ids, c["ids"], err_msg=name)
        np.testing.assert_array_equal(sc, c["scores"], err_msg=name)


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_scan_f32_vs_oracle_multi_round(oracle, metric):
    # n spans several 16384-row rounds and nq several 1024-query chunks'
    # worth of CTA tiles; k = 1, 100, 2048 (the limit)
    rng = np.random.default_rng(31 + metric)
    X = (rng.normal(size=(40_000, 77)) * rng.uniform(0.1, 5, size=77)).astype(np.float32)
    X[5000:5100] = X[:100]            # duplicated rows: exact score ties
    Q = (rng.normal(size=(70, 77)) * rng.uniform(0.1, 5, size=77)).astype(np.float32)
    xn, qn = oracle.norms_f32(X), oracle.norms_f32(Q)
    for k in (1, 100, 2048):
        sc, ids = _backend.scan_topk(X, Q, k, metric, xn, qn)
        osc, oids = oracle.scan_topk_f32(X, Q, k, metric, xn, qn)
        np.testing.assert_array_equal(ids, oids)
        np.testing.assert_array_equal(sc, osc)


def test_scan_f32_many_queries_and_id_offset(oracle):
    rng = np.random.default_rng(8)
    X = np.round(rng.normal(size=(3000, 20)) * 3).astype(np.float32)   # heavy ties
    Q = np.round(rng.normal(size=(2500, 20)) * 3).astype(np.float32)   # > 1 query chunk
    sc, ids = dev.scan_topk_f32(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), 10, 1,
                                id_offset=1000)
    osc, oids = oracle.scan_topk_f32(X, Q, 10, 1)
    np.testing.assert_array_equal(ids.cpu().numpy(), oids + 1000)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)


@pytest.mark.parametrize("cfg", [0, 1, 3])
def test_ground_truth_and_recall_cfg_minis(golden_cfg, cfg):
    # GPU float32 ground truth == the reference's (gt32 fixture), and the
    # int8 search's recall against it equals the reference's exactly
    g = golden_cfg[f"cfg{cfg}"]
    X, Q = synth.generate(cfg, n=6000, nq=24)
    metric = qa.Metric(synth.CONFIGS[cfg]["metric"])
    gt = qa.batch_ground_truth(qa.DenseDataset(X), qa.DenseDataset(Q), 100, metric)
    np.testing.assert_array_equal(gt.ids, g["gt32"])
    r = qa.recall_at_k(gt, g["ids"], 100)
    r_ref = qa.recall_at_k(qa.GroundTruth(g["gt32"]), g["ids"], 100)
    assert r.mean == r_ref.mean


# ------------------------------------------------------------ sharding --

@pytest.mark.parametrize("G,k", [(2, 100), (3, 100), (8, 100), (3, 3000), (5, 2500)])
def test_virtual_shards_merge_equals_full(oracle, G, k):
    # k > 2048: the merge-path tree (shared-memory merge beyond its limit)
    from paper_2110_08919_b200.sharded import pad_topk, shard_bounds

    rng = np.random.default_rng(G + k)
    X = _rand_codes(rng, 10_007, 32, -6, 7, nonzero=True)   # many ties across shards
    Q = _rand_codes(rng, 40 if k <= 100 else 6, 32, -6, 7, nonzero=True)
    for metric in (0, 1, 2):
        db = dev.DeviceCodes.from_host(X)
        qs = dev.DeviceCodes.from_host(Q)
        kin = min(k, -(-X.shape[0] // G))
        parts_s, parts_i = [], []
        for r in range(G):
            lo, hi = shard_bounds(X.shape[0], G, r)
            s, i = dev.scan_topk(db.slice_rows(lo, hi), qs, k, metric, id_offset=lo)
            s, i = pad_topk(s, i, kin)
            parts_s.append(s)
            parts_i.append(i)
        ms, mi = dev.merge_topk(torch.stack(parts_s), torch.stack(parts_i), k)
        osc, oids = _scan_oracle(oracle, X, Q, k, metric)
        np.testing.assert_array_equal(mi.cpu().numpy(), oids)
        np.testing.assert_array_equal(ms.cpu().numpy(), osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
@pytest.mark.parametrize("stratify", [False, True])
def test_norm_sorted_index_equals_unsorted(oracle, metric, stratify):
    # The index stores rows in norm bands (tight per-unit filter bounds; with
    # `stratify` after a stratified sample region, which needs >= 131072
    # rows) and reports/tie-breaks by the caller's ids via row_ids: results
    # must be identical to the unsorted layout and to the oracle.
    rng = np.random.default_rng(31 + metric)
    X = _rand_codes(rng, 140_011, 64, -20, 21, nonzero=True)
    Q = _rand_codes(rng, 300, 64, -20, 21, nonzero=True)
    db = dev.DeviceCodes.from_host(X)
    qs = dev.DeviceCodes.from_host(Q)
    srt = db.sorted_by_norm(stratify=stratify)
    ids = srt.ids.cpu().numpy()
    assert sorted(ids.tolist()) == list(range(X.shape[0]))
    sq = srt.sqnorm.cpu().numpy()
    full = (sq.shape[0] // 128) * 128
    assert (np.diff(sq[:full].reshape(-1, 128), axis=1) >= 0).all()  # sorted within tiles
    np.testing.assert_array_equal(srt.to_host(), X[ids])
    a = dev.scan_topk(db, qs, 100, metric)
    b = dev.scan_topk(srt, qs, 100, metric, id_offset=7)
    np.testing.assert_array_equal(a[1].cpu().numpy() + 7, b[1].cpu().numpy())
    np.testing.assert_array_equal(a[0].cpu().numpy(), b[0].cpu().numpy())
    osc, oids = _scan_oracle(oracle, X, Q, 100, metric)
    np.testing.assert_array_equal(a[1].cpu().numpy(), oids)
    np.testing.assert_array_equal(a[0].cpu().numpy(), osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
@pytest.mark.parametrize("force_j", [None, "1"])
def test_threshold_estimate_path_exact(oracle, monkeypatch, metric, force_j):
    # The estimated-bound final pass (qa_api.cu plan_scan): a small prefix
    # triggers it at this size; j=1 (the best prefix score as the bound)
    # makes the estimate fail for many queries, which must then be
    # recomputed without it -- results exact either way.
    from paper_2110_08919_b200 import _lib

    monkeypatch.setenv("QA_B200_EST_ROWS", "2048")
    if force_j:
        monkeypatch.setenv("QA_B200_EST_J", force_j)
    rng = np.random.default_rng(400 + metric)
    X = _rand_codes(rng, 40_000, 64, -30, 31, nonzero=True)
    Q = _rand_codes(rng, 300, 64, -30, 31, nonzero=True)
    db = dev.DeviceCodes.from_host(X).sorted_by_norm()
    qs = dev.DeviceCodes.from_host(Q)
    sc, ids = dev.scan_topk(db, qs, 20, metric)
    st = _lib.last_scan_stats()
    osc, oids = _scan_oracle(oracle, X, Q, 20, metric)
    np.testing.assert_array_equal(ids.cpu().numpy(), oids)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    if force_j:
        assert st["retries"] >= 1  # the recompute path ran


# ------------------------------------------------ filter effectiveness --

@pytest.mark.parametrize("metric", [0, 1])
def test_filter_bounds_hold_on_large_dots(oracle, metric):
    # SIFT-like codes under min/max calibration sit near -128, so dots are
    # ~1e6 -- beyond one bias MMA's range (516k).  The filter must still
    # reject most rows (a bound clamped to the bias range used to pass them
    # all) and the L2 threshold estimate must hold (no recompute).
    from paper_2110_08919_b200 import _lib
    X, Q = synth.generate(2, n=300_000, nq=512)
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric(metric), "minmax")
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    sc, ids = index.search_codes(qc, 100)
    st = _lib.last_scan_stats()
    assert st["retries"] == 0
    assert st["candidates"] < 60 * 100 * 512, st
    Xc = index.codes_in_input_order()
    osc, oids = _scan_oracle(oracle, Xc, qc.to_host()[:16], 100, metric)
    np.testing.assert_array_equal(ids[:16].cpu().numpy(), oids)
    np.testing.assert_array_equal(sc[:16].cpu().numpy(), osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
@pytest.mark.parametrize("force_j", [None, "1"])
@pytest.mark.parametrize("layout", ["plain", "bands"])
def test_sampled_estimate_exact(oracle, monkeypatch, metric, force_j, layout):
    # The estimate pass (filter mode 4) reads every stride-th tile, keeps the
    # best row per (query, bucket), and the j-th best bucket bounds one pass
    # over every row; the check after it needs the k-th at least as good.
    # j = 1 makes the estimate fail for most queries (recompute path); exact
    # either way, on caller order and on the interleaved norm blocks.
    from paper_2110_08919_b200 import _lib

    monkeypatch.setenv("QA_B200_EST_ROWS", "8192")
    if force_j:
        monkeypatch.setenv("QA_B200_EST_J", force_j)
    rng = np.random.default_rng(500 + metric)
    X = _rand_codes(rng, 60_000, 64, -30, 31, nonzero=True)
    Q = _rand_codes(rng, 300, 64, -30, 31, nonzero=True)
    db = dev.DeviceCodes.from_host(X)
    if layout == "bands":
        db = db.sorted_by_norm(stratify=False)
    qs = dev.DeviceCodes.from_host(Q)
    sc, ids = dev.scan_topk(db, qs, 20, metric)
    st = _lib.last_scan_stats()
    osc, oids = _scan_oracle(oracle, X, Q, 20, metric)
    np.testing.assert_array_equal(ids.cpu().numpy(), oids)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    assert st["rounds"] <= 2 + (3 * st["retries"] + 20)
    if force_j:
        assert st["retries"] >= 1
    else:
        assert st["rounds"] == 2 and st["retries"] == 0, st


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_large_k_beyond_int8_select(oracle, metric):
    # k above the int8 select's limit (2048) runs the float64-exact scan on
    # the codes (norm-sorted index: stored rows are scattered back to caller
    # order first) -- results identical to the reference order.
    rng = np.random.default_rng(900 + metric)
    X = _rand_codes(rng, 9000, 40, -6, 7, nonzero=True)   # heavy ties
    Q = _rand_codes(rng, 7, 40, -6, 7, nonzero=True)
    db = dev.DeviceCodes.from_host(X).sorted_by_norm()
    qs = dev.DeviceCodes.from_host(Q)
    for k in (2049, 5000, 9000):
        sc, ids = dev.scan_topk(db, qs, k, metric, id_offset=3)
        osc, oids = _scan_oracle(oracle, X, Q, k, metric)
        np.testing.assert_array_equal(ids.cpu().numpy(), oids + 3)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)
    # any k (reference: keff = min(k, n) for every k, _core.pyx:348-365):
    # beyond the shared-memory select, every score is sorted per query
    Xb = _rand_codes(rng, 20_000, 8, nonzero=True)
    Qb = _rand_codes(rng, 3, 8, nonzero=True)
    big = dev.DeviceCodes.from_host(Xb).sorted_by_norm()
    for k in (16_000, 20_000, 25_000):
        sc, ids = dev.scan_topk(big, dev.DeviceCodes.from_host(Qb), k, metric)
        osc, oids = _scan_oracle(oracle, Xb, Qb, k, metric)
        np.testing.assert_array_equal(ids.cpu().numpy(), oids)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_any_k_float32_path(oracle, metric):
    rng = np.random.default_rng(950 + metric)
    X = rng.standard_normal((18_000, 9)).astype(np.float32)
    X[::7] = X[3]  # ties
    Q = rng.standard_normal((2, 9)).astype(np.float32)
    xn, qn = oracle.norms_f32(X), oracle.norms_f32(Q)
    sc, ids = _backend.scan_topk(X, Q, 17_000, metric, xn, qn)
    osc, oids = oracle.scan_topk_f32(X, Q, 17_000, metric, xn, qn)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(sc, osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_rows_wider_than_int32_safe_bound(oracle, metric):
    # d beyond the int32-exact worst case (L2: 33025, others: 131071) takes
    # the float64-exact route; equal to the reference whenever its int32 sums
    # do not wrap (small codes here)
    rng = np.random.default_rng(990 + metric)
    d = 33_100 if metric == 1 else 131_100
    X = _rand_codes(rng, 300, d, -3, 4, nonzero=True)
    Q = _rand_codes(rng, 2, d, -3, 4, nonzero=True)
    sc, ids = _scan_gpu(X, Q, 20, metric, oracle.norms_i8(X), oracle.norms_i8(Q))
    osc, oids = _scan_oracle(oracle, X, Q, 20, metric)
    np.testing.assert_array_equal(ids, oids)
    np.testing.assert_array_equal(sc, osc)


def test_pair_distances_backend_and_module():
    # reference test_distances.py:32-54 hand values, through _backend.dot /
    # l2sq (the seam's pair kernels) and the distances module wrappers
    from paper_2110_08919_b200 import distances as D
    assert _backend.dot(np.int8([1, 2, 3]), np.int8([4, 5, 6])) == 32.0
    assert _backend.dot(np.int8([127] * 3), np.int8([127] * 3)) == 48387.0
    assert _backend.l2sq(np.int8([-128]), np.int8([127])) == 65025.0
    assert _backend.l2sq(np.int8([1, 2]), np.int8([4, 6])) == 25.0
    assert _backend.dot(np.int8([]), np.int8([])) == 0.0
    assert D.dot_i8(np.int8([1, -2]), np.int8([3, 4])) == -5
    with pytest.raises(ValueError, match="length mismatch"):
        _backend.dot(np.int8([1]), np.int8([1, 2]))
    with pytest.raises(ValueError, match="dtype mismatch"):
        _backend.l2sq(np.int8([1]), np.float32([1]))
    with pytest.raises(qa.DimensionMismatch):
        D.dot_f32(np.float32([1]), np.float32([1, 2]))
    rng = np.random.default_rng(3)
    for _ in range(5):
        a = rng.normal(size=77).astype(np.float32)
        b = rng.normal(size=77).astype(np.float32)
        acc = 0.0
        for x, y in zip(a.tolist(), b.tolist()):
            acc += x * y                        # float64, sequential: _dot_f
        assert D.dot_f32(a, b) == acc
        l2 = 0.0
        for x, y in zip(a.tolist(), b.tolist()):
            t = x - y
            l2 += t * t
        assert D.l2sq_f32(a, b) == l2
        assert D.distance(qa.Metric.INNER_PRODUCT, a, b) == -acc
        na, nb = float(np.sqrt(D.dot_f32(a, a))), float(np.sqrt(D.dot_f32(b, b)))
        assert D.angular(a, b) == 1.0 - acc / (na * nb)
    with pytest.raises(qa.ZeroNorm):
        D.angular(np.int8([0, 0]), np.int8([1, 1]))


def test_index_angular_rejects_zero_norm_codes():
    # reference exact.py:67-69: angular needs nonzero vectors (ZeroNorm)
    X = np.zeros((300, 8), np.float32)
    X[:, 0] = np.linspace(0.0, 1.0, 300, dtype=np.float32)   # row 0 (all zero) -> code norm 0
    idx = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric.ANGULAR, "symmetric")
    zero_rows = int((idx.codes.sqnorm == 0).sum())
    q = torch.from_numpy(np.ones((2, 8), np.float32)).cuda()
    if zero_rows:
        with pytest.raises(qa.ZeroNorm):
            idx.search(q, 5)
    qz = torch.zeros((1, 8), dtype=torch.float32, device="cuda")
    X2 = np.ones((50, 8), np.float32)
    idx2 = qa.Int8Index.build(torch.from_numpy(X2).cuda(), qa.Metric.ANGULAR, "symmetric")
    with pytest.raises(qa.ZeroNorm):
        idx2.search(qz, 5)


@pytest.mark.parametrize("n", [1, 50, 127, 128, 129, 300])
def test_sorted_index_tiny(oracle, n):
    # layouts of indexes smaller than one tile / one norm block
    rng = np.random.default_rng(n)
    X = _rand_codes(rng, n, 8, nonzero=True)
    Q = _rand_codes(rng, 3, 8, nonzero=True)
    for stratify in (False, True):
        db = dev.DeviceCodes.from_host(X).sorted_by_norm(stratify=stratify)
        assert sorted(db.ids.cpu().numpy().tolist()) == list(range(n))
        sc, ids = dev.scan_topk(db, dev.DeviceCodes.from_host(Q), 5, 1)
        osc, oids = _scan_oracle(oracle, X, Q, 5, 1)
        np.testing.assert_array_equal(ids.cpu().numpy(), oids)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)


def test_acceptance_gate4_pipeline_matches_reference():
    # The reference's gate 4 (test_acceptance.py:176-193, synthetic corpus),
    # every step on the GPU: float32 ground truth (float64-exact scan),
    # estimate_stats -> fit(ABS_MAX) -> quantize_dataset (encode kernel) ->
    # int8 ground truth (tensor-core scan) -> recall@100.  Ids, windows and
    # recall equal the reference's own run (tests/golden/gate4.npz).
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "gate4.npz")
    corpus = qa.generate_synthetic(50_000, 64, 0.0, 0.05, 2)
    queries = qa.generate_synthetic(100, 64, 0.0, 0.05, 1002)
    gt = qa.batch_ground_truth(corpus, queries, 100, qa.Metric.INNER_PRODUCT)
    np.testing.assert_array_equal(gt.ids, g["gt"])
    params = qa.fit(qa.estimate_stats(corpus), 8, qa.QuantMode.ABS_MAX).params
    np.testing.assert_array_equal(params.k, g["k"])
    np.testing.assert_array_equal(params.sb, g["sb"])
    np.testing.assert_array_equal(params.se, g["se"])
    ci8 = qa.quantize_dataset(corpus, params)
    qi8 = qa.quantize_dataset(queries, params)
    approx = qa.batch_ground_truth(ci8, qi8, 100, qa.Metric.INNER_PRODUCT)
    np.testing.assert_array_equal(approx.ids, g["approx"])
    rec = qa.recall_at_k(gt, approx, 100).mean
    assert rec == float(g["recall"]) and rec >= 0.95


# ------------------------------------------------- asynchronous search --

@pytest.mark.parametrize("metric", [0, 1, 2])
def test_async_search_repairs_overflow_on_device(oracle, metric):
    # heavy ties overflow the candidate lists; the asynchronous entry has no
    # host retry -- the flagged queries are recomputed by the device-side
    # repair pass, in stream order
    rng = np.random.default_rng(1300 + metric)
    X = _rand_codes(rng, 60_000, 8, -2, 3, nonzero=True)
    X[:20_000] = X[0]
    Q = _rand_codes(rng, 300, 8, -2, 3, nonzero=True)
    Q[:100] = X[0]
    db = dev.DeviceCodes.from_host(X).sorted_by_norm()
    qs = dev.DeviceCodes.from_host(Q)
    for k in (10, 100, 700):
        sc, ids = dev.scan_topk(db, qs, k, metric, id_offset=2, sync=False)
        osc, oids = _scan_oracle(oracle, X, Q, k, metric)
        np.testing.assert_array_equal(ids.cpu().numpy(), oids + 2)
        np.testing.assert_array_equal(sc.cpu().numpy(), osc)


@pytest.mark.parametrize("metric", [0, 1, 2])
def test_async_search_repairs_failed_estimates(oracle, monkeypatch, metric):
    # j = 1 makes the threshold estimate fail for many queries
    monkeypatch.setenv("QA_B200_EST_ROWS", "2048")
    monkeypatch.setenv("QA_B200_EST_J", "1")
    rng = np.random.default_rng(1400 + metric)
    X = _rand_codes(rng, 40_000, 64, -30, 31, nonzero=True)
    Q = _rand_codes(rng, 300, 64, -30, 31, nonzero=True)
    db = dev.DeviceCodes.from_host(X).sorted_by_norm()
    qs = dev.DeviceCodes.from_host(Q)
    sc, ids = dev.scan_topk(db, qs, 20, metric, sync=False)
    osc, oids = _scan_oracle(oracle, X, Q, 20, metric)
    np.testing.assert_array_equal(ids.cpu().numpy(), oids)
    np.testing.assert_array_equal(sc.cpu().numpy(), osc)


def test_async_index_batches_back_to_back(oracle):
    # many stream-ordered searches without a host synchronisation between
    # them, outputs into preallocated buffers (the serving loop)
    X, Q = synth.generate(2, n=200_000, nq=3 * 300)
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric.L2_SQUARED, "minmax")
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    outs = [(torch.empty((300, 100), dtype=torch.float64, device="cuda"),
             torch.empty((300, 100), dtype=torch.int32, device="cuda")) for _ in range(3)]
    for i in range(3):
        index.search_codes(qc.slice_rows(300 * i, 300 * (i + 1)), 100, out=outs[i])
    Xc = index.codes_in_input_order()
    Qc = qc.to_host()
    for i in range(3):
        osc, oids = _scan_oracle(oracle, Xc, Qc[300 * i: 300 * i + 8], 100, 1)
        np.testing.assert_array_equal(outs[i][1][:8].cpu().numpy(), oids)
        np.testing.assert_array_equal(outs[i][0][:8].cpu().numpy(), osc)


def test_ip_index_on_sorted_caller_rows_keeps_estimate(oracle):
    # a caller corpus sorted by norm (clustered input) must not reach the
    # threshold estimate in caller order: the IP index stores a fixed
    # pseudo-random order, so no query needs the recompute
    from paper_2110_08919_b200 import _lib

    X, Q = synth.sift_like(300_000, 64, 128, 7)
    X = X[np.argsort((X.astype(np.float64) ** 2).sum(1))[::-1]].copy()
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric.INNER_PRODUCT, "minmax")
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    sc, ids = index.search_codes(qc, 10, sync=True)
    assert _lib.last_scan_stats()["retries"] == 0
    Xc = index.codes_in_input_order()
    osc, oids = _scan_oracle(oracle, Xc, qc.to_host()[:6], 10, 0)
    np.testing.assert_array_equal(ids[:6].cpu().numpy(), oids)
    np.testing.assert_array_equal(sc[:6].cpu().numpy(), osc)
