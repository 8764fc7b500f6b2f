"""Host-side API semantics mirrored from the reference's own tests
(test_quantizer.py, test_exact.py validation, test_bench.py recall) --
everything that runs before or around the kernels."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2110_08919_b200 as qa
from paper_2110_08919_b200.quantizer import RangeStats


def _stats(mu, half, sigma=None):
    mu = np.asarray(mu, dtype=np.float64)
    half = np.asarray(half, dtype=np.float64)
    sigma = half if sigma is None else np.asarray(sigma, dtype=np.float64)
    return qa.DimensionStats(mu=mu, sigma=sigma, min=mu - half, max=mu + half,
                             trimmed_absmax=half, pooled_mu=float(mu.mean()),
                             pooled_sigma=float(sigma.mean()), count=2)


def test_backend_identity():
    assert qa.BACKEND == "cuda"
    from paper_2110_08919_b200._backend import get_backend

    assert get_backend().BACKEND == "cuda"
    with pytest.raises(ValueError):
        get_backend("fortran")


def test_dataset_invariants():
    ds = qa.DenseDataset(np.zeros((3, 2), dtype=np.float32))
    assert not ds.data.flags.writeable and ds.n == 3 and ds.d == 2
    assert ds.elem is qa.ElemKind.FLOAT32
    with pytest.raises(ValueError):
        qa.DenseDataset(np.zeros(3, dtype=np.float32))
    with pytest.raises(ValueError):
        qa.DenseDataset(np.zeros((2, 2), dtype=np.float64))
    with pytest.raises(qa.DimensionMismatch):
        qa.DenseDataset(np.zeros((1, qa.MAX_DIM + 1), dtype=np.int8))
    f = np.asfortranarray(np.arange(6, dtype=np.float32).reshape(2, 3))
    assert qa.DenseDataset(f).data.flags.c_contiguous


def test_ground_truth_validation():
    gt = qa.GroundTruth(np.array([[0, 1], [2, 3]], dtype=np.int64))
    assert gt.ids.dtype == np.int32 and gt.nq == 2 and gt.k == 2
    with pytest.raises(ValueError):
        qa.GroundTruth(np.array([[0, 0]]))
    with pytest.raises(ValueError):
        qa.GroundTruth(np.array([[-1, 0]]))


def test_params_validation():
    f = np.float32
    with pytest.raises(ValueError):
        qa.QuantizerParams(bits=9, mode=qa.QuantMode.ABS_MAX, k=f([0]), sb=f([-1]), se=f([1]))
    with pytest.raises(ValueError):
        qa.QuantizerParams(bits=8, mode=qa.QuantMode.ABS_MAX, k=f([0]), sb=f([1]), se=f([1]))
    p = qa.QuantizerParams(bits=8, mode=1, k=f([0]), sb=f([-1]), se=f([1]))
    assert p.lo_code == -128 and p.hi_code == 127 and p.mode is qa.QuantMode.ABS_MAX


def test_fit_formulas_and_degeneracy():
    # test_quantizer.py:71-76 sigma clamp; 108-114 degenerate widening
    p = qa.fit(_stats([0.0], [0.1]), 8, qa.QuantMode.SIGMA_CLAMP).params
    assert p.k[0] == np.float32(0.0) and p.sb[0] == np.float32(-0.1) and p.se[0] == np.float32(0.1)
    r = qa.fit(_stats([0.5, 1.5], [0.0, 0.5]), 8, qa.QuantMode.SIGMA_CLAMP)
    assert r.degenerate_dims == (0,)
    assert r.params.sb[0] == np.float32(0.5 - 1e-6) and r.params.se[0] == np.float32(0.5 + 1e-6)
    # float32 collapse around a large centre -> ulp window (test_quantizer.py:117-123)
    r = qa.fit(_stats([1e8], [4e-6]), 8, qa.QuantMode.SIGMA_CLAMP)
    p = r.params
    assert r.degenerate_dims == (0,) and float(p.sb[0]) < float(p.k[0]) < float(p.se[0])
    for bits in (0, 9, -1):
        with pytest.raises(ValueError):
            qa.fit(_stats([0.0], [1.0]), bits, qa.QuantMode.SIGMA_CLAMP)


def test_fit_minmax_and_symmetric_match_golden(golden_cfg):
    for cfg in (0, 1, 3):
        g = golden_cfg[f"cfg{cfg}"]
        st = RangeStats(min=g["mn"], max=g["mx"], count=6000)
        p = (qa.fit_symmetric(st) if cfg == 1 else qa.fit_minmax(st)).params
        np.testing.assert_array_equal(p.k, g["k"])
        np.testing.assert_array_equal(p.sb, g["sb"])
        np.testing.assert_array_equal(p.se, g["se"])


def test_quantize_value_hand_cases():
    p = qa.fit(_stats([0.0], [0.1]), 8, qa.QuantMode.SIGMA_CLAMP).params
    assert [qa.quantize_value(x, 0, p) for x in (0.0, 0.05, -0.1, 0.1, 0.5, -0.2)] == \
        [0, 64, -128, 127, 127, -128]
    assert qa.quantize_value(float("nan"), 0, p) == -128
    assert qa.dequantize_value(0, 0, p) == pytest.approx(0.000390625, abs=1e-9)


def test_metric_parse():
    assert qa.Metric.parse("ip") is qa.Metric.INNER_PRODUCT
    assert qa.Metric.parse("L2") is qa.Metric.L2_SQUARED
    assert qa.Metric.ANGULAR.short_name == "angular"
    with pytest.raises(ValueError):
        qa.Metric.parse("cosine-ish")


def test_exact_validation_before_device():
    corpus = qa.DenseDataset(np.int8([[1, 2]]))
    with pytest.raises(qa.EmptyCorpus):
        qa.exact_topk(qa.DenseDataset(np.empty((0, 2), dtype=np.int8)), np.int8([1, 2]), 1,
                      qa.Metric.L2_SQUARED)
    with pytest.raises(ValueError):
        qa.exact_topk(corpus, np.int8([1, 2]), 0, qa.Metric.L2_SQUARED)
    with pytest.raises(qa.DimensionMismatch):
        qa.exact_topk(corpus, np.int8([1, 2, 3]), 1, qa.Metric.L2_SQUARED)
    with pytest.raises(qa.ElementKindMismatch):
        qa.exact_topk(corpus, np.float32([1, 2]), 1, qa.Metric.L2_SQUARED)
    with pytest.raises(qa.DimensionMismatch):
        qa.exact_topk(corpus, np.int8([[1, 2]]), 1, qa.Metric.L2_SQUARED)


def test_recall_at_k():
    exp = qa.GroundTruth(np.array([[0, 1, 2], [3, 4, 5]]))
    act = np.array([[2, 1, 9], [5, 4, 3]])
    r = qa.recall_at_k(exp, act, 3)
    assert r.per_query.tolist() == [2 / 3, 1.0] and math.isclose(r.mean, 5 / 6)
    assert r.hit_total == 5
    with pytest.raises(qa.LengthMismatch):
        qa.recall_at_k(exp, act[:1], 3)
    with pytest.raises(ValueError):
        qa.recall_at_k(exp, act, 4)


def test_acceptance_gate1_quantizer_order_range_reconstruction():
    # reference test_acceptance.py:77-113 (gate 1), through this package's
    # scalar quantize_value / dequantize_value
    rng = np.random.default_rng(11)
    checked = 0
    for _ in range(100):
        bits = int(rng.integers(1, 9))
        c = np.float32(rng.uniform(-5.0, 5.0))
        h = np.float32(rng.uniform(1e-3, 5.0))
        sb, se = np.float32(c - h), np.float32(c + h)
        k = np.float32((float(sb) + float(se)) / 2.0)
        p = qa.QuantizerParams(bits=bits, mode=qa.QuantMode.SIGMA_CLAMP, k=np.array([k]),
                               sb=np.array([sb]), se=np.array([se]))
        width = float(se) - float(sb)
        xs = np.sort(rng.uniform(float(c) - 3 * float(h), float(c) + 3 * float(h), size=(100, 2)),
                     axis=1)
        for x, y in xs:
            qx, qy = qa.quantize_value(float(x), 0, p), qa.quantize_value(float(y), 0, p)
            assert qx <= qy and p.lo_code <= qx <= p.hi_code and p.lo_code <= qy <= p.hi_code
            checked += 1
        for x in rng.uniform(float(sb), float(se), size=50):
            q = qa.quantize_value(float(x), 0, p)
            assert abs(qa.dequantize_value(q, 0, p) - float(x)) <= width / (1 << bits)
    assert checked == 10_000


def test_ground_truth_from_scan_matches_constructor():
    """GroundTruth.from_scan (the scan's own id matrix: distinct rows by
    construction) equals the checked constructor on valid input, freezes the
    array, and falls back to the checked constructor for anything else."""
    import numpy as np
    import pytest

    import paper_2110_08919_b200 as qa

    ids = np.array([[3, 1, 2], [0, 2, 5]], dtype=np.int32)
    a = qa.GroundTruth(ids=ids.copy())
    b = qa.GroundTruth.from_scan(ids.copy())
    assert a == b and b.nq == 2 and b.k == 3
    assert not b.ids.flags.writeable
    c = qa.GroundTruth.from_scan(ids.astype(np.int64))   # not int32: the checked path
    assert c == a and c.ids.dtype == np.int32
    with pytest.raises(ValueError):
        qa.GroundTruth.from_scan(np.array([[1, 1]], dtype=np.int64))  # duplicates still caught there
