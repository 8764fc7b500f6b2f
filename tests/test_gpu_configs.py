"""Parity at the BASELINE configs' full sizes (BASELINE.json configs 2, 3, 4),
where the scan plans differ from the small parity cases: doubling rounds and
the threshold estimate at n = 1M (cfg2), the small-batch plans with 64-query
tiles at n = 10M (cfg4), d = 256 inner product (cfg3 law), and the
device-generated cfg3 corpus that the cfg3 benchmark line uses.

Every check compares against the C oracle (oracle/qa_oracle.c, pinned to the
reference's _core.pyx:301-365 by tests/test_oracle.py) on a query subset the
oracle finishes in seconds, plus size-independent properties on all queries
(rows ascending by (score, id), ids unique and in range, scores equal to the
exact score of the reported row)."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_08919_b200 as qa  # noqa: E402
import synth  # noqa: E402
from paper_2110_08919_b200 import _lib  # noqa: E402


def _exact_scores(Xc, Qc, ids, metric):
    """The float64 score of every reported (query, row) pair, recomputed."""
    X = Xc[ids.reshape(-1)].astype(np.int64).reshape(ids.shape[0], ids.shape[1], -1)
    Q = Qc.astype(np.int64)[:, None, :]
    dots = (X * Q).sum(-1)
    if metric == 0:
        return -dots.astype(np.float64)
    if metric == 1:
        return ((X - Q) ** 2).sum(-1).astype(np.float64)
    xn = np.sqrt((X * X).sum(-1).astype(np.float64)).astype(np.float32).astype(np.float64)
    qn = np.sqrt((Q * Q).sum(-1).astype(np.float64)).astype(np.float32).astype(np.float64)
    return 1.0 - dots / (qn * xn)


def _check(oracle, Xc, Qc, sc, ids, k, metric, subset):
    sc = sc.cpu().numpy()
    ids = ids.cpu().numpy()
    n = Xc.shape[0]
    keff = min(k, n)
    assert sc.shape == ids.shape == (Qc.shape[0], keff)
    # properties on every query
    assert ((ids >= 0) & (ids < n)).all()
    assert all(len(np.unique(r)) == keff for r in ids)
    s0 = sc + 0.0
    order_ok = (s0[:, 1:] > s0[:, :-1]) | ((s0[:, 1:] == s0[:, :-1]) & (ids[:, 1:] > ids[:, :-1]))
    assert order_ok.all()
    np.testing.assert_array_equal(s0, _exact_scores(Xc, Qc, ids, metric) + 0.0)
    # bit-exact against the oracle on a subset
    m = min(subset, Qc.shape[0])
    osc, oids = oracle.scan_topk_i8(Xc, Qc[:m], k, metric, oracle.norms_i8(Xc),
                                    oracle.norms_i8(Qc[:m]))
    np.testing.assert_array_equal(ids[:m], oids)
    np.testing.assert_array_equal(sc[:m], osc)


def test_cfg2_full_size_l2(oracle):
    # BASELINE configs[2]: 1M x 128 SIFT-like, min/max int8, L2, a 1024-query batch
    X, Q = synth.generate(2, nq=1024)
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric.L2_SQUARED, "minmax")
    mn, mx = oracle.minmax(X)
    k_, sb, se = oracle.fit_range((mn + mx) / 2.0, (mx - mn) / 2.0)
    np.testing.assert_array_equal(index.params.sb, sb)
    np.testing.assert_array_equal(index.params.se, se)
    Xc = index.codes_in_input_order()
    rows = np.random.default_rng(2).choice(X.shape[0], 20_000, replace=False)
    np.testing.assert_array_equal(Xc[rows], oracle.encode(X[rows], k_, sb, se, 8))
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    np.testing.assert_array_equal(qc.to_host(), oracle.encode(Q, k_, sb, se, 8))
    sc, ids = index.search_codes(qc, 100)
    st = _lib.last_scan_stats()
    assert st["rounds"] == 2, st  # the estimate pass, one pass over every row
    _check(oracle, Xc, qc.to_host(), sc, ids, 100, 1, 48)


@pytest.fixture(scope="module")
def cfg4_data():
    X, Q = synth.generate(4, nq=64)  # 10M x 128 SIFT-like
    return X, Q


@pytest.mark.parametrize("metric", [1, 0])
def test_cfg4_full_size_small_batches(oracle, cfg4_data, metric):
    # BASELINE configs[4]: 10M x 128, batches 1 / 8 / 64, k 10 / 100, L2 and IP
    X, Q = cfg4_data
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric(metric), "minmax")
    Xc = index.codes_in_input_order()
    qc_all = index.encode_queries(torch.from_numpy(Q).cuda())
    Qc = qc_all.to_host()
    for B in (1, 8, 64):
        qc = qc_all.slice_rows(0, B)
        for k in (10, 100):
            sc, ids = index.search_codes(qc, k)
            _check(oracle, Xc, Qc[:B], sc, ids, k, metric, 4)
    del index
    torch.cuda.empty_cache()


def test_cfg3_law_inner_product_d256(oracle):
    # the config-3 law (Gaussian mixture, 1024 clusters, d = 256) at 2M rows
    X, Q = synth.generate(3, n=2_000_000, nq=300)
    index = qa.Int8Index.build(torch.from_numpy(X).cuda(), qa.Metric.INNER_PRODUCT, "minmax")
    Xc = index.codes_in_input_order()
    p = index.params
    rows = np.random.default_rng(3).choice(X.shape[0], 20_000, replace=False)
    np.testing.assert_array_equal(Xc[rows], oracle.encode(X[rows], p.k, p.sb, p.se, 8))
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    sc, ids = index.search_codes(qc, 100)
    _check(oracle, Xc, qc.to_host(), sc, ids, 100, 0, 24)


def test_cfg3_device_generated_corpus_encode(oracle):
    # the cfg3 benchmark generates its 61 GB fp32 source on the device and
    # encodes it chunk by chunk (tools/bench_configs.py): re-encode a row
    # sample of those device rows with the oracle, with the streamed window
    from paper_2110_08919_b200 import device as dev
    from paper_2110_08919_b200.quantizer import RangeStats, fit_minmax
    from tools.bench_configs import mixture_on_device

    n, d = 1_000_000, 256
    gen = mixture_on_device(n, 0, d, 1024, 3, chunk=1 << 18)
    mn = torch.full((d,), float("inf"), device="cuda")
    mx = torch.full((d,), float("-inf"), device="cuda")
    for _, _, x in gen(n):
        a, b = dev.minmax(x)
        torch.minimum(mn, a, out=mn)
        torch.maximum(mx, b, out=mx)
    p = fit_minmax(RangeStats(mn.cpu().numpy().astype(np.float64),
                              mx.cpu().numpy().astype(np.float64), n)).params
    kk, sb, se = (torch.from_numpy(np.array(v, dtype=np.float32)).cuda() for v in (p.k, p.sb, p.se))
    gen = mixture_on_device(n, 0, d, 1024, 3, chunk=1 << 18)
    for i, (lo, hi, x) in enumerate(gen(n)):
        if i % 2:
            continue
        codes = dev.encode(x, kk, sb, se, 8)
        sel = torch.arange(0, hi - lo, 97, device="cuda")
        xs = x[sel].cpu().numpy()
        np.testing.assert_array_equal(codes.to_host()[sel.cpu().numpy()],
                                      oracle.encode(xs, p.k, p.sb, p.se, 8))
