"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs only in the dev container (needs /root/reference): imports the
reference package from /root/reference/pkg/src (its numpy quantizer) and
its compiled kernel module quantann._core built from the reference sources
by ``make -C oracle ref``.  The outputs are small .npz files committed next
to this script; the tests read them on any machine.

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import importlib.util
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")

sys.path.insert(0, str(ROOT))


def load_reference():
    """The reference package (pure-numpy backend from the source tree) and
    its compiled _core from oracle/_ref."""
    sys.path.insert(0, str(REF_SRC))
    import quantann  # noqa: E402  (reference, /root/reference/pkg/src)

    spec = importlib.util.spec_from_file_location(
        "quantann._core", next((ROOT / "oracle/_ref/quantann").glob("_core*.so")))
    core = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(core)
    assert core.BACKEND == "compiled"
    return quantann, core


def encode_cases(qa):
    from quantann.quantizer import (QuantizerParams, QuantMode, estimate_stats, fit,
                                    quantize_dataset)
    from quantann import DenseDataset

    cases = {}
    # hand window of test_quantizer.py:_fit_window(-0.1, 0.1)
    st = estimate_stats(DenseDataset(np.asarray([[-0.1], [0.1]], dtype=np.float32)))
    p = fit(st, 8, QuantMode.SIGMA_CLAMP).params
    x = np.asarray([[0.0], [0.05], [-0.1], [0.1], [0.5], [-0.2], [np.nan], [np.inf], [-np.inf]],
                   dtype=np.float32)
    cases["hand"] = (x, p, quantize_dataset(DenseDataset(x), p).data)
    rng = np.random.default_rng(123)
    for bits in range(1, 9):
        for mode in (QuantMode.SIGMA_CLAMP, QuantMode.ABS_MAX, QuantMode.UNIFORM_SIGMA_CLAMP):
            d = int(rng.integers(1, 70))
            n = int(rng.integers(8, 300))
            data = (rng.normal(0.0, rng.uniform(0.01, 3.0), size=(n, d))
                    + rng.normal(0.0, 2.0, size=d)).astype(np.float32)
            p = fit(estimate_stats(DenseDataset(data)), bits, mode).params
            probe = data.copy()
            probe[0] = p.sb
            probe[1] = p.se
            probe[2] = p.k
            probe[3] = np.nextafter(p.sb, np.float32(-np.inf))
            probe[4] = np.nextafter(p.se, np.float32(np.inf))
            probe[5, : min(d, 4)] = [np.nan, np.inf, -np.inf, 1e-40][: min(d, 4)]
            probe[6] = np.float32(1e-42)  # denormal
            codes = quantize_dataset(DenseDataset(probe), p).data
            cases[f"b{bits}_m{int(mode)}"] = (probe, p, codes)
    arrays = {}
    for name, (x, p, c) in cases.items():
        arrays[f"{name}__x"] = x
        arrays[f"{name}__k"] = p.k
        arrays[f"{name}__sb"] = p.sb
        arrays[f"{name}__se"] = p.se
        arrays[f"{name}__bits"] = np.int64(p.bits)
        arrays[f"{name}__codes"] = c
    np.savez_compressed(OUT / "encode_cases.npz", **arrays)
    return len(cases)


def scan_cases(core):
    arrays = {}
    rng = np.random.default_rng(7)
    count = 0
    for i in range(36):
        metric = i % 3
        n = int(rng.integers(1, 700))
        d = int(rng.integers(1, 48))
        nq = int(rng.integers(1, 6))
        lo, hi = (-127, 128) if i % 4 else (-3, 4)  # every 4th case: heavy ties
        X = rng.integers(lo, hi, size=(n, d)).astype(np.int8)
        Q = rng.integers(lo, hi, size=(nq, d)).astype(np.int8)
        if metric == 2:
            X[~X.any(axis=1), 0] = 1
            Q[~Q.any(axis=1), 0] = 1
        k = int(rng.choice([1, 10, 100, n, n + 1]))
        xn, qn = core.norms(X), core.norms(Q)
        sc, ids = core.scan_topk(X, Q, k, metric, xn, qn)
        pre = f"c{i}"
        arrays.update({f"{pre}__X": X, f"{pre}__Q": Q, f"{pre}__k": np.int64(k),
                       f"{pre}__metric": np.int64(metric), f"{pre}__xn": xn,
                       f"{pre}__qn": qn, f"{pre}__scores": sc, f"{pre}__ids": ids})
        count += 1
    np.savez_compressed(OUT / "scan_cases.npz", **arrays)
    return count


def scan_f32_cases(core):
    """float32 exhaustive search (_scan_f32) known answers: mixed scales,
    integer-valued rows (exact score ties), duplicated rows, signed zeros,
    d not a multiple of the GPU's 16-dim stage."""
    arrays = {}
    rng = np.random.default_rng(11)
    count = 0
    for i in range(30):
        metric = i % 3
        n = int(rng.integers(1, 500))
        d = int(rng.integers(1, 150)) if i % 5 else int(rng.integers(1, 8))
        nq = int(rng.integers(1, 5))
        kind = i % 4
        if kind == 0:
            X = rng.normal(size=(n, d)) * rng.uniform(0.01, 100.0, size=d)
            Q = rng.normal(size=(nq, d)) * rng.uniform(0.01, 100.0, size=d)
        elif kind == 1:   # integer-valued: many exactly tied scores
            X = rng.integers(-3, 4, size=(n, d)).astype(np.float64)
            Q = rng.integers(-3, 4, size=(nq, d)).astype(np.float64)
        elif kind == 2:   # sift-like non-negative
            X = np.clip(np.round(np.abs(rng.normal(0, 40, size=(n, d)))), 0, 255)
            Q = np.clip(np.round(np.abs(rng.normal(0, 40, size=(nq, d)))), 0, 255)
        else:             # duplicated rows and signed zeros
            base = rng.normal(size=(max(1, n // 3), d))
            X = base[rng.integers(0, base.shape[0], size=n)]
            X[rng.random((n, d)) < 0.2] = -0.0
            Q = rng.normal(size=(nq, d))
        X = X.astype(np.float32)
        Q = Q.astype(np.float32)
        if metric == 2:
            X[~X.any(axis=1), 0] = 1.0
            Q[~Q.any(axis=1), 0] = 1.0
        k = int(rng.choice([1, 10, 100, n, n + 1]))
        xn, qn = core.norms(X), core.norms(Q)
        sc, ids = core.scan_topk(X, Q, k, metric, xn, qn)
        pre = f"f{i}"
        arrays.update({f"{pre}__X": X, f"{pre}__Q": Q, f"{pre}__k": np.int64(k),
                       f"{pre}__metric": np.int64(metric), f"{pre}__xn": xn,
                       f"{pre}__qn": qn, f"{pre}__scores": sc, f"{pre}__ids": ids})
        count += 1
    np.savez_compressed(OUT / "scan_f32_cases.npz", **arrays)
    return count


def vecs_cases():
    """Framing known answers for the vector-file loaders (dataset.py:160-275):
    byte strings -> the reference loader's array or its error class/message
    (the path in messages is written as {path})."""
    import os
    import struct
    import tempfile

    from quantann import dataset as rd

    def rec(d, payload):
        return struct.pack("<i", d) + payload

    f4 = lambda vals: np.asarray(vals, "<f4").tobytes()
    cases = {
        "f_ok": ("fvecs", rec(3, f4([1, 2, 3])) + rec(3, f4([-0.0, np.inf, 1e-40]))),
        "f_empty": ("fvecs", b""),
        "f_short_header": ("fvecs", b"\x03\x00"),
        "f_zero_d": ("fvecs", rec(0, b"")),
        "f_neg_d": ("fvecs", rec(-2, f4([1, 2]))),
        "f_mixed": ("fvecs", rec(2, f4([1, 2])) + rec(3, f4([1, 2, 3]))),
        "f_mixed_whole": ("fvecs", rec(2, f4([1, 2])) + rec(2, f4([1, 2])) + rec(1, f4([5]))
                          + struct.pack("<i", 2)),
        "f_trunc_payload": ("fvecs", rec(2, f4([1, 2])) + rec(2, f4([1]))),
        "f_trunc_header": ("fvecs", rec(2, f4([1, 2])) + b"\x02\x00"),
        "f_later_neg": ("fvecs", rec(1, f4([1])) + rec(1, f4([2])) + rec(-1, f4([3]))),
        "f_later_zero_walk": ("fvecs", rec(1, f4([1])) + rec(0, b"") + b"\x00"),
        "i_ok": ("ivecs", rec(2, np.asarray([5, 7], "<i4").tobytes())
                 + rec(2, np.asarray([0, 3], "<i4").tobytes())),
        "i_dup": ("ivecs", rec(2, np.asarray([5, 5], "<i4").tobytes())),
        "b8_ok": ("i8vecs", rec(4, bytes([0, 127, 128, 255])) + rec(4, bytes([1, 2, 3, 4]))),
        "b8_trunc": ("i8vecs", rec(4, bytes([0, 1, 2, 3])) + rec(4, bytes([1, 2]))),
        "bv_ok": ("bvecs", rec(3, bytes([0, 128, 255])) + rec(3, bytes([127, 129, 1]))),
        "bv_mixed": ("bvecs", rec(3, bytes([0, 128, 255])) + rec(2, bytes([1, 2])) + b"\x00"),
    }
    loaders = {"fvecs": rd.load_fvecs, "ivecs": rd.load_ivecs, "i8vecs": rd.load_i8vecs,
               "bvecs": rd.load_bvecs}
    arrays = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, (kind, blob) in cases.items():
            path = os.path.join(tmp, f"{name}.{kind}")
            with open(path, "wb") as fh:
                fh.write(blob)
            arrays[f"{name}__kind"] = np.array(kind)
            arrays[f"{name}__blob"] = np.frombuffer(blob, np.uint8)
            try:
                out = loaders[kind](path)
                arrays[f"{name}__out"] = out.ids if kind == "ivecs" else out.data
            except Exception as exc:  # noqa: BLE001 - record the reference's outcome
                arrays[f"{name}__error"] = np.array(type(exc).__name__)
                arrays[f"{name}__message"] = np.array(str(exc).replace(path, "{path}"))
    np.savez_compressed(OUT / "vecs_cases.npz", **arrays)
    return len(cases)


def stats_inputs():
    """Seeded inputs of the estimate_stats known answers (regenerated by the
    tests from the same seeds; only the reference's outputs are stored)."""
    def gen(seed, n, d, kind):
        rng = np.random.default_rng(seed)
        if kind == "normal":
            x = rng.normal(size=(n, d)) * rng.uniform(0.01, 50, size=d) + rng.normal(0, 5, size=d)
        elif kind == "ints":   # heavy ties: order statistics on repeated values
            x = rng.integers(-3, 4, size=(n, d)).astype(np.float64)
        elif kind == "sift":
            x = np.clip(np.round(np.abs(rng.normal(0, 40, size=(n, d)))), 0, 255)
            x[rng.random((n, d)) < 0.1] = 0
        elif kind == "const":  # zero-width dimensions
            x = rng.normal(size=(n, d))
            x[:, ::3] = 1.25
        elif kind == "nan":
            x = rng.normal(size=(n, d))
            x[rng.integers(0, n), 0] = np.nan
        elif kind == "tiny":   # denormals and signed zeros
            x = rng.normal(size=(n, d)) * 1e-39
            x[::5] = -0.0
        else:
            raise ValueError(kind)
        return x.astype(np.float32)

    specs = [("s_normal_small", 1, 2, 1, "normal"), ("s_normal_7", 2, 7, 3, "normal"),
             ("s_normal_9", 3, 9, 5, "normal"), ("s_normal_129", 4, 129, 70, "normal"),
             ("s_normal_5000", 5, 5000, 70, "normal"), ("s_ints", 6, 3001, 65, "ints"),
             ("s_sift_100k", 7, 100_000, 128, "sift"), ("s_const", 8, 1000, 10, "const"),
             ("s_nan", 9, 500, 4, "nan"), ("s_tiny", 10, 777, 33, "tiny"),
             ("s_wide", 11, 300, 200, "normal"), ("s_glove", 12, 50_000, 100, "normal")]
    return [(name, gen(seed, n, d, kind)) for name, seed, n, d, kind in specs], specs


def stats_cases():
    from quantann import DenseDataset
    from quantann.quantizer import QuantMode, estimate_stats, fit

    arrays = {}
    cases, specs = stats_inputs()
    for (name, x), spec in zip(cases, specs):
        st = estimate_stats(DenseDataset(x))
        arrays[f"{name}__spec"] = np.array(spec[1:4], dtype=np.int64)
        arrays[f"{name}__kind"] = np.array(spec[4])
        for f in ("mu", "sigma", "min", "max", "trimmed_absmax"):
            arrays[f"{name}__{f}"] = getattr(st, f)
        arrays[f"{name}__pooled"] = np.array([st.pooled_mu, st.pooled_sigma])
        for mode in (QuantMode.SIGMA_CLAMP, QuantMode.ABS_MAX, QuantMode.UNIFORM_SIGMA_CLAMP):
            try:
                p = fit(st, 8, mode).params
                arrays[f"{name}__fit{int(mode)}"] = np.stack([p.k, p.sb, p.se])
            except Exception:  # noqa: BLE001 - e.g. NaN windows are rejected
                pass
    np.savez_compressed(OUT / "stats_cases.npz", **arrays)
    return len(cases)


def gate4_case():
    """The reference's acceptance gate 4 pipeline (test_acceptance.py:176-193,
    synthetic corpus): float32 ground truth, estimate_stats -> fit(ABS_MAX)
    -> quantize_dataset -> int8 ground truth, recall@100 -- run by the
    reference (compiled backend) and stored for an end-to-end GPU check."""
    import importlib
    sys.path.insert(0, str(REF_SRC))
    import quantann
    from quantann import (DenseDataset, Metric, QuantMode, batch_ground_truth, estimate_stats,
                          fit, generate_synthetic, quantize_dataset, recall_at_k)
    # the compiled kernels from oracle/_ref stand in for the package's own build
    core = load_reference()[1]
    import quantann._backend as be
    be.scan_topk, be.norms, be.BACKEND = core.scan_topk, core.norms, core.BACKEND
    import quantann.exact as ex
    importlib.reload(ex)
    corpus = generate_synthetic(50_000, 64, 0.0, 0.05, 2)
    queries = generate_synthetic(100, 64, 0.0, 0.05, 1002)
    gt = ex.batch_ground_truth(corpus, queries, 100, Metric.INNER_PRODUCT)
    params = fit(estimate_stats(corpus), 8, QuantMode.ABS_MAX).params
    ci8 = quantize_dataset(corpus, params)
    qi8 = quantize_dataset(queries, params)
    approx = ex.batch_ground_truth(ci8, qi8, 100, Metric.INNER_PRODUCT)
    rec = recall_at_k(gt, approx, 100).mean
    np.savez_compressed(OUT / "gate4.npz", gt=gt.ids, approx=approx.ids, recall=np.float64(rec),
                        k=params.k, sb=params.sb, se=params.se)
    return rec


def cfg_minis(qa, core):
    """BASELINE cfg0 (L2, min/max) and cfg1 (angular, symmetric) at reduced
    size through the reference pipeline: constructed stats -> fit(ABS_MAX)
    -> quantize_dataset -> compiled scan_topk."""
    import synth
    from quantann import DenseDataset
    from quantann.quantizer import DimensionStats, QuantMode, fit, quantize_dataset

    arrays = {}
    for cfg, (n, nq) in ((0, (6000, 24)), (1, (6000, 24)), (3, (6000, 24))):
        X, Q = synth.generate(cfg, n=n, nq=nq)
        mn = X.astype(np.float64).min(axis=0)
        mx = X.astype(np.float64).max(axis=0)
        if cfg == 1:
            center = np.zeros_like(mn)
            half = np.maximum(np.abs(mn), np.abs(mx))
        else:
            center = (mn + mx) / 2.0
            half = (mx - mn) / 2.0
        z = np.zeros_like(center)
        stats = DimensionStats(mu=center, sigma=z, min=center - half, max=center + half,
                               trimmed_absmax=half, pooled_mu=0.0, pooled_sigma=0.0, count=n)
        p = fit(stats, 8, QuantMode.ABS_MAX).params
        Xc = quantize_dataset(DenseDataset(X), p).data
        Qc = quantize_dataset(DenseDataset(Q), p).data
        metric = synth.CONFIGS[cfg]["metric"]
        xn, qn = core.norms(Xc), core.norms(Qc)
        sc, ids = core.scan_topk(Xc, Qc, 100, metric, xn, qn)
        f_xn, f_qn = core.norms(X), core.norms(Q)
        _, gt32 = core.scan_topk(X, Q, 100, metric, f_xn, f_qn)
        pre = f"cfg{cfg}"
        arrays.update({f"{pre}__k": p.k, f"{pre}__sb": p.sb, f"{pre}__se": p.se,
                       f"{pre}__mn": mn, f"{pre}__mx": mx,
                       f"{pre}__codes_sha": np.frombuffer(
                           __import__("hashlib").sha256(Xc.tobytes()).digest(), np.uint8),
                       f"{pre}__qcodes": Qc, f"{pre}__scores": sc, f"{pre}__ids": ids,
                       f"{pre}__gt32": gt32})
    np.savez_compressed(OUT / "cfg_minis.npz", **arrays)


def main():
    qa, core = load_reference()
    if len(sys.argv) > 1:   # regenerate only the named fixtures, e.g. scan_f32
        for name in sys.argv[1:]:
            fn = {"encode": lambda: encode_cases(qa), "scan": lambda: scan_cases(core),
                  "scan_f32": lambda: scan_f32_cases(core), "vecs": vecs_cases, "stats": stats_cases, "gate4": gate4_case, "cfg": lambda: cfg_minis(qa, core)}[name]
            print(name, fn())
        return
    nf = scan_f32_cases(core)
    vecs_cases()
    stats_cases()
    gate4_case()
    ne = encode_cases(qa)
    ns = scan_cases(core)
    cfg_minis(qa, core)
    print(f"wrote {ne} encode cases, {ns} scan cases, {nf} float32 scan cases, cfg minis to {OUT}")


if __name__ == "__main__":
    main()
