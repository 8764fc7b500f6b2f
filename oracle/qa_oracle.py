"""TEST INFRASTRUCTURE ONLY: CPU restatement of the reference hot path.

Two independent checkers:

* ``libqa_oracle.so`` (qa_oracle.c): plain-C restatement of
  quantizer.py:291-300 (encode), _core.pyx:137-157 (norms) and
  _core.pyx:301-365 (int8 scan_topk), built by ``make -C oracle``;
* ``ref_core()``: the reference's OWN compiled kernel module
  (``quantann._core`` from /root/reference/pkg/src/quantann/_core.pyx),
  built by ``make -C oracle ref`` into oracle/_ref/ -- the pin for the
  restatement and the CPU baseline timed by bench.py.

Plus small numpy restatements (``encode_np``, ``fit_range``) used to check
the C restatement against the reference's numpy formula.
"""

from __future__ import annotations

import ctypes
import importlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = HERE / "libqa_oracle.so"
        if not path.exists():
            raise ImportError(f"{path} missing: run `make -C oracle`")
        L = ctypes.CDLL(str(path))
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.qo_encode_i8.argtypes = [vp, i64, i64, vp, vp, vp, ctypes.c_int, vp]
        L.qo_encode_i8.restype = None
        L.qo_norms_i8.argtypes = [vp, i64, i64, vp]
        L.qo_norms_i8.restype = None
        L.qo_minmax_f32.argtypes = [vp, i64, i64, vp, vp]
        L.qo_minmax_f32.restype = None
        L.qo_scan_topk_i8.argtypes = [vp, i64, i64, vp, i64, i64, ctypes.c_int, vp, vp, vp, vp]
        L.qo_scan_topk_i8.restype = i64
        L.qo_pair_scores_i8.argtypes = [vp, i64, i64, vp, i64, vp, i64, ctypes.c_int, vp, vp, vp]
        L.qo_pair_scores_i8.restype = None
        L.qo_norms_f32.argtypes = [vp, i64, i64, vp]
        L.qo_norms_f32.restype = None
        L.qo_scan_topk_f32.argtypes = [vp, i64, i64, vp, i64, i64, ctypes.c_int, vp, vp, vp, vp]
        L.qo_scan_topk_f32.restype = i64
        _LIB = L
    return _LIB


def _ptr(a):
    return None if a is None else a.ctypes.data


def encode(x: np.ndarray, k, sb, se, bits: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    k, sb, se = (np.ascontiguousarray(a, dtype=np.float32) for a in (k, sb, se))
    out = np.empty(x.shape, dtype=np.int8)
    lib().qo_encode_i8(_ptr(x), x.shape[0], x.shape[1], _ptr(k), _ptr(sb), _ptr(se), int(bits),
                       _ptr(out))
    return out


def norms_i8(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.int8)
    out = np.empty(x.shape[0], dtype=np.float32)
    lib().qo_norms_i8(_ptr(x), x.shape[0], x.shape[1], _ptr(out))
    return out


def sqnorms_i8(x: np.ndarray) -> np.ndarray:
    w = x.astype(np.int64)
    return (w * w).sum(axis=1)


def minmax(x: np.ndarray):
    x = np.ascontiguousarray(x, dtype=np.float32)
    mn = np.empty(x.shape[1], dtype=np.float64)
    mx = np.empty(x.shape[1], dtype=np.float64)
    lib().qo_minmax_f32(_ptr(x), x.shape[0], x.shape[1], _ptr(mn), _ptr(mx))
    return mn, mx


def scan_topk_i8(X, Q, k, metric, xn=None, qn=None):
    X = np.ascontiguousarray(X, dtype=np.int8)
    Q = np.ascontiguousarray(Q, dtype=np.int8)
    n, d = X.shape
    nq = Q.shape[0]
    keff = min(int(k), n)
    od = np.empty((nq, keff), dtype=np.float64)
    oi = np.empty((nq, keff), dtype=np.int32)
    if metric == 2:
        xn = np.ascontiguousarray(xn, dtype=np.float32)
        qn = np.ascontiguousarray(qn, dtype=np.float32)
    lib().qo_scan_topk_i8(_ptr(X), n, d, _ptr(Q), nq, int(k), int(metric), _ptr(xn), _ptr(qn),
                          _ptr(od), _ptr(oi))
    return od, oi


def pair_scores_i8(X, Q, cand, metric, xn=None, qn=None) -> np.ndarray:
    """float64 [nq, m] scores of the listed (query, row id) pairs, the
    reference's _pair_i per pair (_core.pyx:88-96, HnswCore._dq 483-494)."""
    X = np.ascontiguousarray(X, dtype=np.int8)
    Q = np.ascontiguousarray(Q, dtype=np.int8)
    cand = np.ascontiguousarray(cand, dtype=np.int32)
    nq, m = cand.shape
    out = np.empty((nq, m), dtype=np.float64)
    if metric == 2:
        xn = np.ascontiguousarray(xn, dtype=np.float32)
        qn = np.ascontiguousarray(qn, dtype=np.float32)
    lib().qo_pair_scores_i8(_ptr(X), X.shape[0], X.shape[1], _ptr(Q), nq, _ptr(cand), m,
                            int(metric), _ptr(xn) if metric == 2 else None,
                            _ptr(qn) if metric == 2 else None, _ptr(out))
    return out


def norms_f32(x: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape[0], dtype=np.float32)
    lib().qo_norms_f32(_ptr(x), x.shape[0], x.shape[1], _ptr(out))
    return out


def scan_topk_f32(X, Q, k, metric, xn=None, qn=None):
    """_scan_f32 restated (float64 sequential sums, (score, id) heap)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    Q = np.ascontiguousarray(Q, dtype=np.float32)
    n, d = X.shape
    nq = Q.shape[0]
    keff = min(int(k), n)
    od = np.empty((nq, keff), dtype=np.float64)
    oi = np.empty((nq, keff), dtype=np.int32)
    if metric == 2:
        xn = np.ascontiguousarray(xn, dtype=np.float32)
        qn = np.ascontiguousarray(qn, dtype=np.float32)
    lib().qo_scan_topk_f32(_ptr(X), n, d, _ptr(Q), nq, int(k), int(metric), _ptr(xn), _ptr(qn),
                           _ptr(od), _ptr(oi))
    return od, oi


def encode_np(values: np.ndarray, k, sb, se, bits: int) -> np.ndarray:
    """numpy restatement of quantizer.py:291-300 (same operation order)."""
    lo, hi = -(1 << (bits - 1)), (1 << (bits - 1)) - 1
    ratio = (values - k) / (se - sb)
    q = np.floor((np.float32(2.0 ** bits) * ratio).astype(np.float64))
    q = np.clip(q, lo, hi)
    x = values.astype(np.float64)
    above = x > se.astype(np.float64)
    inside = (x >= sb.astype(np.float64)) & (x <= se.astype(np.float64))
    return np.where(inside, q, np.where(above, hi, lo)).astype(np.int8)


def fit_range(center: np.ndarray, half: np.ndarray):
    """Restatement of the ABS_MAX branch of quantizer.py:225-267 for given
    float64 centre/half-width: returns float32 (k, sb, se)."""
    k = center.astype(np.float64).copy()
    sb = k - half
    se = k + half
    deg = se - sb < 1e-12
    sb[deg] = k[deg] - 1e-6
    se[deg] = k[deg] + 1e-6
    k32, sb32, se32 = k.astype(np.float32), sb.astype(np.float32), se.astype(np.float32)
    col = ~(sb32 < se32)
    sb32[col] = np.nextafter(k32[col], np.float32(-np.inf))
    se32[col] = np.nextafter(k32[col], np.float32(np.inf))
    return k32, sb32, se32


def ref_core():
    """The reference's compiled quantann._core (oracle/_ref), or None."""
    ref = HERE / "_ref"
    if not (ref / "quantann").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        return importlib.import_module("quantann._core")
    except ImportError:
        return None
