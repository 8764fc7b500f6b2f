"""Kernel seam: the B200 implementation of the reference's
``quantann._backend`` surface (reference _backend.py:14-46).

The reference picks ``_core`` (Cython, one CPU core) or ``_kernels_py``
(numpy) at import; this package has exactly one backend, ``"cuda"``: the
sm_100a kernels of libqa_b200.so.  There is no CPU fallback -- importing
this module fails if the library is missing.

Surface (host numpy in, host numpy out, reference semantics):

* ``scan_topk(data, queries, k, metric, data_norms=None, query_norms=None)``
  -> (float64 [nq, keff], int32 [nq, keff]), _core.pyx:333-365;
* ``norms(mat)`` -> float32 [n], _core.pyx:137-157;
* ``dot(a, b)`` / ``l2sq(a, b)`` -- single pairs, _core.pyx:99-134 (through
  the same kernels with n = nq = 1; the batch paths are the hot ones);
* ``quantize(values, k, sb, se, bits)`` -> int8 [n, d] -- the encode hook the
  reference lacks (its quantizer.py:291-300 calls numpy directly).

float32 inputs take the float64-exact path (``qa_scan_topk_f32`` /
``qa_norms_f32``, bit-exact with ``_scan_f32`` and the float32 ``norms``
branch, _core.pyx:150-153, 270-298): the ground truth for recall.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device as _dev
from ._lib import lib  # noqa: F401  (fails loudly when the library is missing)

BACKEND = "cuda"


def _to_dev(arr: np.ndarray, dev) -> torch.Tensor:
    """Upload a (possibly read-only) host array without writing to it."""
    arr = np.ascontiguousarray(arr)
    return torch.from_numpy(arr if arr.flags.writeable else arr.copy()).to(dev)


def _check_pair(data, queries):
    if data.ndim != 2 or queries.ndim != 2:
        raise ValueError("data and queries must be 2-D")
    if data.dtype != queries.dtype:
        raise ValueError("dtype mismatch between data and queries")
    if data.shape[1] != queries.shape[1]:
        raise ValueError("dimension mismatch between data and queries")


def scan_topk(data, queries, k, metric, data_norms=None, query_norms=None):
    """Exhaustive top-k per query; rows ascending by (score, id)."""
    _check_pair(data, queries)
    if k < 0:
        raise ValueError("k must be >= 0")
    n, nq = data.shape[0], queries.shape[0]
    keff = min(int(k), n)
    if n == 0 or nq == 0 or keff == 0:
        return (np.empty((nq, keff), dtype=np.float64), np.empty((nq, keff), dtype=np.int32))
    if int(metric) == 2 and (data_norms is None or query_norms is None
                             or data_norms.shape[0] != n or query_norms.shape[0] != nq):
        raise ValueError("angular metric needs data and query norms")
    dev = _dev.default_device()
    if data.dtype == np.float32:
        dn = qn = None
        if int(metric) == 2:
            dn = torch.from_numpy(np.ascontiguousarray(data_norms, dtype=np.float32)).to(dev)
            qn = torch.from_numpy(np.ascontiguousarray(query_norms, dtype=np.float32)).to(dev)
        scores, ids = _dev.scan_topk_f32(_to_dev(data, dev), _to_dev(queries, dev), int(k),
                                         int(metric), dn, qn)
        return scores.cpu().numpy(), ids.cpu().numpy()
    if data.dtype != np.int8:
        raise ValueError("dtype must be float32 or int8")
    db = _dev.DeviceCodes.from_host(data, dev)
    qs = _dev.DeviceCodes.from_host(queries, dev)
    dn = qn = None
    if int(metric) == 2:
        dn = torch.from_numpy(np.ascontiguousarray(data_norms, dtype=np.float32)).to(dev)
        qn = torch.from_numpy(np.ascontiguousarray(query_norms, dtype=np.float32)).to(dev)
    scores, ids = _dev.scan_topk(db, qs, int(k), int(metric), dn, qn)
    return scores.cpu().numpy(), ids.cpu().numpy()


def _pair(a, b, metric: int) -> float:
    """One pair through the exhaustive-scan kernels (n = nq = 1, k = 1)."""
    if a.shape[0] != b.shape[0]:
        raise ValueError("length mismatch")
    if a.dtype != b.dtype:
        raise ValueError("dtype mismatch")
    if a.shape[0] == 0:
        return 0.0
    x = np.ascontiguousarray(b).reshape(1, -1)
    q = np.ascontiguousarray(a).reshape(1, -1)
    scores, _ = scan_topk(x, q, 1, metric)
    return float(scores[0, 0])


def dot(a, b):
    """Inner product of two 1-D vectors of equal dtype (_core.pyx:99-115):
    float32 -> float64 sequential sum, int8 -> exact int32 sum, as float."""
    return -_pair(a, b, 0) + 0.0   # score = -dot; + 0.0 turns -0.0 into 0.0


def l2sq(a, b):
    """Squared Euclidean distance of two 1-D vectors (_core.pyx:118-134)."""
    return _pair(a, b, 1)


def norms(mat):
    """float32(sqrt(int64 sum c^2)) of every int8 row."""
    if mat.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    n, d = mat.shape
    if n == 0 or d == 0:
        return np.zeros(n, dtype=np.float32)
    if mat.dtype == np.float32:
        return _dev.norms_f32(_to_dev(mat, _dev.default_device())).cpu().numpy()
    if mat.dtype != np.int8:
        raise ValueError("dtype must be float32 or int8")
    dc = _dev.DeviceCodes.from_host(mat)
    return dc.norm.cpu().numpy()


def quantize(values, k, sb, se, bits):
    """Eq. 1 encode of a float32 [n, d] host matrix on the GPU."""
    from .quantizer import QuantizerParams, QuantMode, quantize_array

    p = QuantizerParams(bits=int(bits), mode=QuantMode.ABS_MAX, k=np.asarray(k, np.float32),
                        sb=np.asarray(sb, np.float32), se=np.asarray(se, np.float32))
    return quantize_array(np.asarray(values), p)


def get_backend(name=None):
    """Return the kernel module: None or "cuda" -> this module.  The
    reference's "compiled"/"pure" CPU backends do not exist here."""
    import sys

    if name is None or name == "cuda":
        return sys.modules[__name__]
    raise ValueError(f"unknown backend {name!r}")
