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
  reference lacks (its quantizer.py:291-300 calls numpy directly);
* ``pair_scores(data, queries, cand, metric, ...)`` -> float64 [nq, m] -- the
  batched form of ``HnswCore._dq`` (_core.pyx:483-494): distances from each
  query to its listed candidate rows, for a host-side graph traversal.

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
    return _dev.host_to_device(arr, dev)


def _check_pair(data, queries):
    if data.ndim != 2 or queries.ndim != 2:
        raise ValueError("data and queries must be 2-D")
    if data.dtype != queries.dtype:
        raise ValueError("dtype mismatch between data and queries")
    if data.shape[1] != queries.shape[1]:
        raise ValueError("dimension mismatch between data and queries")


# ---- device-resident corpora ---------------------------------------------
#
# The reference's callers hand the same frozen corpus array to every call
# (DenseDataset freezes its array, reference dataset.py:82; exact.py:105-117
# passes ``corpus.data`` each time).  A read-only int8 array is therefore
# uploaded once and kept resident in the form the scan wants, keyed on the
# array object (weakly) plus its address, shape, strides and a strided
# content fingerprint; writable arrays are never cached.  Forms:
#
#   "rows"  caller order (query batches; norms)
#   "bands" index layout of L2 / angular: interleaved norm blocks
#   "ip"    index layout of inner product: a fixed pseudo-random row order
#
# The index layouts (qa_layout.cu) are what the scan's threshold estimate and
# per-unit bounds assume; ids still report caller rows (DeviceCodes.ids).

_RESIDENT: dict = {}
_FORM_OF_METRIC = {0: "ip", 1: "bands", 2: "bands"}


def _fingerprint(arr: np.ndarray) -> int:
    flat = arr.reshape(-1).view(np.uint8)
    step = max(1, flat.shape[0] // 4096)
    return hash(flat[::step].tobytes())


def _make_form(base: _dev.DeviceCodes, form: str) -> _dev.DeviceCodes:
    if form == "rows":
        return base
    if form == "ip":
        return base.shuffled()
    return base.sorted_by_norm(stratify=False)


def _resident(arr: np.ndarray, dev, form: str = "rows") -> _dev.DeviceCodes:
    if arr.flags.writeable:
        return _make_form(_dev.DeviceCodes.from_host(arr, dev), form)
    key = (arr.__array_interface__["data"][0], arr.shape, arr.strides, str(dev),
           _fingerprint(arr))
    ent = _RESIDENT.get(id(arr))
    if ent is None or ent[0]() is not arr or ent[1] != key:
        import weakref

        ident = id(arr)
        ent = (weakref.ref(arr, lambda _r, i=ident: _RESIDENT.pop(i, None)), key, {})
        _RESIDENT[ident] = ent
    forms = ent[2]
    dc = forms.get(form)
    if dc is None:
        base = forms.get("rows") or _dev.DeviceCodes.from_host(arr, dev)
        dc = _make_form(base, form)
        forms[form] = dc
    return dc


# pinned host staging for results (reused between calls; the caller gets
# fresh arrays copied out of it)
_PINNED: dict = {}


def _pinned(name: str, shape, dtype) -> torch.Tensor:
    n = int(np.prod(shape))
    buf = _PINNED.get(name)
    if buf is None or buf.numel() < n or buf.dtype != dtype:
        buf = torch.empty(max(n, 1 << 16), dtype=dtype, pin_memory=True)
        _PINNED[name] = buf
    return buf[:n].view(*shape)


def _results_to_host(scores: torch.Tensor, ids: torch.Tensor, want_scores: bool = True):
    """The result matrices through pinned staging with one stream sync."""
    hi = _pinned("ids", tuple(ids.shape), torch.int32)
    hi.copy_(ids, non_blocking=True)
    hs = None
    if want_scores:
        hs = _pinned("scores", tuple(scores.shape), torch.float64)
        hs.copy_(scores, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return (hs.numpy().copy() if want_scores else None), hi.numpy().copy()


def _norms_on(norms, dc: _dev.DeviceCodes, dev):
    """Caller norms (caller row order) as a device vector in ``dc``'s stored
    order; the resident copy when they are the matrix' own stored norms
    (bit-identical: both are the int8 norm kernel's)."""
    if getattr(dc, "_host_norm", None) is norms:
        return dc.norm
    t = torch.from_numpy(np.ascontiguousarray(norms, dtype=np.float32)).to(dev)
    return t if dc.ids is None else t[dc.ids.long()]


def scan_topk(data, queries, k, metric, data_norms=None, query_norms=None, *, _ids_only=False):
    """Exhaustive top-k per query; rows ascending by (score, id).
    (``_ids_only``: package-internal, batch_ground_truth drops the scores --
    the first element of the result is then None.)"""
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
    if int(metric) not in _FORM_OF_METRIC:
        raise ValueError(f"unknown metric {metric}")
    db = _resident(data, dev, _FORM_OF_METRIC[int(metric)])
    qs = _resident(queries, dev, "rows")
    dn = qn = None
    if int(metric) == 2:
        dn = _norms_on(data_norms, db, dev)
        qn = _norms_on(query_norms, qs, dev)
    # L2 / inner product: the stream-ordered search (no host round trip inside
    # the scan); angular keeps the synchronous entry, which reports a zero
    # norm the way exact.py does
    scores, ids = _dev.scan_topk(db, qs, int(k), int(metric), dn, qn, sync=int(metric) == 2)
    return _results_to_host(scores, ids, not _ids_only)


def pair_scores(data, queries, cand, metric, data_norms=None, query_norms=None):
    """Scores of listed pairs: float64 [nq, m], out[i, j] = the reference's
    pair score of ``queries[i]`` and ``data[cand[i, j]]`` (_core.pyx:88-96).
    This is the batched form of HnswCore._dq (_core.pyx:483-494): a host beam
    search hands the neighbour lists of a whole query batch to the GPU per
    hop.  ``cand`` int32 [nq, m]; ids outside [0, n) give +inf.  The frozen
    corpus stays resident between calls like in ``scan_topk``."""
    _check_pair(data, queries)
    if data.dtype != np.int8:
        raise ValueError("dtype must be int8")
    cand = np.ascontiguousarray(cand, dtype=np.int32)
    if cand.ndim != 2 or cand.shape[0] != queries.shape[0]:
        raise ValueError("cand must be [nq, m]")
    nq, m = cand.shape
    if nq == 0 or m == 0 or data.shape[0] == 0:
        return np.full((nq, m), np.inf, dtype=np.float64)
    if int(metric) not in _FORM_OF_METRIC:
        raise ValueError(f"unknown metric {metric}")
    if int(metric) == 2 and (data_norms is None or query_norms is None
                             or data_norms.shape[0] != data.shape[0]
                             or query_norms.shape[0] != nq):
        raise ValueError("angular metric needs data and query norms")
    dev = _dev.default_device()
    db = _resident(data, dev, "rows")
    qs = _resident(queries, dev, "rows")
    dn = qn = None
    if int(metric) == 2:
        dn = _norms_on(data_norms, db, dev)
        qn = _norms_on(query_norms, qs, dev)
    out = _dev.gather_scores(db, qs, torch.from_numpy(cand).to(dev), int(metric), dn, qn)
    return out.cpu().numpy()


# ---- single pairs: host arithmetic, exactly the reference's loops ---------

def _pair_check(a, b):
    if a.shape[0] != b.shape[0]:
        raise ValueError("length mismatch")
    if a.dtype != b.dtype:
        raise ValueError("dtype mismatch")


def _wrap_i32(v: int) -> int:
    """C ``int`` accumulation (two's complement wrap), _core.pyx:49-63."""
    return ((int(v) + (1 << 31)) % (1 << 32)) - (1 << 31)


def dot(a, b):
    """Inner product of two 1-D vectors of equal dtype (_core.pyx:99-115).
    One pair is O(d) host work, so it stays on the CPU: float32 -> float64
    products summed in order (np.cumsum is a sequential sum), int8 -> the
    exact int sum as a C int."""
    _pair_check(a, b)
    if a.shape[0] == 0:
        return 0.0
    if a.dtype == np.float32:
        return float(np.cumsum(a.astype(np.float64) * b.astype(np.float64))[-1])
    if a.dtype != np.int8:
        raise ValueError("dtype must be float32 or int8")
    return float(_wrap_i32(int(np.dot(a.astype(np.int64), b.astype(np.int64)))))


def l2sq(a, b):
    """Squared Euclidean distance of two 1-D vectors (_core.pyx:118-134)."""
    _pair_check(a, b)
    if a.shape[0] == 0:
        return 0.0
    if a.dtype == np.float32:
        t = a.astype(np.float64) - b.astype(np.float64)
        return float(np.cumsum(t * t)[-1])
    if a.dtype != np.int8:
        raise ValueError("dtype must be float32 or int8")
    t = a.astype(np.int64) - b.astype(np.int64)
    return float(_wrap_i32(int(np.dot(t, t))))


def resident_norms(mat, corpus: bool = False):
    """``norms(mat)`` as a read-only array that stays identical between
    calls for a frozen int8 matrix: passing it back as ``data_norms`` /
    ``query_norms`` lets ``scan_topk`` use the device copy instead of
    uploading it (exact.py).  ``corpus``: the matrix is an angular corpus
    (its resident form is the angular index layout)."""
    if mat.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    n, d = mat.shape
    if n == 0 or d == 0 or mat.dtype != np.int8:
        return norms(mat)
    dc = _resident(mat, _dev.default_device(), "bands" if corpus else "rows")
    out = getattr(dc, "_host_norm", None)
    if out is None:
        stored = dc.norm.cpu().numpy()
        if dc.ids is None:
            out = stored
        else:
            out = np.empty_like(stored)
            out[dc.ids.cpu().numpy()] = stored
        out.flags.writeable = False
        if not mat.flags.writeable:
            dc._host_norm = out
    return out


def norms(mat):
    """float32(sqrt(int64 sum c^2)) of every int8 row (float32 rows: the
    sequential float64 sum), _core.pyx:137-157.  A fresh array per call."""
    if mat.ndim != 2:
        raise ValueError("expected a 2-D matrix")
    n, d = mat.shape
    if n == 0 or d == 0:
        return np.zeros(n, dtype=np.float32)
    if mat.dtype == np.float32:
        return _dev.norms_f32(_to_dev(mat, _dev.default_device())).cpu().numpy()
    if mat.dtype != np.int8:
        raise ValueError("dtype must be float32 or int8")
    return np.array(resident_norms(mat))


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
