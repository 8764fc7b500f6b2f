"""ctypes binding of the C-ABI in include/qa_b200.h (libqa_b200.so).

This is the binding a ctypes-based drop-in of the reference's kernel seam
(quantann/_backend.py:14-46) uses.  The library is built in-tree by
``__graft_entry__.build()`` (or ``make -C paper_2110_08919_b200/csrc``).
There is deliberately no fallback: if the library cannot be loaded the
import fails loudly.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
# QA_B200_LIB: alternate build of the same library (A/B timing of kernel
# variants on one box); the default is the in-tree build.
LIB_PATH = Path(os.environ["QA_B200_LIB"]) if os.environ.get("QA_B200_LIB") else _HERE / "libqa_b200.so"

QA_OK = 0
QA_EINVAL = 1
QA_ECUDA = 2
QA_ENOMEM = 3
QA_EUNSUPPORTED = 4
QA_EIO = 5
QA_ETRUNCATED = 6
QA_ENONPOSITIVE = 7
QA_EDIM = 8
QA_EZERONORM = 9

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_vp = ctypes.c_void_p
c_dp = ctypes.POINTER(ctypes.c_double)


class ScanStats(ctypes.Structure):
    _fields_ = [
        ("rounds", c_i64),
        ("candidates", c_i64),
        ("launches", c_i64),
        ("retries", c_i64),
        ("filter_launches", c_i64),
        ("filter_ops", ctypes.c_double),
        ("filter_ms", ctypes.c_double),
        ("select_ms", ctypes.c_double),
    ]


# name -> (restype, argtypes); every symbol include/qa_b200.h declares.
SIGNATURES = {
    "qa_version": (c_int, []),
    "qa_last_error": (ctypes.c_char_p, []),
    "qa_device_count": (c_int, []),
    "qa_code_stride": (c_i64, [c_i64]),
    "qa_minmax_f32": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "qa_encode_i8": (
        c_int,
        [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_int, c_vp, c_i64, c_vp, c_vp, c_vp],
    ),
    "qa_norms_i8": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "qa_scan_topk_i8": (
        c_int,
        [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
         c_i64, c_int, c_i64, c_vp, c_vp, c_vp],
    ),
    "qa_scan_topk_i8_async": (
        c_int,
        [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
         c_i64, c_int, c_i64, c_vp, c_vp, c_vp],
    ),
    "qa_order_rows_by_norm": (c_int, [c_vp, c_i64, c_int, c_vp, c_vp]),
    "qa_permute_rows_i8": (c_int, [c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "qa_scan_topk_i8_host": (
        c_int,
        [c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_int, c_vp, c_vp, c_vp, c_vp],
    ),
    "qa_scan_topk_f32": (
        c_int,
        [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_int, c_i64,
         c_vp, c_vp, c_vp],
    ),
    "qa_norms_f32": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "qa_vecs_probe": (c_int, [ctypes.c_char_p, c_int, ctypes.POINTER(c_i64),
                              ctypes.POINTER(c_i64)]),
    "qa_vecs_read": (c_int, [ctypes.c_char_p, c_int, c_i64, c_i64, c_i64, c_vp, c_i64, c_int,
                             c_int, c_vp]),
    "qa_vecs_write": (c_int, [ctypes.c_char_p, c_int, c_vp, c_i64, c_i64, c_i64]),
    "qa_estimate_stats_f32": (c_int, [c_vp, c_i64, c_i64, c_i64] + [c_vp] * 9 + [c_vp]),
    "qa_gather_scores_i8": (c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                                    c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    "qa_merge_topk": (c_int, [c_vp, c_vp, c_i64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "qa_debug_dots_i8": (c_int, [c_vp, c_i64, c_vp, c_i64, c_i64, c_int, c_vp, c_vp]),
    "qa_last_scan_stats": (c_int, [ctypes.POINTER(ScanStats)]),
    "qa_set_profiling": (c_int, [c_int]),
    "qa_scan_totals": (c_int, [ctypes.POINTER(ScanStats)]),
    "qa_reset_scan_totals": (c_int, []),
}


class QAError(RuntimeError):
    """A CUDA-side failure reported by libqa_b200 (QA_ECUDA / QA_ENOMEM)."""


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (no CPU fallback exists)"
        )
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc: int) -> None:
    """Map a QA_* status to the exception the reference raises."""
    if rc == QA_OK:
        return
    msg = lib.qa_last_error().decode("utf-8", "replace")
    if rc == QA_EINVAL:
        raise ValueError(msg)
    if rc == QA_EUNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == QA_EZERONORM:
        from .errors import ZeroNorm
        raise ZeroNorm(msg)
    if rc in (QA_ETRUNCATED, QA_ENONPOSITIVE, QA_EDIM):
        from . import errors
        raise {QA_ETRUNCATED: errors.TruncatedRecord, QA_ENONPOSITIVE: errors.NonPositiveDim,
               QA_EDIM: errors.DimensionMismatch}[rc](msg)
    if rc == QA_EIO:
        if "No such file" in msg:
            raise FileNotFoundError(msg)
        raise OSError(msg)
    raise QAError(msg)


def code_stride(d: int) -> int:
    return int(lib.qa_code_stride(int(d)))


def last_scan_stats() -> dict:
    s = ScanStats()
    check(lib.qa_last_scan_stats(ctypes.byref(s)))
    return {name: getattr(s, name) for name, _ in ScanStats._fields_}


def scan_totals() -> dict:
    """qa_scan_stats summed over every scan since reset_scan_totals()."""
    s = ScanStats()
    check(lib.qa_scan_totals(ctypes.byref(s)))
    return {name: getattr(s, name) for name, _ in ScanStats._fields_}


def reset_scan_totals() -> None:
    check(lib.qa_reset_scan_totals())


def set_profiling(on: bool) -> None:
    check(lib.qa_set_profiling(1 if on else 0))
