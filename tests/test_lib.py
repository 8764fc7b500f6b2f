"""The C-ABI library loads, exports every symbol include/qa_b200.h declares,
and rejects bad arguments with the reference's errors before touching a
device (no compute calls here)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2110_08919_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "qa_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(qa_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(_lib.lib, name), name
        assert name in _lib.SIGNATURES, f"{name} declared but not bound in _lib.py"


def test_library_is_sm100a_cuda_build():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_identification():
    assert _lib.lib.qa_version() >= 1
    assert _lib.lib.qa_device_count() >= 0
    assert [_lib.code_stride(d) for d in (0, 1, 32, 33, 64, 65, 100, 128, 129, 256, 300)] == \
        [32, 32, 32, 64, 64, 128, 128, 128, 256, 256, 384]


def test_invalid_arguments_map_to_reference_errors():
    L = _lib.lib
    # unknown metric / negative k -> ValueError (_core.pyx:340-347)
    with pytest.raises(ValueError, match="metric"):
        _lib.check(L.qa_scan_topk_i8(None, 10, 4, 32, None, None, None, None, 1, 32, None, None, 5, 7,
                                     0, None, None, None))
    with pytest.raises(ValueError, match="k must be >= 0"):
        _lib.check(L.qa_scan_topk_i8(None, 10, 4, 32, None, None, None, None, 1, 32, None, None, -1, 0,
                                     0, None, None, None))
    with pytest.raises(ValueError, match="angular metric needs data and query norms"):
        _lib.check(L.qa_scan_topk_i8(None, 10, 4, 32, None, None, None, None, 1, 32, None, None, 5, 2,
                                     0, None, None, None))
    with pytest.raises(ValueError, match="stride"):
        _lib.check(L.qa_scan_topk_i8(None, 10, 4, 16, None, None, None, None, 1, 32, None, None, 5, 0,
                                     0, None, None, None))
    with pytest.raises(ValueError, match="bits must be between 1 and 8"):
        _lib.check(L.qa_encode_i8(None, 1, 1, 1, None, None, None, 9, None, 32, None, None, None))
    with pytest.raises(ValueError, match="k exceeds"):
        _lib.check(L.qa_merge_topk(None, None, 2, 1, 3, 7, None, None, None))
    with pytest.raises(NotImplementedError, match="int32 ids"):  # any k is served; n is not
        _lib.check(L.qa_scan_topk_i8(None, 2**31 + 1, 8, 32, None, None, None, None, 1, 32, None,
                                     None, 10, 0, 0, None, None, None))
    # empty problems are valid no-ops (_core.pyx:352-353)
    _lib.check(L.qa_scan_topk_i8(None, 0, 4, 32, None, None, None, None, 3, 32, None, None, 5, 0, 0,
                                 None, None, None))
    _lib.check(L.qa_scan_topk_i8(None, 10, 4, 32, None, None, None, None, 0, 32, None, None, 5, 0, 0,
                                 None, None, None))


def test_stats_struct_roundtrip():
    s = _lib.ScanStats()
    assert _lib.lib.qa_last_scan_stats(ctypes.byref(s)) == 0
