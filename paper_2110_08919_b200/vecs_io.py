"""On-disk formats either side of the path.

* vector files -- fvecs / ivecs / i8vecs / bvecs (reference dataset.py:160-275):
  ``load_fvecs``, ``load_ivecs``, ``load_i8vecs``, ``load_bvecs``,
  ``save_fvecs``, ``save_ivecs``, ``save_i8vecs`` keep the reference's names,
  return types and error kinds (TruncatedRecord, NonPositiveDim,
  DimensionMismatch, ElementKindMismatch).  Framing is validated and parsed by
  the native reader of libqa_b200 (csrc/qa_vecs.cu, ``qa_vecs_probe`` /
  ``qa_vecs_read`` / ``qa_vecs_write``).
* device loaders -- ``load_fvecs_to_device`` / ``load_i8vecs_to_device`` /
  ``load_bvecs_to_device`` stream one rank's row shard straight into HBM
  (pinned double-buffered staging, header-stripping 2-D DMA): float32 rows
  for encoding, or int8 rows at the padded code stride with their norms.
* quantizer params -- the QZP1 layout (quantizer.py:330-369):
  ``save_params`` / ``load_params``, bit-exact round trips, errors BadMagic /
  UnsupportedVersion / TruncatedFile.
"""

from __future__ import annotations

import ctypes
import os
import struct
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import check, lib
from .dataset import DenseDataset, ElemKind, GroundTruth
from .errors import BadMagic, ElementKindMismatch, TruncatedFile, UnsupportedVersion


def _path(path) -> bytes:
    return os.fsencode(os.fspath(path))


def probe(path, itemsize: int) -> tuple[int, int]:
    """(n, d) of a record file after validating its whole framing."""
    n, d = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib.qa_vecs_probe(_path(path), int(itemsize), ctypes.byref(n), ctypes.byref(d)))
    return int(n.value), int(d.value)


def _read_host(path, itemsize: int, dtype, recenter: bool = False) -> np.ndarray:
    n, d = probe(path, itemsize)
    if d == 0:
        return np.empty((0, 0), dtype=dtype)
    out = np.empty((n, d), dtype=dtype)
    check(lib.qa_vecs_read(_path(path), int(itemsize), d, 0, n, out.ctypes.data, d * itemsize, 0,
                           1 if recenter else 0, None))
    return out


def load_fvecs(path) -> DenseDataset:
    """float32 dataset in fvecs framing (dataset.py:212-218)."""
    return DenseDataset(_read_host(path, 4, np.float32))


def load_ivecs(path) -> GroundTruth:
    """Ground-truth id lists in ivecs framing (dataset.py:221-227)."""
    return GroundTruth(_read_host(path, 4, np.int32))


def load_i8vecs(path) -> DenseDataset:
    """Signed int8 dataset in i8vecs framing (dataset.py:240-245)."""
    return DenseDataset(_read_host(path, 1, np.int8))


def load_bvecs(path) -> DenseDataset:
    """bvecs bytes re-centred to int8, v - 128 (dataset.py:230-237)."""
    return DenseDataset(_read_host(path, 1, np.int8, recenter=True))


def load_dataset(path) -> DenseDataset:
    """fvecs / bvecs / i8vecs chosen by extension (dataset.py:296-305)."""
    ext = Path(path).suffix.lower()
    loader = {".fvecs": load_fvecs, ".bvecs": load_bvecs, ".i8vecs": load_i8vecs}.get(ext)
    if loader is None:
        raise ValueError(f"cannot infer dataset format from extension {ext!r}")
    return loader(path)


def _write(path, itemsize: int, arr: np.ndarray) -> None:
    arr = np.ascontiguousarray(arr)
    n, d = arr.shape
    check(lib.qa_vecs_write(_path(path), int(itemsize), arr.ctypes.data if arr.size else None, n,
                            d, d * itemsize))


def save_fvecs(ds: DenseDataset, path) -> None:
    if ds.elem is not ElemKind.FLOAT32:
        raise ElementKindMismatch("save_fvecs needs a Float32 dataset")
    _write(path, 4, ds.data.astype("<f4", copy=False))


def save_ivecs(gt: GroundTruth, path) -> None:
    _write(path, 4, gt.ids.astype("<i4", copy=False))


def save_i8vecs(ds: DenseDataset, path) -> None:
    if ds.elem is not ElemKind.INT8:
        raise ElementKindMismatch("save_i8vecs needs an Int8 dataset")
    _write(path, 1, ds.data)


# ------------------------------------------------------------ to the device --

def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    from .sharded import shard_bounds
    return shard_bounds(n, world, rank)


def load_fvecs_to_device(path, rank: int = 0, world: int = 1, device=None):
    """This rank's contiguous row shard of an fvecs file as a float32
    [rows, d] CUDA tensor (input of the encode kernel).  Returns
    (tensor, row offset, total n)."""
    import torch

    from . import device as dev

    n, d = probe(path, 4)
    lo, hi = shard_rows(n, world, rank)
    device = device or dev.default_device()
    out = torch.empty((hi - lo, d), dtype=torch.float32, device=device)
    if hi > lo:
        check(lib.qa_vecs_read(_path(path), 4, d, lo, hi, out.data_ptr(), d * 4, 1, 0,
                               torch.cuda.current_stream(device).cuda_stream))
    return out, lo, n


def _load_codes_to_device(path, recenter: bool, rank: int, world: int, device):
    import torch

    from . import device as dev

    n, d = probe(path, 1)
    lo, hi = shard_rows(n, world, rank)
    device = device or dev.default_device()
    codes = dev.DeviceCodes.empty(hi - lo, d, device)
    if hi > lo:
        if codes.ld != d:
            codes.codes.zero_()   # pad columns must be zero (K padding of the MMA)
        check(lib.qa_vecs_read(_path(path), 1, d, lo, hi, codes.codes.data_ptr(), codes.ld, 1,
                               1 if recenter else 0,
                               torch.cuda.current_stream(device).cuda_stream))
        dev.norms_(codes)
    return codes, lo, n


def load_i8vecs_to_device(path, rank: int = 0, world: int = 1, device=None):
    """This rank's row shard of an i8vecs file as DeviceCodes (padded code
    stride, int32 sqnorm + float32 norm).  Returns (codes, row offset, n)."""
    return _load_codes_to_device(path, False, rank, world, device)


def load_bvecs_to_device(path, rank: int = 0, world: int = 1, device=None):
    """bvecs shard as DeviceCodes, bytes re-centred v - 128 on the way."""
    return _load_codes_to_device(path, True, rank, world, device)


# ---------------------------------------------------------------- QZP1 params --

_PARAMS_MAGIC = b"QZP1"
_PARAMS_VERSION = 1
# magic, version, bits, mode, reserved (4 x u8), d (u32), little-endian
_HEADER = struct.Struct("<4s4BI")


def save_params(p, path) -> None:
    """QuantizerParams -> QZP1 file: header, then d (k, sb, se) float32
    triples (quantizer.py:330-341)."""
    head = _HEADER.pack(_PARAMS_MAGIC, _PARAMS_VERSION, p.bits, int(p.mode), 0, p.d)
    body = np.stack([p.k, p.sb, p.se], axis=1).astype("<f4").tobytes()
    Path(path).write_bytes(head + body)


def load_params(path):
    """QZP1 file -> QuantizerParams, bit-exact (quantizer.py:344-369)."""
    from .quantizer import QuantizerParams, QuantMode

    raw = Path(path).read_bytes()
    if len(raw) < _HEADER.size:
        raise TruncatedFile(f"{path}: shorter than the fixed header")
    magic, version, bits, mode_code, _, d = _HEADER.unpack_from(raw)
    if magic != _PARAMS_MAGIC:
        raise BadMagic(f"{path}: not a params file")
    if version != _PARAMS_VERSION:
        raise UnsupportedVersion(f"{path}: version {version} not supported")
    want = _HEADER.size + 12 * d
    if len(raw) != want:
        raise TruncatedFile(f"{path}: {len(raw)} bytes but header implies {want}")
    if mode_code not in {int(m) for m in QuantMode}:
        raise UnsupportedVersion(f"{path}: unknown mode code {mode_code}")
    t = np.frombuffer(raw, dtype="<f4", offset=_HEADER.size).reshape(d, 3).astype(np.float32)
    return QuantizerParams(bits=bits, mode=QuantMode(mode_code), k=t[:, 0].copy(),
                           sb=t[:, 1].copy(), se=t[:, 2].copy())


__all__ = ["load_dataset", "load_fvecs", "load_ivecs", "load_i8vecs", "load_bvecs", "save_fvecs", "save_ivecs",
           "save_i8vecs", "load_fvecs_to_device", "load_i8vecs_to_device",
           "load_bvecs_to_device", "save_params", "load_params", "probe"]
_ = _lib  # the library must be loadable (no fallback)
