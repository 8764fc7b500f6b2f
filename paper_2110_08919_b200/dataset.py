"""Host-side dataset containers (reference dataset.py:32-153, 278-293).

``DenseDataset`` and ``GroundTruth`` keep the reference's invariants exactly
(C-contiguous, frozen read-only arrays; d <= MAX_DIM; ground-truth rows free
of duplicates and negative ids) so results produced by this package compare
equal to the reference's.  The device-resident counterpart of a dataset is
``paper_2110_08919_b200.device.DeviceCodes``.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch

# d * 127 * 127 < 2**31 bound of the reference (dataset.py:32-34).
MAX_DIM = 133_000


class ElemKind(enum.IntEnum):
    FLOAT32 = 0
    INT8 = 1

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float32) if self is ElemKind.FLOAT32 else np.dtype(np.int8)

    @property
    def itemsize(self) -> int:
        return 4 if self is ElemKind.FLOAT32 else 1


_KINDS = {np.dtype(np.float32): ElemKind.FLOAT32, np.dtype(np.int8): ElemKind.INT8}


@dataclass(frozen=True)
class DenseDataset:
    """Row-major n x d float32 or int8 matrix, frozen on construction."""

    data: np.ndarray

    def __post_init__(self):
        arr = self.data
        if not isinstance(arr, np.ndarray) or arr.ndim != 2:
            raise ValueError("dataset data must be a 2-D numpy array")
        if arr.dtype not in _KINDS:
            raise ValueError(f"unsupported element dtype {arr.dtype}")
        if not arr.flags.c_contiguous:
            arr = np.ascontiguousarray(arr)
            object.__setattr__(self, "data", arr)
        if arr.shape[1] > MAX_DIM:
            raise DimensionMismatch(f"d={arr.shape[1]} exceeds the supported maximum {MAX_DIM}")
        arr.flags.writeable = False

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def d(self) -> int:
        return self.data.shape[1]

    @property
    def elem(self) -> ElemKind:
        return _KINDS[self.data.dtype]

    def row(self, i: int) -> np.ndarray:
        return self.data[i]

    def __eq__(self, other) -> bool:
        if not isinstance(other, DenseDataset):
            return NotImplemented
        return (self.data.dtype == other.data.dtype and self.data.shape == other.data.shape
                and np.array_equal(self.data, other.data))


QuerySet = DenseDataset


@dataclass(frozen=True)
class GroundTruth:
    """Per-query ordered neighbour id lists (0-based int32)."""

    ids: np.ndarray

    def __post_init__(self):
        ids = self.ids
        if not isinstance(ids, np.ndarray) or ids.ndim != 2:
            raise ValueError("ground truth ids must be a 2-D numpy array")
        if ids.dtype != np.int32:
            ids = ids.astype(np.int32)
        if not ids.flags.c_contiguous:
            ids = np.ascontiguousarray(ids)
        object.__setattr__(self, "ids", ids)
        if ids.size:
            if ids.min() < 0:
                raise ValueError("neighbor ids must be non-negative")
            srt = np.sort(ids, axis=1)
            if bool((srt[:, 1:] == srt[:, :-1]).any()):
                raise ValueError("a per-query neighbor list contains duplicates")
        ids.flags.writeable = False

    @classmethod
    def from_scan(cls, ids: np.ndarray) -> "GroundTruth":
        """Wrap the int32 [nq, k] id matrix of an exhaustive scan.  Its rows
        are distinct, non-negative corpus rows by construction, so the
        constructor's O(nq k log k) duplicate check is skipped."""
        if not (isinstance(ids, np.ndarray) and ids.ndim == 2 and ids.dtype == np.int32
                and ids.flags.c_contiguous):
            return cls(ids=ids)
        self = object.__new__(cls)
        object.__setattr__(self, "ids", ids)
        ids.flags.writeable = False
        return self

    @property
    def nq(self) -> int:
        return self.ids.shape[0]

    @property
    def k(self) -> int:
        return self.ids.shape[1]

    def validate_against(self, corpus: DenseDataset) -> None:
        if self.ids.size and int(self.ids.max()) >= corpus.n:
            raise ValueError("ground truth references ids beyond the corpus")

    def __eq__(self, other) -> bool:
        if not isinstance(other, GroundTruth):
            return NotImplemented
        return self.ids.shape == other.ids.shape and np.array_equal(self.ids, other.ids)


def generate_synthetic(n: int, d: int, mean: float, stddev: float, seed: int) -> DenseDataset:
    """i.i.d. Normal(mean, stddev) float32 corpus; same seed, same bits
    (reference dataset.py:278-293)."""
    if n < 0 or d < 1:
        raise ValueError("need n >= 0 and d >= 1")
    if stddev < 0:
        raise ValueError("stddev must be >= 0")
    rng = np.random.default_rng(seed)
    return DenseDataset(rng.normal(loc=mean, scale=stddev, size=(n, d)).astype(np.float32))
