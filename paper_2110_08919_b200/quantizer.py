"""Per-dimension clamped linear quantization (reference quantizer.py).

Window fitting (``fit``) is O(d) float64 host arithmetic identical to the
reference's (quantizer.py:225-267).  The O(n*d) parts -- the calibration
reductions and the Eq. 1 encode -- run on the GPU (libqa_b200):

* ``minmax_stats``  per-dimension min/max (exact, order-free), the statistic
  every BASELINE configuration calibrates from;
* ``fit_minmax`` / ``fit_symmetric`` build the reference's ABS_MAX fit from
  those statistics (window [min, max], resp. [-max|x|, +max|x|]) through the
  same ``fit`` arithmetic the reference uses;
* ``quantize_dataset`` / ``quantize_query`` encode through the fused encode
  kernel, bit-exact with numpy's float32 evaluation order.

* ``estimate_stats`` the reference's full statistics (mean, sigma, trimmed
  abs-max, pooled) for its own SIGMA_CLAMP / ABS_MAX / UNIFORM_SIGMA_CLAMP
  modes, reproducing numpy's float64 summation orders on the GPU
  (csrc/qa_stats.cu).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass

import numpy as np

from .dataset import DenseDataset, ElemKind
from .errors import DimensionMismatch, ElementKindMismatch, TooFewSamples

DEGENERATE_WIDTH = 1e-12
DEGENERATE_HALF_WIDTH = 1e-6


class QuantMode(enum.IntEnum):
    SIGMA_CLAMP = 0
    ABS_MAX = 1
    UNIFORM_SIGMA_CLAMP = 2

    @classmethod
    def parse(cls, name: str) -> "QuantMode":
        key = name.strip().lower()
        table = {"sigma": cls.SIGMA_CLAMP, "sigmaclamp": cls.SIGMA_CLAMP, "absmax": cls.ABS_MAX,
                 "uniform": cls.UNIFORM_SIGMA_CLAMP, "uniformsigma": cls.UNIFORM_SIGMA_CLAMP}
        if key not in table:
            raise ValueError(f"unknown mode {name!r}; expected sigma, absmax, or uniform")
        return table[key]

    @property
    def short_name(self) -> str:
        return ("sigma", "absmax", "uniform")[int(self)]


def _frozen(arr: np.ndarray) -> np.ndarray:
    arr = np.ascontiguousarray(arr)
    arr.flags.writeable = False
    return arr


@dataclass(frozen=True)
class DimensionStats:
    """Per-dimension statistics feeding ``fit`` (reference quantizer.py:85-112)."""

    mu: np.ndarray
    sigma: np.ndarray
    min: np.ndarray
    max: np.ndarray
    trimmed_absmax: np.ndarray
    pooled_mu: float
    pooled_sigma: float
    count: int

    def __post_init__(self):
        for name in ("mu", "sigma", "min", "max", "trimmed_absmax"):
            arr = getattr(self, name)
            if arr.ndim != 1 or arr.dtype != np.float64:
                raise ValueError(f"{name} must be a 1-D float64 array")
            object.__setattr__(self, name, _frozen(arr))

    @property
    def d(self) -> int:
        return self.mu.shape[0]


@dataclass(frozen=True)
class QuantizerParams:
    """Fitted float32 window constants (reference quantizer.py:115-165)."""

    bits: int
    mode: QuantMode
    k: np.ndarray
    sb: np.ndarray
    se: np.ndarray

    def __post_init__(self):
        if not 1 <= self.bits <= 8:
            raise ValueError("bits must be between 1 and 8")
        object.__setattr__(self, "mode", QuantMode(self.mode))
        for name in ("k", "sb", "se"):
            arr = getattr(self, name)
            if arr.ndim != 1 or arr.dtype != np.float32:
                raise ValueError(f"{name} must be a 1-D float32 array")
            object.__setattr__(self, name, _frozen(arr))
        if not (self.k.shape == self.sb.shape == self.se.shape):
            raise ValueError("k, sb, se must share a shape")
        if not bool(np.all(self.sb < self.se)):
            raise ValueError("every dimension needs sb < se")

    @property
    def d(self) -> int:
        return self.k.shape[0]

    @property
    def lo_code(self) -> int:
        return -(1 << (self.bits - 1))

    @property
    def hi_code(self) -> int:
        return (1 << (self.bits - 1)) - 1

    def __eq__(self, other) -> bool:
        if not isinstance(other, QuantizerParams):
            return NotImplemented
        return (self.bits == other.bits and self.mode == other.mode
                and self.k.shape == other.k.shape and np.array_equal(self.k, other.k)
                and np.array_equal(self.sb, other.sb) and np.array_equal(self.se, other.se))


@dataclass(frozen=True)
class FitResult:
    params: QuantizerParams
    degenerate_dims: tuple


def fit(stats: DimensionStats, bits: int, mode: QuantMode) -> FitResult:
    """Window constants from statistics, float64 then float32 (quantizer.py:225-267)."""
    if not 1 <= bits <= 8:
        raise ValueError("bits must be between 1 and 8")
    mode = QuantMode(mode)
    d = stats.d
    if mode is QuantMode.SIGMA_CLAMP:
        center, half = stats.mu.copy(), stats.sigma.copy()
    elif mode is QuantMode.UNIFORM_SIGMA_CLAMP:
        center = np.full(d, stats.pooled_mu, dtype=np.float64)
        half = np.full(d, stats.pooled_sigma, dtype=np.float64)
    else:
        center, half = stats.mu.copy(), stats.trimmed_absmax.copy()
    lo = center - half
    hi = center + half
    degenerate = hi - lo < DEGENERATE_WIDTH
    if degenerate.any():
        lo[degenerate] = center[degenerate] - DEGENERATE_HALF_WIDTH
        hi[degenerate] = center[degenerate] + DEGENERATE_HALF_WIDTH
    k32, sb32, se32 = center.astype(np.float32), lo.astype(np.float32), hi.astype(np.float32)
    collapsed = ~(sb32 < se32)
    if collapsed.any():
        sb32[collapsed] = np.nextafter(k32[collapsed], np.float32(-np.inf))
        se32[collapsed] = np.nextafter(k32[collapsed], np.float32(np.inf))
        degenerate = degenerate | collapsed
    params = QuantizerParams(bits=bits, mode=mode, k=k32, sb=sb32, se=se32)
    return FitResult(params=params, degenerate_dims=tuple(int(i) for i in np.flatnonzero(degenerate)))


@dataclass(frozen=True)
class RangeStats:
    """Exact per-dimension min/max of a float32 corpus (float64 copies)."""

    min: np.ndarray
    max: np.ndarray
    count: int

    @property
    def d(self) -> int:
        return self.min.shape[0]


def minmax_stats(data) -> RangeStats:
    """Per-dimension min/max on the GPU.  ``data`` is a float32 DenseDataset,
    numpy [n, d] array or CUDA tensor."""
    import torch

    from . import device as dev

    if isinstance(data, DenseDataset):
        if data.elem is not ElemKind.FLOAT32:
            raise ElementKindMismatch("statistics are estimated on Float32 corpora")
        data = data.data
    if isinstance(data, np.ndarray):
        if data.dtype != np.float32 or data.ndim != 2:
            raise ElementKindMismatch("statistics are estimated on Float32 corpora")
        t = dev.host_to_device(data)
    else:
        t = data
    n = t.shape[0]
    if n < 2:
        raise TooFewSamples(f"need at least 2 vectors, got {n}")
    mn, mx = dev.minmax(t)
    return RangeStats(min=mn.double().cpu().numpy(), max=mx.double().cpu().numpy(), count=n)


def estimate_stats(data) -> DimensionStats:
    """The reference's calibration statistics (quantizer.py:176-222), on the
    GPU and bit-exact with its numpy evaluation (csrc/qa_stats.cu): per-dim
    mean, MLE sigma, min, max, 0.1%/99.9%-trimmed abs-max, pooled mean and
    sigma.  ``data``: float32 DenseDataset, numpy [n, d] array or CUDA tensor."""
    import ctypes

    import torch

    from . import device as dev
    from ._lib import check, lib

    if isinstance(data, DenseDataset):
        if data.elem is not ElemKind.FLOAT32:
            raise ElementKindMismatch("statistics are estimated on Float32 corpora")
        data = data.data
    if isinstance(data, np.ndarray):
        if data.dtype != np.float32 or data.ndim != 2:
            raise ElementKindMismatch("statistics are estimated on Float32 corpora")
        t = dev.host_to_device(data)
    else:
        t = data
    if t.dtype != torch.float32 or t.dim() != 2:
        raise ElementKindMismatch("statistics are estimated on Float32 corpora")
    n, d = t.shape
    if n < 2:
        raise TooFewSamples(f"need at least 2 vectors, got {n}")
    t = t if t.stride(1) == 1 else t.contiguous()
    out = {k: np.empty(d, dtype=np.float64) for k in ("mu", "sigma", "min", "max", "tam")}
    pm, ps = ctypes.c_double(0.0), ctypes.c_double(0.0)
    check(lib.qa_estimate_stats_f32(t.data_ptr(), n, d, t.stride(0), out["mu"].ctypes.data,
                                    out["sigma"].ctypes.data, out["min"].ctypes.data,
                                    out["max"].ctypes.data, out["tam"].ctypes.data, None, None,
                                    ctypes.addressof(pm), ctypes.addressof(ps),
                                    torch.cuda.current_stream(t.device).cuda_stream))
    return DimensionStats(mu=out["mu"], sigma=out["sigma"], min=out["min"], max=out["max"],
                          trimmed_absmax=out["tam"], pooled_mu=float(pm.value),
                          pooled_sigma=float(ps.value), count=int(n))


def _range_fit(center: np.ndarray, half: np.ndarray, count: int, bits: int) -> FitResult:
    zeros = np.zeros_like(center)
    stats = DimensionStats(mu=center, sigma=zeros, min=center - half, max=center + half,
                           trimmed_absmax=half, pooled_mu=0.0, pooled_sigma=0.0, count=count)
    return fit(stats, bits, QuantMode.ABS_MAX)


def fit_minmax(stats: RangeStats, bits: int = 8) -> FitResult:
    """Per-dimension min/max affine window: the reference's ABS_MAX fit with
    mu = (min+max)/2 and half-width (max-min)/2 (float64), i.e. sb = min,
    se = max up to float64 rounding -- exactly the values the reference's
    ``fit`` produces from those statistics."""
    center = (stats.min + stats.max) / 2.0
    half = (stats.max - stats.min) / 2.0
    return _range_fit(center, half, stats.count, bits)


def fit_symmetric(stats: RangeStats, bits: int = 8) -> FitResult:
    """Symmetric window [-M_j, +M_j], M_j = max |x_j| (BASELINE config 1)."""
    half = np.maximum(np.abs(stats.min), np.abs(stats.max))
    return _range_fit(np.zeros_like(half), half, stats.count, bits)


def quantize_value(x: float, dim: int, p: QuantizerParams) -> int:
    """One coordinate through Eq. 1 (scalar utility, quantizer.py:270-288);
    same float32 operation order as the encode kernel."""
    sb, se = float(p.sb[dim]), float(p.se[dim])
    if sb <= x <= se:
        ratio = (np.float32(x) - p.k[dim]) / (p.se[dim] - p.sb[dim])
        q = math.floor(float(np.float32(2.0 ** p.bits) * ratio))
        return max(p.lo_code, min(p.hi_code, q))
    return p.hi_code if x > se else p.lo_code


def dequantize_value(q: int, dim: int, p: QuantizerParams) -> float:
    """Bin centre of a code (quantizer.py:323-327)."""
    width = float(p.se[dim]) - float(p.sb[dim])
    return float(p.k[dim]) + (q + 0.5) * width / (2.0 ** p.bits)


def _params_on(p: QuantizerParams, device):
    import torch

    return tuple(torch.from_numpy(np.array(a, dtype=np.float32)).to(device) for a in (p.k, p.sb, p.se))


def quantize_array(values: np.ndarray, p: QuantizerParams) -> np.ndarray:
    """Encode a float32 [n, d] host array on the GPU; returns int8 [n, d]."""
    import torch

    from . import device as dev

    if values.dtype != np.float32 or values.ndim != 2:
        raise ElementKindMismatch("quantization input must be float32")
    n, d = values.shape
    if n == 0:
        return np.empty((0, d), dtype=np.int8)
    device = dev.default_device()
    x = dev.host_to_device(values, device)
    k, sb, se = _params_on(p, device)
    codes = dev.encode(x, k, sb, se, p.bits)
    return codes.to_host()


def quantize_dataset(ds: DenseDataset, p: QuantizerParams) -> DenseDataset:
    """Quantize a float corpus to int8 codes (quantizer.py:303-309)."""
    if ds.elem is not ElemKind.FLOAT32:
        raise ElementKindMismatch("quantization input must be Float32")
    if ds.d != p.d:
        raise DimensionMismatch(f"dataset d={ds.d} but params d={p.d}")
    return DenseDataset(quantize_array(ds.data, p))


def quantize_query(q: np.ndarray, p: QuantizerParams) -> np.ndarray:
    """Quantize one float32 vector with the corpus mapping (quantizer.py:312-320)."""
    if q.ndim != 1:
        raise DimensionMismatch("expected a 1-D query vector")
    if q.dtype != np.float32:
        raise ElementKindMismatch("quantization input must be float32")
    if q.shape[0] != p.d:
        raise DimensionMismatch(f"query d={q.shape[0]} but params d={p.d}")
    return quantize_array(q[np.newaxis, :], p)[0]
