"""Device-resident data and the calls into libqa_b200 on torch-managed HBM.

PyTorch supplies device memory and the current CUDA stream; every compute
step is a kernel of libqa_b200.so reached through the C-ABI
(include/qa_b200.h).  Layout in HBM:

* codes   int8  [n, ld]  row stride ld = qa_code_stride(d) (32, 64 or a
                          multiple of 128 bytes; pad columns are zero) -- the
                          K granularity of the tcgen05 kind::i8 MMA and the
                          TMA swizzle width;
* sqnorm  int32 [n]      sum of squared codes (L2 epilogue correction);
* norm    fp32  [n]      float32(sqrt(double(sqnorm))) (angular metric,
                          reference _core.pyx:154-156).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2110_08919_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def host_to_device(arr: np.ndarray, device=None) -> torch.Tensor:
    """Copy a C-contiguous host array to the device without an extra host
    copy.  Read-only arrays (frozen DenseDatasets) are only ever read: the
    tensor wrapping them is the source of one H2D copy and then dropped."""
    import warnings

    arr = np.ascontiguousarray(arr)
    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message=".*not writable.*")
        src = torch.from_numpy(arr)
    return src.to(device or default_device())


@dataclass
class DeviceCodes:
    """int8 code matrix resident in HBM plus its per-row norms."""

    codes: torch.Tensor    # int8 [n, ld]
    d: int
    sqnorm: torch.Tensor   # int32 [n]
    norm: torch.Tensor     # float32 [n]
    ids: torch.Tensor | None = None  # int32 [n]: stored row -> reported id (None: identity)

    @property
    def n(self) -> int:
        return self.codes.shape[0]

    @property
    def ld(self) -> int:
        return self.codes.shape[1]

    @property
    def device(self) -> torch.device:
        return self.codes.device

    @classmethod
    def empty(cls, n: int, d: int, device=None) -> "DeviceCodes":
        device = device or default_device()
        ld = _lib.code_stride(d)
        return cls(
            codes=torch.empty((n, ld), dtype=torch.int8, device=device),
            d=d,
            sqnorm=torch.empty((n,), dtype=torch.int32, device=device),
            norm=torch.empty((n,), dtype=torch.float32, device=device),
        )

    @classmethod
    def from_host(cls, arr: np.ndarray, device=None) -> "DeviceCodes":
        """Upload an int8 [n, d] host matrix and compute its norms on device."""
        arr = np.ascontiguousarray(arr)
        if arr.dtype != np.int8 or arr.ndim != 2:
            raise ValueError("expected a 2-D int8 array")
        n, d = arr.shape
        out = cls.empty(n, d, device)
        if n:
            if out.ld != d:
                out.codes.zero_()
            if d:
                import warnings

                with warnings.catch_warnings():
                    warnings.filterwarnings("ignore", message=".*not writable.*")
                    src = torch.from_numpy(arr)
                out.codes[:, :d].copy_(src, non_blocking=False)
            elif out.ld:
                out.codes.zero_()
            norms_(out)
        return out

    def to_host(self) -> np.ndarray:
        return self.codes[:, : self.d].cpu().numpy()

    def slice_rows(self, lo: int, hi: int) -> "DeviceCodes":
        ids = None if self.ids is None else self.ids[lo:hi]
        return DeviceCodes(self.codes[lo:hi], self.d, self.sqnorm[lo:hi], self.norm[lo:hi], ids)

    def shuffled(self, seed: int = 0) -> "DeviceCodes":
        """Copy with rows in a fixed pseudo-random order (``ids`` map back):
        any prefix is a uniform sample of the rows, which the scan's threshold
        estimate assumes, whatever order the caller's rows come in."""
        g = torch.Generator(device=self.device)
        g.manual_seed(seed)
        perm = torch.randperm(self.n, generator=g, device=self.device, dtype=torch.int64).to(torch.int32)
        return self._permuted(perm)

    def _permuted(self, perm: torch.Tensor) -> "DeviceCodes":
        out = DeviceCodes.empty(self.n, self.d, self.device)
        check(lib.qa_permute_rows_i8(_p(self.codes), _p(self.sqnorm), _p(self.norm), self.n,
                                     self.ld, _p(perm), _p(out.codes), _p(out.sqnorm),
                                     _p(out.norm), _stream()))
        out.ids = perm if self.ids is None else self.ids[perm.long()]
        return out

    def sorted_by_norm(self, stratify: bool = True) -> "DeviceCodes":
        """Copy with rows in ascending-norm order (stable) and ``ids`` mapping
        each stored row back to its position in this matrix.  The scan's
        per-warp bounds are tight on such a layout (qa_layout.cu)."""
        perm = torch.empty((self.n,), dtype=torch.int32, device=self.device)
        check(lib.qa_order_rows_by_norm(_p(self.sqnorm), self.n, 1 if stratify else 0, _p(perm),
                                        _stream()))
        return self._permuted(perm)


def norms_(dc: DeviceCodes) -> None:
    """(Re)compute sqnorm/norm of a DeviceCodes in place (_core.pyx:137-157)."""
    check(lib.qa_norms_i8(_p(dc.codes), dc.n, dc.d, dc.ld, _p(dc.sqnorm), _p(dc.norm), _stream()))


def minmax(x: torch.Tensor):
    """Per-dimension (min, max) of a float32 [n, d] device matrix, exact."""
    if x.dtype != torch.float32 or x.dim() != 2 or not x.is_cuda:
        raise ValueError("expected a float32 [n, d] CUDA tensor")
    x = x if x.stride(1) == 1 else x.contiguous()
    n, d = x.shape
    mn = torch.empty(d, dtype=torch.float32, device=x.device)
    mx = torch.empty(d, dtype=torch.float32, device=x.device)
    check(lib.qa_minmax_f32(_p(x), n, d, x.stride(0), _p(mn), _p(mx), _stream()))
    return mn, mx


def encode(x: torch.Tensor, k: torch.Tensor, sb: torch.Tensor, se: torch.Tensor, bits: int,
           out: DeviceCodes | None = None) -> DeviceCodes:
    """Eq. 1 encode of a float32 [n, d] device matrix (quantizer.py:291-300),
    fused with the code norms."""
    if x.dtype != torch.float32 or x.dim() != 2 or not x.is_cuda:
        raise ValueError("expected a float32 [n, d] CUDA tensor")
    x = x if x.stride(1) == 1 else x.contiguous()
    n, d = x.shape
    for name, t in (("k", k), ("sb", sb), ("se", se)):
        if t.dtype != torch.float32 or t.shape != (d,) or t.device != x.device:
            raise ValueError(f"{name} must be float32[{d}] on {x.device}")
    if out is None:
        out = DeviceCodes.empty(n, d, x.device)
    elif out.n != n or out.d != d or out.device != x.device:
        raise ValueError(f"out must hold {n} signed code rows of width {d} on {x.device}")
    check(lib.qa_encode_i8(_p(x), n, d, x.stride(0), _p(k.contiguous()), _p(sb.contiguous()),
                           _p(se.contiguous()), int(bits), _p(out.codes), out.ld,
                           _p(out.sqnorm), _p(out.norm), _stream()))
    return out


def scan_topk(db: DeviceCodes, q: DeviceCodes, k: int, metric: int, db_norm=None, q_norm=None,
              id_offset: int = 0, out=None, sync: bool = True):
    """Exhaustive top-k of every query over the database (_core.pyx:333-365).

    Returns (scores float64 [nq, keff], ids int32 [nq, keff]) on the device,
    rows ascending by (score, id), keff = min(k, n).  For the angular metric
    ``db_norm``/``q_norm`` (float32 device vectors) override the stored code
    norms, as the reference takes them from the caller.

    ``sync=False``: qa_scan_topk_i8_async -- no host round trip; flagged
    queries are recomputed on the device; a zero angular norm is not
    reported (the caller's check).
    """
    if db.d != q.d:
        raise ValueError("dimension mismatch between data and queries")
    if k < 0:
        raise ValueError("k must be >= 0")
    keff = min(k, db.n)
    dev = db.device
    if out is None:
        scores = torch.empty((q.n, keff), dtype=torch.float64, device=dev)
        ids = torch.empty((q.n, keff), dtype=torch.int32, device=dev)
    else:
        scores, ids = out
        for t, dt in ((scores, torch.float64), (ids, torch.int32)):
            if (t.dtype != dt or tuple(t.shape) != (q.n, keff) or t.device != dev
                    or not t.is_contiguous()):
                raise ValueError(f"out tensors must be contiguous [{q.n}, {keff}] "
                                 f"float64/int32 on {dev}")
    dn = db.norm if db_norm is None else db_norm
    qn = q.norm if q_norm is None else q_norm
    fn = lib.qa_scan_topk_i8 if sync else lib.qa_scan_topk_i8_async
    check(fn(_p(db.codes), db.n, db.d, db.ld, _p(db.sqnorm), _p(dn), _p(db.ids), _p(q.codes), q.n,
             q.ld, _p(q.sqnorm), _p(qn), int(k), int(metric), int(id_offset), _p(scores), _p(ids),
             _stream()))
    return scores, ids


def gather_scores(db: DeviceCodes, q: DeviceCodes, cand: torch.Tensor, metric: int, db_norm=None,
                  q_norm=None, row_of_id: torch.Tensor | None = None) -> torch.Tensor:
    """float64 [nq, m] scores of the listed pairs: out[i, j] = the reference's
    pair score of query i and database row ``cand[i, j]`` (_core.pyx:88-96;
    HnswCore._dq / _dist_rows, 472-494).  ``cand``: int32 [nq, m] device
    tensor of caller ids; ids outside [0, n) (e.g. -1 padding of ragged
    neighbour lists) give +inf.  ``row_of_id`` maps caller id -> stored row
    for a database kept in an index layout (see ``inverse_ids``)."""
    if db.d != q.d:
        raise ValueError("dimension mismatch between data and queries")
    if cand.dtype != torch.int32 or cand.dim() != 2 or cand.shape[0] != q.n or not cand.is_cuda:
        raise ValueError(f"cand must be an int32 [{q.n}, m] CUDA tensor")
    cand = cand if cand.stride(1) == 1 else cand.contiguous()
    m = cand.shape[1]
    out = torch.empty((q.n, m), dtype=torch.float64, device=db.device)
    dn = db.norm if db_norm is None else db_norm
    qn = q.norm if q_norm is None else q_norm
    check(lib.qa_gather_scores_i8(_p(db.codes), db.n, db.d, db.ld, _p(db.sqnorm), _p(dn),
                                  _p(row_of_id), _p(q.codes), q.n, q.ld, _p(q.sqnorm), _p(qn),
                                  _p(cand), m, cand.stride(0), int(metric), _p(out), _stream()))
    return out


def inverse_ids(dc: DeviceCodes) -> torch.Tensor | None:
    """caller id -> stored row of an index-layout DeviceCodes (None: identity)."""
    if dc.ids is None:
        return None
    inv = torch.empty((dc.n,), dtype=torch.int32, device=dc.device)
    inv[dc.ids.long()] = torch.arange(dc.n, dtype=torch.int32, device=dc.device)
    return inv


def _f32_matrix(x: torch.Tensor, what: str) -> torch.Tensor:
    if x.dtype != torch.float32 or x.dim() != 2 or not x.is_cuda:
        raise ValueError(f"{what} must be a float32 [n, d] CUDA tensor")
    return x if x.stride(1) == 1 else x.contiguous()


def norms_f32(x: torch.Tensor) -> torch.Tensor:
    """float32(sqrt(sequential float64 sum of x^2)) per row (_core.pyx:150-153)."""
    x = _f32_matrix(x, "x")
    out = torch.empty((x.shape[0],), dtype=torch.float32, device=x.device)
    check(lib.qa_norms_f32(_p(x), x.shape[0], x.shape[1], x.stride(0), _p(out), _stream()))
    return out


def scan_topk_f32(db: torch.Tensor, q: torch.Tensor, k: int, metric: int, db_norm=None,
                  q_norm=None, id_offset: int = 0):
    """float32 exhaustive top-k, bit-exact with the reference's _scan_f32
    (_core.pyx:270-298): float64 scores, rows ascending by (score, id)."""
    db = _f32_matrix(db, "data")
    q = _f32_matrix(q, "queries")
    if db.shape[1] != q.shape[1]:
        raise ValueError("dimension mismatch between data and queries")
    if k < 0:
        raise ValueError("k must be >= 0")
    keff = min(k, db.shape[0])
    scores = torch.empty((q.shape[0], keff), dtype=torch.float64, device=db.device)
    ids = torch.empty((q.shape[0], keff), dtype=torch.int32, device=db.device)
    check(lib.qa_scan_topk_f32(_p(db), db.shape[0], db.shape[1], db.stride(0), _p(db_norm),
                               _p(q), q.shape[0], q.stride(0), _p(q_norm), int(k), int(metric),
                               int(id_offset), _p(scores), _p(ids), _stream()))
    return scores, ids


def merge_topk(scores: torch.Tensor, ids: torch.Tensor, k: int):
    """Merge G per-shard sorted lists [G, nq, kin] (global ids) into the
    (score, id)-first k per query."""
    G, nq, kin = scores.shape
    out_s = torch.empty((nq, k), dtype=torch.float64, device=scores.device)
    out_i = torch.empty((nq, k), dtype=torch.int32, device=scores.device)
    check(lib.qa_merge_topk(_p(scores.contiguous()), _p(ids.contiguous()), G, nq, kin, k,
                            _p(out_s), _p(out_i), _stream()))
    return out_s, out_i


def debug_dots(db: DeviceCodes, q: DeviceCodes, impl: int = 0) -> torch.Tensor:
    """Full int32 dot matrix [nq, n] through one unfiltered pass
    (impl 0 = tcgen05 tensor cores, 1 = dp4a CUDA cores)."""
    out = torch.empty((q.n, db.n), dtype=torch.int32, device=db.device)
    check(lib.qa_debug_dots_i8(_p(db.codes), db.n, _p(q.codes), q.n, db.d, int(impl), _p(out),
                               _stream()))
    return out
