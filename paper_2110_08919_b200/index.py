"""Device-resident quantized index: the serving form of the hot path.

``Int8Index.build`` calibrates (GPU min/max), fits the window on the host
(O(d), reference ``fit``), encodes the fp32 database into int8 codes plus
norms in HBM, and keeps the float32 window constants on the device so
queries are encoded by the same kernel with the corpus parameters
(reference quantizer.py:312-320, bench.py:200-202).  ``search`` encodes a
query batch and runs the tensor-core scan; nothing leaves the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as dev
from .distances import Metric
from .quantizer import FitResult, QuantizerParams, fit_minmax, fit_symmetric, minmax_stats


@dataclass
class Int8Index:
    params: QuantizerParams
    metric: Metric
    codes: dev.DeviceCodes
    k_dev: torch.Tensor
    sb_dev: torch.Tensor
    se_dev: torch.Tensor
    id_offset: int = 0

    @property
    def n(self) -> int:
        return self.codes.n

    @property
    def d(self) -> int:
        return self.codes.d

    @classmethod
    def from_params(cls, x: torch.Tensor, params: QuantizerParams, metric: Metric,
                    id_offset: int = 0, sort_rows: bool = True) -> "Int8Index":
        """Encode ``x`` with ``params``.  The stored rows are ordered for the
        scan (ids still report positions in ``x``): narrow per-unit filter
        bounds, and a threshold-estimate sample (every stride-th tile) that
        spans the whole index."""
        device = x.device
        k, sb, se = (torch.from_numpy(np.array(a, dtype=np.float32)).to(device)
                     for a in (params.k, params.sb, params.se))
        codes = dev.encode(x, k, sb, se, params.bits)
        metric = Metric(metric)
        if sort_rows:
            # L2 / angular: interleaved norm blocks (qa_layout.cu) -- every
            # 4096-row block is one narrow norm band, so work units have tight
            # bounds and the strided estimate sample meets every band.  Inner
            # product: a fixed pseudo-random order -- its bound does not use
            # norms, and norm order clusters the high-norm rows where the best
            # dots live (2.5x the candidates and failed estimates on cfg4).
            if metric == Metric.INNER_PRODUCT:
                codes = codes.shuffled()
            else:
                codes = codes.sorted_by_norm(stratify=False)
        return cls(params, metric, codes, k, sb, se, id_offset)

    def codes_in_input_order(self) -> np.ndarray:
        """int8 codes [n, d] in the order of the encoded input rows."""
        host = self.codes.to_host()
        if self.codes.ids is None:
            return host
        out = np.empty_like(host)
        out[self.codes.ids.cpu().numpy()] = host
        return out

    @classmethod
    def build(cls, x: torch.Tensor, metric: Metric, calibration: str = "minmax",
              bits: int = 8) -> "Int8Index":
        stats = minmax_stats(x)
        fr: FitResult = fit_symmetric(stats, bits) if calibration == "symmetric" \
            else fit_minmax(stats, bits)
        return cls.from_params(x, fr.params, metric)

    def encode_queries(self, q: torch.Tensor, out: dev.DeviceCodes | None = None):
        return dev.encode(q, self.k_dev, self.sb_dev, self.se_dev, self.params.bits, out=out)

    def search_codes(self, qc: dev.DeviceCodes, k: int, out=None, sync: bool | None = None):
        """Top-k of the query codes, (scores f64, ids i32) on the device.

        ``sync=False`` (the default for L2 and inner product) is the stream-
        ordered search: no host round trip, queries that need a recompute are
        redone on the device (qa_scan_topk_i8_async).  ``sync=True`` (the
        default for angular) also reports a zero code norm as ZeroNorm
        (checked on the device inside the scan, reference exact.py:67-69);
        callers that guarantee nonzero vectors may pass ``sync=False``."""
        if sync is None:
            sync = self.metric == Metric.ANGULAR
        return dev.scan_topk(self.codes, qc, k, int(self.metric), id_offset=self.id_offset,
                             out=out, sync=sync)

    def search(self, q: torch.Tensor, k: int):
        """fp32 query batch on the device -> (scores f64, ids i32) on the device."""
        return self.search_codes(self.encode_queries(q), k)
