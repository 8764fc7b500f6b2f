"""estimate_stats on the GPU (csrc/qa_stats.cu) against the reference's own
outputs (tests/golden/stats_cases.npz, made by tests/golden/make_golden.py
from quantann.quantizer.estimate_stats on the same seeded inputs): every
statistic bit-exact, and the fitted windows of all three modes equal."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_08919_b200 as qa  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(GOLDEN))
from make_golden import stats_inputs  # noqa: E402


def _cases():
    z = np.load(GOLDEN / "stats_cases.npz")
    out = {}
    for key in z.files:
        name, field = key.split("__", 1)
        out.setdefault(name, {})[field] = z[key]
    return out


CASES = _cases()
INPUTS = dict(stats_inputs()[0])


@pytest.mark.parametrize("name", sorted(CASES))
def test_estimate_stats_bit_exact(name):
    g = CASES[name]
    x = INPUTS[name]
    st = qa.estimate_stats(qa.DenseDataset(x))
    for f in ("mu", "sigma", "min", "max", "trimmed_absmax"):
        np.testing.assert_array_equal(getattr(st, f), g[f], err_msg=f"{name}.{f}")
    np.testing.assert_array_equal([st.pooled_mu, st.pooled_sigma], g["pooled"], err_msg=name)
    assert st.count == x.shape[0]
    for mode in (qa.QuantMode.SIGMA_CLAMP, qa.QuantMode.ABS_MAX, qa.QuantMode.UNIFORM_SIGMA_CLAMP):
        key = f"fit{int(mode)}"
        if key in g:
            p = qa.fit(st, 8, mode).params
            np.testing.assert_array_equal(np.stack([p.k, p.sb, p.se]), g[key],
                                          err_msg=f"{name}.{key}")


def test_estimate_stats_errors():
    with pytest.raises(qa.TooFewSamples):
        qa.estimate_stats(qa.DenseDataset(np.zeros((1, 3), np.float32)))
    with pytest.raises(qa.ElementKindMismatch):
        qa.estimate_stats(qa.DenseDataset(np.zeros((4, 3), np.int8)))
