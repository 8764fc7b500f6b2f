"""Files straight into HBM: row shards of fvecs / i8vecs / bvecs land on the
device byte-for-byte (header-stripping DMA), with zero pad columns and the
code norms of the encode path."""

from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2110_08919_b200 as qa  # noqa: E402
from paper_2110_08919_b200 import vecs_io  # noqa: E402


def test_fvecs_shards_to_device(tmp_path, monkeypatch):
    monkeypatch.setenv("QA_B200_VECS_CHUNK", str(1 << 16))  # many staging chunks
    rng = np.random.default_rng(3)
    x = rng.normal(size=(70_001, 33)).astype(np.float32)
    vecs_io.save_fvecs(qa.DenseDataset(x), tmp_path / "x.fvecs")
    parts = []
    for rank in range(4):
        t, lo, n = vecs_io.load_fvecs_to_device(tmp_path / "x.fvecs", rank, 4)
        assert n == 70_001
        parts.append(t.cpu().numpy())
    np.testing.assert_array_equal(np.concatenate(parts), x)


def test_i8vecs_and_bvecs_to_device_codes(tmp_path, oracle, monkeypatch):
    monkeypatch.setenv("QA_B200_VECS_CHUNK", str(10_000))
    rng = np.random.default_rng(4)
    c = rng.integers(-128, 128, size=(5000, 100)).astype(np.int8)
    vecs_io.save_i8vecs(qa.DenseDataset(c), tmp_path / "c.i8vecs")
    dc, lo, n = vecs_io.load_i8vecs_to_device(tmp_path / "c.i8vecs")
    assert (lo, n) == (0, 5000) and dc.ld == 128
    np.testing.assert_array_equal(dc.to_host(), c)
    assert not dc.codes[:, 100:].cpu().numpy().any()
    np.testing.assert_array_equal(dc.norm.cpu().numpy(), oracle.norms_i8(c))
    # bvecs: the same bytes written unsigned (v + 128) load back as c
    raw = (c.astype(np.int16) + 128).astype(np.uint8)
    hdr = np.full((5000, 1), 100, "<i4").view(np.uint8)
    (tmp_path / "c.bvecs").write_bytes(np.concatenate([hdr, raw], axis=1).tobytes())
    db, _, _ = vecs_io.load_bvecs_to_device(tmp_path / "c.bvecs", 1, 2)
    np.testing.assert_array_equal(db.to_host(), c[2500:])
    np.testing.assert_array_equal(vecs_io.load_bvecs(tmp_path / "c.bvecs").data, c)
    # a search over the file-loaded codes equals the host path
    q = c[:7].copy()
    from paper_2110_08919_b200 import device as dev
    qs = dev.DeviceCodes.from_host(q)
    s1, i1 = dev.scan_topk(dc, qs, 10, 1)
    s2, i2 = oracle.scan_topk_i8(c, q, 10, 1)
    np.testing.assert_array_equal(i1.cpu().numpy(), i2)
    np.testing.assert_array_equal(s1.cpu().numpy(), s2)
