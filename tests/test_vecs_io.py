"""Vector-file and params formats (reference dataset.py:160-275,
quantizer.py:330-369) through the native reader/writer of libqa_b200.
Pinned on tests/golden/vecs_cases.npz (outcomes of the reference's own
loaders on the same bytes).  Host-only: no GPU calls."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

import paper_2110_08919_b200 as qa
from paper_2110_08919_b200 import _lib, errors, vecs_io

GOLDEN = Path(__file__).resolve().parent / "golden" / "vecs_cases.npz"
LOADERS = {"fvecs": vecs_io.load_fvecs, "ivecs": vecs_io.load_ivecs,
           "i8vecs": vecs_io.load_i8vecs, "bvecs": vecs_io.load_bvecs}


def _cases():
    z = np.load(GOLDEN)
    cases = {}
    for key in z.files:
        name, field = key.split("__", 1)
        cases.setdefault(name, {})[field] = z[key]
    return cases


@pytest.mark.parametrize("name", sorted(_cases()))
def test_loaders_match_reference_outcomes(tmp_path, name):
    c = _cases()[name]
    kind = str(c["kind"])
    path = tmp_path / f"{name}.{kind}"
    path.write_bytes(c["blob"].tobytes())
    if "error" in c:
        err = str(c["error"])
        cls = ValueError if err == "ValueError" else getattr(errors, err)
        with pytest.raises(cls) as ei:
            LOADERS[kind](path)
        assert str(ei.value) == str(c["message"]).replace("{path}", str(path))
    else:
        out = LOADERS[kind](path)
        got = out.ids if kind == "ivecs" else out.data
        assert got.dtype == c["out"].dtype and got.shape == c["out"].shape
        np.testing.assert_array_equal(got.view(np.uint8), c["out"].view(np.uint8))
        assert not got.flags.writeable


def test_missing_file_is_oserror(tmp_path):
    with pytest.raises(FileNotFoundError):
        vecs_io.load_fvecs(tmp_path / "nope.fvecs")


def test_round_trips(tmp_path):
    rng = np.random.default_rng(0)
    f = qa.DenseDataset(rng.normal(size=(1234, 37)).astype(np.float32))
    vecs_io.save_fvecs(f, tmp_path / "a.fvecs")
    assert vecs_io.load_fvecs(tmp_path / "a.fvecs") == f
    b = qa.DenseDataset(rng.integers(-128, 128, size=(999, 100)).astype(np.int8))
    vecs_io.save_i8vecs(b, tmp_path / "a.i8vecs")
    assert vecs_io.load_i8vecs(tmp_path / "a.i8vecs") == b
    g = qa.GroundTruth(np.argsort(rng.random((50, 300)), axis=1)[:, :20].astype(np.int32))
    vecs_io.save_ivecs(g, tmp_path / "a.ivecs")
    assert vecs_io.load_ivecs(tmp_path / "a.ivecs") == g
    # an empty dataset writes an empty file, which loads as (0, 0)
    vecs_io.save_fvecs(qa.DenseDataset(np.empty((0, 5), np.float32)), tmp_path / "e.fvecs")
    assert vecs_io.load_fvecs(tmp_path / "e.fvecs").data.shape == (0, 0)
    with pytest.raises(qa.ElementKindMismatch):
        vecs_io.save_fvecs(b, tmp_path / "x.fvecs")
    with pytest.raises(qa.ElementKindMismatch):
        vecs_io.save_i8vecs(f, tmp_path / "x.i8vecs")


def test_row_range_reads_are_shards(tmp_path):
    rng = np.random.default_rng(1)
    x = rng.normal(size=(1001, 9)).astype(np.float32)
    vecs_io.save_fvecs(qa.DenseDataset(x), tmp_path / "s.fvecs")
    parts = []
    for rank in range(3):
        lo, hi = vecs_io.shard_rows(1001, 3, rank)
        out = np.full((hi - lo, 16), -7.0, np.float32)   # padded destination stride
        _lib.check(_lib.lib.qa_vecs_read(str(tmp_path / "s.fvecs").encode(), 4, 9, lo, hi,
                                         out.ctypes.data, 64, 0, 0, None))
        assert (out[:, 9:] == -7.0).all()
        parts.append(out[:, :9])
    np.testing.assert_array_equal(np.concatenate(parts), x)


def test_params_round_trip_and_errors(tmp_path):
    p = qa.QuantizerParams(bits=6, mode=qa.QuantMode.SIGMA_CLAMP,
                           k=np.float32([0.0, -1.5, 3e-39]), sb=np.float32([-1, -2, 0]),
                           se=np.float32([1, np.nextafter(np.float32(-2), np.float32(0)), 1e-38]))
    vecs_io.save_params(p, tmp_path / "p.qzp")
    raw = (tmp_path / "p.qzp").read_bytes()
    assert raw[:4] == b"QZP1" and len(raw) == 12 + 12 * 3
    assert vecs_io.load_params(tmp_path / "p.qzp") == p
    (tmp_path / "bad.qzp").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(qa.BadMagic):
        vecs_io.load_params(tmp_path / "bad.qzp")
    (tmp_path / "v.qzp").write_bytes(raw[:4] + b"\x02" + raw[5:])
    with pytest.raises(qa.UnsupportedVersion):
        vecs_io.load_params(tmp_path / "v.qzp")
    (tmp_path / "m.qzp").write_bytes(raw[:6] + b"\x09" + raw[7:])
    with pytest.raises(qa.UnsupportedVersion):
        vecs_io.load_params(tmp_path / "m.qzp")
    (tmp_path / "t.qzp").write_bytes(raw[:-1])
    with pytest.raises(qa.TruncatedFile):
        vecs_io.load_params(tmp_path / "t.qzp")
    (tmp_path / "h.qzp").write_bytes(raw[:7])
    with pytest.raises(qa.TruncatedFile):
        vecs_io.load_params(tmp_path / "h.qzp")


def test_load_dataset_by_extension(tmp_path):
    x = qa.DenseDataset(np.arange(12, dtype=np.float32).reshape(3, 4))
    qa.save_fvecs(x, tmp_path / "a.FVECS")
    assert qa.load_dataset(tmp_path / "a.FVECS") == x
    with pytest.raises(ValueError, match="cannot infer dataset format"):
        qa.load_dataset(tmp_path / "a.ivecs")
