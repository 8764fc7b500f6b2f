"""Command-line front end (reference cli.py fit / quantize / gt; tests modelled
on reference tests/test_cli.py): files, stdout lines and exit codes."""

from __future__ import annotations

import subprocess
import sys

import numpy as np
import pytest

from paper_2110_08919_b200 import DenseDataset, load_i8vecs, load_ivecs, save_fvecs
from paper_2110_08919_b200.cli import main

N, D, NQ = 300, 8, 10


@pytest.fixture(scope="module")
def workdir(tmp_path_factory):
    root = tmp_path_factory.mktemp("cli")
    rng = np.random.default_rng(0)
    save_fvecs(DenseDataset(rng.uniform(-0.1, 0.1, size=(N, D)).astype(np.float32)),
               root / "corpus.fvecs")
    save_fvecs(DenseDataset(rng.uniform(-0.1, 0.1, size=(NQ, D)).astype(np.float32)),
               root / "queries.fvecs")
    return root


def test_unknown_flag_exits_2(workdir):
    with pytest.raises(SystemExit) as exc:
        main(["fit", "--input", str(workdir / "corpus.fvecs"), "--frobnicate"])
    assert exc.value.code == 2


def test_no_subcommand_exits_2():
    with pytest.raises(SystemExit) as exc:
        main([])
    assert exc.value.code == 2


def test_missing_input_exits_1(tmp_path, capsys):
    rc = main(["fit", "--input", str(tmp_path / "nope.fvecs"), "--out", str(tmp_path / "x.qzp")])
    assert rc == 1
    capsys.readouterr()


def test_module_entry_point_help():
    proc = subprocess.run([sys.executable, "-m", "paper_2110_08919_b200", "--help"],
                          capture_output=True, text=True, timeout=120)
    assert proc.returncode == 0
    for name in ("fit", "quantize", "gt"):
        assert name in proc.stdout


@pytest.mark.gpu
def test_fit_quantize_gt_pipeline(workdir, oracle, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    params = workdir / "params.qzp"
    assert main(["fit", "--input", str(workdir / "corpus.fvecs"), "--bits", "8",
                 "--mode", "absmax", "--out", str(params)]) == 0
    assert "fit d=8 bits=8 mode=absmax" in capsys.readouterr().out
    codes = workdir / "corpus.i8vecs"
    assert main(["quantize", "--input", str(workdir / "corpus.fvecs"), "--params", str(params),
                 "--out", str(codes)]) == 0
    assert codes.stat().st_size == N * (4 + D)
    first = codes.read_bytes()
    assert main(["quantize", "--input", str(workdir / "corpus.fvecs"), "--params", str(params),
                 "--out", str(codes)]) == 0
    assert codes.read_bytes() == first  # deterministic re-run
    # the codes are the reference encode of the fitted window
    from paper_2110_08919_b200 import load_dataset, load_params

    p = load_params(params)
    X = load_dataset(workdir / "corpus.fvecs").data
    np.testing.assert_array_equal(load_i8vecs(codes).data, oracle.encode(X, p.k, p.sb, p.se, 8))
    gt_path = workdir / "gt.ivecs"
    assert main(["gt", "--corpus", str(workdir / "corpus.fvecs"),
                 "--queries", str(workdir / "queries.fvecs"), "--k", "10", "--metric", "l2",
                 "--out", str(gt_path)]) == 0
    assert f"ground truth {NQ} queries k=10" in capsys.readouterr().out
    gt = load_ivecs(gt_path)
    Q = load_dataset(workdir / "queries.fvecs").data
    _, want = oracle.scan_topk_f32(X, Q, 10, 1)
    np.testing.assert_array_equal(gt.ids, want)
    # int8 ground truth over the quantized files
    qcodes = workdir / "queries.i8vecs"
    assert main(["quantize", "--input", str(workdir / "queries.fvecs"), "--params", str(params),
                 "--out", str(qcodes)]) == 0
    assert main(["gt", "--corpus", str(codes), "--queries", str(qcodes), "--k", "7",
                 "--metric", "ip", "--out", str(gt_path)]) == 0
    Xc, Qc = load_i8vecs(codes).data, load_i8vecs(qcodes).data
    _, want = oracle.scan_topk_i8(Xc, Qc, 7, 0)
    np.testing.assert_array_equal(load_ivecs(gt_path).ids, want)
    capsys.readouterr()


@pytest.mark.gpu
def test_validation_failures_exit_2(workdir, tmp_path, capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    assert main(["fit", "--input", str(workdir / "corpus.fvecs"), "--bits", "9",
                 "--out", str(tmp_path / "p.qzp")]) == 2
    params = tmp_path / "p.qzp"
    assert main(["fit", "--input", str(workdir / "corpus.fvecs"), "--out", str(params)]) == 0
    rng = np.random.default_rng(1)
    save_fvecs(DenseDataset(rng.uniform(-1, 1, size=(5, D + 3)).astype(np.float32)),
               tmp_path / "wide.fvecs")
    assert main(["quantize", "--input", str(tmp_path / "wide.fvecs"), "--params", str(params),
                 "--out", str(tmp_path / "w.i8vecs")]) == 2
    data = DenseDataset(np.array([[1.0, 0.0], [0.0, 0.0]], dtype=np.float32))
    save_fvecs(data, tmp_path / "z.fvecs")
    assert main(["gt", "--corpus", str(tmp_path / "z.fvecs"), "--queries", str(tmp_path / "z.fvecs"),
                 "--k", "1", "--normalize", "--out", str(tmp_path / "z.ivecs")]) == 2
    one = DenseDataset(np.array([[1.0, 2.0, 3.0]], dtype=np.float32))
    save_fvecs(one, tmp_path / "one.fvecs")
    assert main(["gt", "--corpus", str(tmp_path / "one.fvecs"),
                 "--queries", str(tmp_path / "one.fvecs"), "--k", "1",
                 "--out", str(tmp_path / "one.ivecs")]) == 0
    assert load_ivecs(tmp_path / "one.ivecs").ids.tolist() == [[0]]
    capsys.readouterr()
