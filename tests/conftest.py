"""Shared fixtures.  ``-m gpu`` tests need a CUDA device and exercise the
libqa_b200 kernels; everything else runs on CPU (oracle vs golden vectors,
host logic, C-ABI exports, gloo multi-process plumbing)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and runs the kernels")


def _split(npz):
    cases = {}
    for key in npz.files:
        name, field = key.split("__", 1)
        cases.setdefault(name, {})[field] = npz[key]
    return cases


@pytest.fixture(scope="session")
def golden_encode():
    return _split(np.load(GOLDEN / "encode_cases.npz"))


@pytest.fixture(scope="session")
def golden_scan():
    return _split(np.load(GOLDEN / "scan_cases.npz"))


@pytest.fixture(scope="session")
def golden_scan_f32():
    return _split(np.load(GOLDEN / "scan_f32_cases.npz"))


@pytest.fixture(scope="session")
def golden_cfg():
    return _split(np.load(GOLDEN / "cfg_minis.npz"))


@pytest.fixture(scope="session")
def oracle():
    from oracle import qa_oracle

    qa_oracle.lib()  # built by __graft_entry__.build() / make -C oracle
    return qa_oracle
