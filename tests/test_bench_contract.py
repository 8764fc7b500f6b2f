"""bench.py's reference arm (the reference's compiled kernel on host cores)
keeps the driver's JSON contract; runs on CPU at a reduced size."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    from oracle import qa_oracle
    if qa_oracle.ref_core() is None:
        pytest.skip("reference _core not built here (make -C oracle ref)")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--n", "20000",
                        "--nq", "64", "--steps", "2", "--warmup", "1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["unit"] == "queries/s" and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["n"] == 20000 and line["config"]["nq"] == 64
