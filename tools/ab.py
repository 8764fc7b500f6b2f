"""A/B timing of library builds / env knobs on one box.

    python tools/ab.py 'old:QA_B200_LIB=abtest/old/paper_2110_08919_b200/libqa_b200.so' 'new:' ...

Each variant runs `bench.py --steps 5 --warmup 3` (no cpu baseline, no e2e)
twice, interleaved, and prints value / filter / select ms per step.
"""
import json
import os
import subprocess
import sys

extra = os.environ.get("AB_ARGS", "").split()
variants = []
for spec in sys.argv[1:]:
    tag, _, envs = spec.partition(":")
    env = dict(os.environ)
    for kv in envs.split():
        k, _, v = kv.partition("=")
        env[k] = v
    variants.append((tag, env))
for rep in range(int(os.environ.get("AB_REPS", "2"))):
    for tag, env in variants:
        p = subprocess.run([sys.executable, "bench.py", "--steps", "5", "--warmup", "3",
                            "--no-cpu-baseline", "--no-e2e", *extra],
                           env=env, capture_output=True, text=True, timeout=600)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
            r = d["roofline"]
            print(f"{tag:12s} rep{rep} q/s={d['value']:.0f} ms={d['ms_per_step']:.3f} "
                  f"filter={r['filter_ms_per_step']:.3f} select={r['select_ms_per_step']:.3f} "
                  f"sm_mhz={d.get('clocks', {}).get('sm_mhz')} parity={d.get('parity_spot_check')}",
                  flush=True)
        except Exception as e:  # noqa: BLE001
            print(tag, "FAILED", e, p.stdout[-500:], p.stderr[-1500:], flush=True)
