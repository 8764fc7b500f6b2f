"""Encode throughput (fp32 -> int8 codes + norms) on device-resident rows.
usage: bench_encode.py [d ...]   (algorithmic bytes: 4 n d + n ld + 8 n)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2110_08919_b200 import device as dev

dims = [int(v) for v in sys.argv[1:]] or [100, 128, 256]
peak = 6540.8
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
for d in dims:
    n = (2 << 30) // (4 * d)  # 2 GiB of fp32
    g = torch.Generator(device="cuda"); g.manual_seed(d)
    x = torch.randn(n, d, device="cuda", generator=g)
    mn, mx = dev.minmax(x)
    k = (mn + mx) / 2
    out = dev.DeviceCodes.empty(n, d, x.device)
    for _ in range(3):
        dev.encode(x, k, mn, mx, 8, out=out)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(10):
        ev[0].record(); dev.encode(x, k, mn, mx, 8, out=out); ev[1].record()
        torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
    ms = sorted(ts)[len(ts) // 2]
    by = 4 * n * d + n * out.ld + 8 * n
    print(json.dumps({"d": d, "n": n, "ms": ms, "GBps": by / ms / 1e6, "frac_hbm": by / ms / 1e6 / peak}), flush=True)
