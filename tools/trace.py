"""Per-round survivor trace of one search on a bench configuration.

    QA_B200_TRACE=1 python tools/trace.py [--config 1] [--k 100]

Prints the library's qa_trace lines (rows scanned per round, mode, valid
candidates reaching select) plus per-round filter/select times from a
separate profiled run.  Diagnostics only; not part of the product.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))

import torch  # noqa: E402

import paper_2110_08919_b200 as qa  # noqa: E402
import synth  # noqa: E402
from paper_2110_08919_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--nq", type=int, default=None)
    args = ap.parse_args()
    c = synth.CONFIGS[args.config]
    X, Q = synth.generate(args.config, nq=args.nq)
    x = torch.from_numpy(X).cuda()
    stats = qa.minmax_stats(x)
    fr = qa.fit_symmetric(stats) if c["calibration"] == "symmetric" else qa.fit_minmax(stats)
    index = qa.Int8Index.from_params(x, fr.params, qa.Metric(c["metric"]))
    qc = index.encode_queries(torch.from_numpy(Q).cuda())
    index.search_codes(qc, args.k)  # warm
    torch.cuda.synchronize()
    print("---- traced search", flush=True)
    index.search_codes(qc, args.k)
    torch.cuda.synchronize()
    st = _lib.last_scan_stats()
    print({k: st[k] for k in ("rounds", "candidates", "retries")}, flush=True)


if __name__ == "__main__":
    main()
