"""Benchmark: int8 exhaustive k=100 search on the BASELINE config-1 workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config 1] [--nq 10000] [--n N]

Workload (BASELINE.json configs[1], the config the metric is quoted on):
1,000,000 x 100 fp32 database (GloVe-like generator, rows L2-normalised),
10,000 queries, symmetric per-dimension int8 quantization, angular
distance, k = 100.  Synthetic data from paper_2110_08919_b200.synth (seed 1).

One STEP = one pass of the hot path over the whole 10,000-query set:
encode the fp32 queries with the corpus window (encode kernel), then the
tensor-core exhaustive scan with exact top-k (filter + select kernels); the
int8 database index (codes + norms) is resident in HBM, built once before
timing.  ``value`` is queries/s with the fp32 queries already in HBM;
``e2e`` is the same through the host-buffer public path: pinned fp32
queries -> H2D -> encode -> scan -> D2H of ids + scores, all inside the
timed region.  L2 is flushed (256 MiB write) before every timed step,
outside the step's CUDA events.

N > 1 (torchrun): the database is row-sharded over the ranks, queries are
replicated, each rank scans its shard and the per-rank top-k lists are
all-gathered over NCCL and merged on the GPU (``sharded.py``).  Step time =
max over ranks of the CUDA-event time.

``--impl reference``: the reference's own CPU kernel (quantann._core
scan_topk compiled from /root/reference into oracle/_ref) on all host cores
(forked workers over query slices), each step a bounded query sample.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC_NAME = "int8 exhaustive k=100 queries/s at 1/2/4/8 B200; % of INT8 TC / HBM roofline"
PEAKS_PATH = ROOT / "MEASURED_PEAKS.json"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def load_peaks():
    if PEAKS_PATH.exists():
        return json.loads(PEAKS_PATH.read_text()), "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------- workload --

def make_workload(cfg: int, n: int | None, nq: int | None):
    from paper_2110_08919_b200 import synth

    c = dict(synth.CONFIGS[cfg])
    X, Q = synth.generate(cfg, n=n, nq=nq)
    c["n"], c["nq"] = X.shape[0], Q.shape[0]
    return c, X, Q


def workload_desc(c, k):
    metric = ("ip", "l2", "angular")[c["metric"]]
    return (f"{c['name']}: {c['n']}x{c['d']} fp32 db -> int8 ({c['calibration']}), "
            f"{c['nq']} queries, {metric}, k={k}")


# ---------------------------------------------------------- CPU reference --

_REF = {}


def _ref_worker(span):
    lo, hi = span
    qn = _REF["qn"][lo:hi] if _REF["qn"] is not None else None
    _REF["core"].scan_topk(_REF["Xc"], _REF["Qc"][lo:hi], _REF["k"], _REF["metric"], _REF["xn"],
                           qn)
    return hi - lo


class CpuReference:
    """The reference's compiled kernel (quantann._core.scan_topk, built from
    /root/reference into oracle/_ref) on all host cores: one forked worker
    per core, each scanning a contiguous query slice of the sample."""

    def __init__(self, c, X, Q, k):
        import multiprocessing as mp

        from oracle import qa_oracle as o

        core = o.ref_core()
        if core is None:
            raise RuntimeError("oracle/_ref reference _core missing (run build() in the dev box)")
        mn, mx = o.minmax(X)
        if c["calibration"] == "symmetric":
            kk, sb, se = o.fit_range(np.zeros_like(mn), np.maximum(np.abs(mn), np.abs(mx)))
        else:
            kk, sb, se = o.fit_range((mn + mx) / 2.0, (mx - mn) / 2.0)
        Xc = o.encode(X, kk, sb, se, 8)
        Qc = o.encode(Q, kk, sb, se, 8)
        metric = c["metric"]
        _REF.update(core=core, Xc=Xc, Qc=Qc, k=k, metric=metric,
                    xn=core.norms(Xc) if metric == 2 else None,
                    qn=core.norms(Qc) if metric == 2 else None)
        self.nq = Qc.shape[0]
        self.cores = os.cpu_count() or 1
        self.pool = mp.get_context("fork").Pool(self.cores)
        self.cursor = 0

    def step(self, sample: int) -> float:
        """Scan `sample` queries (rotating through the query set) on all
        cores; returns wall seconds."""
        lo = self.cursor % self.nq
        hi = min(self.nq, lo + sample)
        self.cursor = hi
        per = -(-(hi - lo) // self.cores)
        spans = [(i, min(hi, i + per)) for i in range(lo, hi, per)]
        t0 = time.perf_counter()
        done = sum(self.pool.map(_ref_worker, spans))
        dt = time.perf_counter() - t0
        assert done == hi - lo
        self.last = hi - lo
        return dt

    def close(self):
        self.pool.close()
        self.pool.join()


def reference_sample_size(c, cores: int, seconds: float) -> int:
    """Queries per sample so the reference spends ~`seconds` of wall time.
    Single-thread int8 scan rate measured in the survey: ~25e6 rows/s."""
    per_query = c["n"] / 25e6 * (c["d"] / 100.0)
    return int(max(cores, min(c["nq"], seconds * cores / max(per_query, 1e-6))))


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- GPU arm --

def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2110_08919_b200 as qa
    from paper_2110_08919_b200 import _lib, device as dev, sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_src = load_peaks()

    c, X, Q = make_workload(args.config, args.n, args.nq)
    n, d, nq, k = c["n"], c["d"], c["nq"], args.k
    metric = qa.Metric(c["metric"])

    # ---- index build (not timed): calibrate on the full corpus, encode this
    # rank's shard.  Calibration is per-dimension min/max -- exact and
    # order-free -- so every rank derives the identical window.
    x_full = torch.from_numpy(X).cuda()
    stats = qa.minmax_stats(x_full)
    fr = qa.fit_symmetric(stats) if c["calibration"] == "symmetric" else qa.fit_minmax(stats)
    lo, hi = sharded.shard_bounds(n, world, rank)
    index = qa.Int8Index.from_params(x_full[lo:hi].contiguous(), fr.params, metric, id_offset=lo)
    del x_full
    q_dev = torch.from_numpy(Q).cuda()
    q_host = torch.from_numpy(Q).pin_memory()
    qcodes = dev.DeviceCodes.empty(nq, d)
    keff = min(k, n)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def search_step(queries_dev):
        index.encode_queries(queries_dev, out=qcodes)
        if world == 1:
            return index.search_codes(qcodes, k)
        return sharded.sharded_search(lambda off: index.search_codes(qcodes, k), n, k)

    def timed(fn, steps, e2e=False):
        times, launches = [], 0
        for _ in range(steps):
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            fn()
            ev1.record(stream)
            torch.cuda.synchronize()
            ms = ev0.elapsed_time(ev1)
            if world > 1:
                t = torch.tensor([ms], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            times.append(ms)
            st = _lib.last_scan_stats()
            launches += 1 + st["launches"] + (1 if world > 1 else 0)
        return times, launches

    out_host = (torch.empty((nq, keff), dtype=torch.float64).pin_memory(),
                torch.empty((nq, keff), dtype=torch.int32).pin_memory())

    def e2e_step():
        qd = q_host.to("cuda", non_blocking=True)
        s, i = search_step(qd)
        out_host[0].copy_(s, non_blocking=True)
        out_host[1].copy_(i, non_blocking=True)

    # warm-up
    for _ in range(max(3, args.warmup)):
        search_step(q_dev)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    _lib.set_profiling(True)
    step_ms, launches = timed(lambda: search_step(q_dev), args.steps)
    st = _lib.last_scan_stats()   # last step's kernel-level event timings
    _lib.set_profiling(False)
    clk = clocks.stop()

    e2e = None
    if not args.no_e2e:
        for _ in range(2):
            e2e_step()
        e2e_ms, _ = timed(e2e_step, args.steps, e2e=True)
        e2e = {"value": nq / (float(np.mean(e2e_ms)) / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": int(nq * d * 4),
               "d2h_bytes_per_step": int(nq * keff * (8 + 4)),
               "ms_per_step": float(np.mean(e2e_ms))}

    # correctness spot check of the last result on a few queries (oracle);
    # outside every timed region
    parity = None
    if rank == 0 and world == 1:
        try:
            from oracle import qa_oracle as o

            s, i = index.search_codes(qcodes, k)
            sub = min(8, nq)
            Xc = index.codes_in_input_order()
            Qc = qcodes.to_host()[:sub]
            osc, oids = o.scan_topk_i8(Xc, Qc, k, int(metric), o.norms_i8(Xc), o.norms_i8(Qc))
            parity = {"queries_checked": sub,
                      "ids_equal": bool(np.array_equal(i[:sub].cpu().numpy(), oids)),
                      "scores_equal": bool(np.array_equal(s[:sub].cpu().numpy(), osc))}
        except Exception as exc:  # pragma: no cover
            parity = {"error": str(exc)[:200]}

    ms = float(np.mean(step_ms))
    value = nq / (ms / 1e3)
    # roofline of the dominant kernel (the fused tcgen05 filter pass):
    # algorithmic ops = 2 * nq * rows * d (unpadded d) per launch, divided by
    # the CUDA-event time of those launches on their stream.
    peak_tops = 2.0 * float(peaks["bf16_tflops"])
    # DRAM traffic of the dominant launch (the final, estimated-bound pass)
    # from the committed ncu --set full capture of this workload; compare to
    # its algorithmic bytes (the database rows it scans, once)
    traffic, traffic_note = None, "no committed ncu capture"
    tfile = ROOT / "profiles" / "r01_filter_traffic.json"
    if tfile.exists() and args.config == 1 and args.n is None and args.nq is None:
        tj = json.loads(tfile.read_text())
        traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
        traffic_note = (f"bytes per launch of the final filter pass ({tj['source']}); "
                        f"algorithmic bytes {tj['algorithmic_db_bytes']}")
    achieved = (st["filter_ops"] / (st["filter_ms"] / 1e3) / 1e12) if st["filter_ms"] > 0 else None
    roofline = {
        "bound": "tensor", "kernel": "filter_tc_kernel (tcgen05 kind::i8 + fused threshold top-k epilogue)",
        "achieved": achieved, "peak": peak_tops, "unit": "TOP/s",
        "frac": (achieved / peak_tops) if achieved else None,
        "peak_source": f"2 x dense bf16 {peaks_src} (int8 dense = 2x bf16 on B200; "
                       f"spec 4500 TOP/s)",
        "frac_of_spec_4500": (achieved / 4500.0) if achieved else None,
        "traffic": traffic,
        "traffic_note": traffic_note,
        "filter_ms_per_step": st["filter_ms"], "select_ms_per_step": st["select_ms"],
        "filter_launches_per_step": st["filter_launches"],
        "filter_share_of_step": st["filter_ms"] / ms if ms else None,
        "scan_stats": {key: st[key] for key in ("rounds", "launches", "retries", "candidates")},
    }
    line = {
        "metric": METRIC_NAME, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": f"synthetic (paper_2110_08919_b200.synth config {args.config}, seed {c['seed']})",
        "config": {"workload": workload_desc(c, k), "n": n, "d": d, "nq": nq, "k": k,
                   "metric": metric.short_name, "calibration": c["calibration"],
                   "parallelism": f"row-shard x{world}, queries replicated, NCCL all-gather of "
                                  f"top-k" if world > 1 else "single GPU",
                   "l2": "flushed (256 MiB write) before every timed step"},
        "database_vectors_per_s": value * n,
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "parity_spot_check": parity,
        "impl": "b200",
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ref = CpuReference(c, X, Q, k)
            sample = reference_sample_size(c, ref.cores, 15.0)
            secs = ref.step(sample)
            sample = ref.last
            ref.close()
            line["cpu_baseline"] = {"value": sample / secs, "unit": "queries/s", "cores": ref.cores,
                                    "kind": "reference",
                                    "sample": f"{sample} of the {nq} queries against the full "
                                              f"{n}x{d} int8 db (reference _core.scan_topk, "
                                              f"{ref.cores} forked workers)"}
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    c, X, Q = make_workload(args.config, args.n, args.nq)
    k = args.k
    ref = CpuReference(c, X, Q, k)
    sample = reference_sample_size(c, ref.cores, 8.0)
    for _ in range(args.warmup):
        ref.step(min(sample, ref.cores))
    secs = [ref.step(sample) for _ in range(args.steps)]
    sample = ref.last
    ref.close()
    value = sample / float(np.mean(secs))
    line = {
        "metric": METRIC_NAME, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(secs)) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": f"synthetic (paper_2110_08919_b200.synth config {args.config}, seed {c['seed']})",
        "config": {"workload": workload_desc(c, k), "n": c["n"], "d": c["d"], "nq": c["nq"],
                   "k": k, "metric": ("ip", "l2", "angular")[c["metric"]],
                   "calibration": c["calibration"], "parallelism": "host cores (forked workers)"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": ref.cores,
                         "kind": "reference",
                         "sample": f"{sample} queries per step against the full {c['n']}x{c['d']} "
                                   f"int8 db (reference quantann._core.scan_topk)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
