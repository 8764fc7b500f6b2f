"""Benchmark: int8 exhaustive k=100 search, BASELINE config 2 by default.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--config 2] [--n N] [--nq NQ] [--batch B]

Workload (BASELINE.json configs[2], the config whose text carries the
metric's "1/2/4/8 B200"): a 1,000,000 x 128 fp32 database (SIFT-like law:
round(|N(0, 40^2)|) clipped to [0, 255], 10 % zeros), 10,000 queries of the
same law issued in batches of 1,024, per-dimension min/max int8
quantization, L2, k = 100.  Seeded synthetic data from ``synth.py`` (the
public SIFT set is not available offline).

One STEP = the whole 10,000-query set, batch after batch: encode the fp32
batch with the corpus window (encode kernel), then the tensor-core
exhaustive scan with exact top-k (filter + select kernels).  The int8 index
(codes + norms, norm-sorted layout) is built once before timing.

* ``value``: queries/s with the fp32 queries already in HBM;
* ``e2e``: the same through the public host-buffer path, per batch: pinned
  fp32 queries -> H2D -> encode -> scan -> D2H of scores + ids;
* ``e2e_reference_api``: the reference-shaped API
  ``batch_ground_truth(corpus, queries, k, metric)`` (reference
  exact.py:105-117) with host int8 DenseDatasets, per batch; the frozen
  corpus stays resident on the device between calls.

L2 is flushed (256 MiB write) before every timed step, outside its events.

N > 1 (torchrun): rows are sharded contiguously; each rank generates and
encodes only its own shard (calibration = NCCL MIN/MAX all-reduce of the
per-shard ranges, so every rank derives the identical window); queries are
replicated; per batch each rank scans its shard and the per-rank top-k lists
are all-gathered over NCCL and merged on the GPU (``sharded.py``).  Step
time = max over ranks of the CUDA-event time.

``--impl reference``: the reference's own CPU kernel (quantann._core
scan_topk compiled from /root/reference into oracle/_ref) on all host cores
(forked workers over query slices); each step scans a bounded sample of the
query set; value = queries scanned / seconds, summed over the timed steps.
This process never imports the B200 package or loads its library.
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
MMA_I8_TOPS = 4430.0  # tools/mma_rate.cu on this pool: 128 cycles per M128.N256.K32 kind::i8


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of a CUDA-graph replay of the step")
    return ap.parse_args()


def load_peaks():
    if PEAKS_PATH.exists():
        return json.loads(PEAKS_PATH.read_text()), "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload(args):
    import synth

    c = dict(synth.CONFIGS[args.config])
    if args.n is not None:
        c["n"] = args.n
    if args.nq is not None:
        c["nq"] = args.nq
    if args.batch is not None:
        c["batch"] = args.batch
    c["batch"] = min(c["batch"], c["nq"])
    return c


def workload_desc(c, k):
    metric = ("ip", "l2", "angular")[c["metric"]]
    return (f"{c['name']}: {c['n']}x{c['d']} fp32 db -> int8 ({c['calibration']}), "
            f"{c['nq']} queries in batches of {c['batch']}, {metric}, k={k}")


def batches(nq, B):
    return [(lo, min(nq, lo + B)) for lo in range(0, nq, B)]


# ---------------------------------------------------------- CPU reference --
#
# Only numpy, the C oracle (setup: the encode the reference's numpy
# quantizer performs, quantizer.py:291-300) and the reference's own compiled
# _core are used here -- never the B200 package.

_REF = {}


def _ref_worker(span):
    lo, hi = span
    qn = _REF["qn"][lo:hi] if _REF["qn"] is not None else None
    _REF["core"].scan_topk(_REF["Xc"], _REF["Qc"][lo:hi], _REF["k"], _REF["metric"], _REF["xn"], qn)
    return hi - lo


class CpuReference:
    """The reference's compiled kernel (quantann._core.scan_topk, built from
    /root/reference into oracle/_ref) on `procs` host cores: one forked
    worker per core, each scanning a contiguous query slice."""

    def __init__(self, c, X, Q, k, procs):
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
        self.procs = procs
        self.pool = mp.get_context("fork").Pool(procs) if procs > 1 else None
        self.cursor = 0

    def step(self, sample: int) -> tuple[int, float]:
        """Scan `sample` queries (a contiguous slice, rotating through the
        query set); returns (queries scanned, wall seconds)."""
        lo = self.cursor
        hi = min(self.nq, lo + sample)
        self.cursor = 0 if hi >= self.nq else hi
        t0 = time.perf_counter()
        if self.pool is None:
            done = _ref_worker((lo, hi))
        else:
            per = -(-(hi - lo) // self.procs)
            spans = [(i, min(hi, i + per)) for i in range(lo, hi, per)]
            done = sum(self.pool.map(_ref_worker, spans))
        dt = time.perf_counter() - t0
        assert done == hi - lo
        return done, dt

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def reference_sample(c, procs: int, seconds: float) -> int:
    """Queries per step so the reference spends about `seconds` of wall
    time (single-thread int8 scan rate measured in the survey: ~25e6
    rows/s at d=128)."""
    per_query = c["n"] / 25e6 * (c["d"] / 128.0)
    return int(max(procs, min(c["nq"], seconds * procs / max(per_query, 1e-9))))


def measure_reference(c, X, Q, k, procs, seconds, steps=1, warmup=0):
    ref = CpuReference(c, X, Q, k, procs)
    try:
        sample = reference_sample(c, procs, seconds)
        for _ in range(warmup):
            ref.step(procs)
        done, secs = 0, 0.0
        for _ in range(steps):
            q, s = ref.step(sample)
            done += q
            secs += s
    finally:
        ref.close()
    return done / secs, done, secs


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
    import synth
    from paper_2110_08919_b200 import _lib, device as dev, sharded

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_src = load_peaks()

    c = workload(args)
    n, d, nq, k, B = c["n"], c["d"], c["nq"], args.k, c["batch"]
    metric = qa.Metric(c["metric"])

    # ---- index build (not timed): this rank generates and encodes only its
    # own row shard; the per-dimension window comes from the exact min/max of
    # the whole corpus (NCCL MIN/MAX all-reduce of the shard ranges).
    lo, hi = sharded.shard_bounds(n, world, rank)
    X_shard = synth.rows(args.config, lo, hi)
    Q = synth.queries(args.config, nq)
    x_dev = torch.from_numpy(X_shard).cuda()
    mn, mx = dev.minmax(x_dev)
    if world > 1:
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    stats = qa.RangeStats(min=mn.double().cpu().numpy(), max=mx.double().cpu().numpy(), count=n)
    fr = qa.fit_symmetric(stats) if c["calibration"] == "symmetric" else qa.fit_minmax(stats)
    index = qa.Int8Index.from_params(x_dev, fr.params, metric, id_offset=lo)
    del x_dev
    torch.cuda.empty_cache()
    spans = batches(nq, B)
    q_dev = torch.from_numpy(Q).cuda()
    q_host = torch.from_numpy(Q).pin_memory()
    qcodes = [dev.DeviceCodes.empty(b - a, d) for a, b in spans]
    keff = min(k, n)
    outs = [(torch.empty((b - a, keff), dtype=torch.float64, device="cuda"),
             torch.empty((b - a, keff), dtype=torch.int32, device="cuda")) for a, b in spans]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def search_batch(i, queries_dev):
        index.encode_queries(queries_dev, out=qcodes[i])
        if world == 1:
            # stream-ordered entry for every metric (graph-capturable); for
            # angular this skips the zero-norm ValueError check, which the
            # synthetic rows (unit vectors, nonzero codes) cannot trigger
            return index.search_codes(qcodes[i], k, out=outs[i], sync=False)
        return sharded.sharded_search(lambda off: index.search_codes(qcodes[i], k), n, k)

    def device_step():
        if world > 1:
            # the all-gather of batch i overlaps the scan of batch i + 1
            def local_for(i, a, b):
                def local(_off):
                    index.encode_queries(q_dev[a:b], out=qcodes[i])
                    return index.search_codes(qcodes[i], k)
                return local
            sharded.sharded_search_batches([local_for(i, a, b) for i, (a, b) in enumerate(spans)],
                                           n, k)
            return
        for i, (a, b) in enumerate(spans):
            search_batch(i, q_dev[a:b])

    def run_timed(fn, steps):
        """CUDA-event time of `steps` calls of fn on the launching stream,
        L2 flushed (256 MiB write) before each, max over ranks."""
        times = []
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
        return times

    def as_graph(fn):
        """The step captured once as a CUDA graph (the search is stream-ordered:
        no host round trip inside), or None when capture is unavailable."""
        if args.no_graph or world > 1:
            return None
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                fn()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            torch.cuda.synchronize()
            return g
        except Exception as exc:  # pragma: no cover - capture failure: eager timing
            print(f"[bench] graph capture unavailable ({exc}); timing eager launches",
                  file=sys.stderr)
            torch.cuda.synchronize()
            return None

    # warm-up
    for _ in range(max(3, args.warmup)):
        device_step()
    torch.cuda.synchronize()
    # one profiled eager step: the kernel-level event timings (filter / select
    # launches on their stream), launch and round counts
    _lib.reset_scan_totals()
    _lib.set_profiling(True)
    device_step()
    torch.cuda.synchronize()
    tot = _lib.scan_totals()
    _lib.set_profiling(False)
    # encode launches + the scan's own launches (+ merge per batch when sharded)
    launches_per_step = len(spans) + tot["launches"] + (len(spans) if world > 1 else 0)
    graph = as_graph(device_step)

    clocks = ClockSampler(local)
    clocks.start()
    step_ms = run_timed(graph.replay if graph is not None else device_step, args.steps)
    launches = launches_per_step * args.steps
    clk = clocks.stop()

    e2e = e2e_api = None
    if not args.no_e2e:
        host_out = [(torch.empty((b - a, keff), dtype=torch.float64).pin_memory(),
                     torch.empty((b - a, keff), dtype=torch.int32).pin_memory()) for a, b in spans]

        q_in = [torch.empty((b - a, d), dtype=torch.float32, device="cuda") for a, b in spans]

        # the copies ride on their own streams (the two copy engines): batch
        # i + 1's queries go up and batch i - 1's results come down while batch
        # i is searched; the timed stream forks them and joins them again, so
        # every copy of the step lies inside the timed region (and inside the
        # captured graph)
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in spans]
        ev_done = [torch.cuda.Event() for _ in spans]

        def e2e_step():
            cur = torch.cuda.current_stream()
            s_in.wait_stream(cur)
            s_out.wait_stream(cur)
            with torch.cuda.stream(s_in):
                for i, (a, b) in enumerate(spans):
                    q_in[i].copy_(q_host[a:b], non_blocking=True)
                    ev_in[i].record(s_in)
            for i, (a, b) in enumerate(spans):
                cur.wait_event(ev_in[i])
                s, ids = search_batch(i, q_in[i])
                ev_done[i].record(cur)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_done[i])
                    host_out[i][0].copy_(s, non_blocking=True)
                    host_out[i][1].copy_(ids, non_blocking=True)
            cur.wait_stream(s_in)
            cur.wait_stream(s_out)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        e2e_graph = as_graph(e2e_step)
        e2e_ms = run_timed(e2e_graph.replay if e2e_graph is not None else e2e_step, args.steps)
        torch.cuda.synchronize()
        host_ok = all(bool(torch.equal(host_out[i][1], outs[i][1].cpu()))
                      and bool(torch.equal(host_out[i][0], outs[i][0].cpu()))
                      for i in (0, len(spans) - 1))
        e2e = {"value": nq / (float(np.mean(e2e_ms)) / 1e3), "unit": "queries/s",
               "host_results_equal_device": host_ok,
               "h2d_bytes_per_step": int(nq * d * 4),
               "d2h_bytes_per_step": int(nq * keff * (8 + 4)),
               "ms_per_step": float(np.mean(e2e_ms)),
               "path": "Int8Index.encode_queries + search_codes per batch, pinned host fp32 "
                       "queries in, pinned host scores + ids out, copies on their own streams "
                       "(forked from and joined to the timed stream)"
                       + (" (the step replayed as one CUDA graph)" if e2e_graph is not None else "")}
        if world == 1:
            # the reference-facing API: host int8 DenseDatasets in, GroundTruth
            # out (exact.py:105-117); the corpus is the frozen host code array
            corpus = qa.DenseDataset(index.codes_in_input_order())
            qcode_host = [qa.DenseDataset(qc.to_host()) for qc in qcodes]
            for _ in range(2):
                for qs in qcode_host:
                    qa.batch_ground_truth(corpus, qs, k, metric)
            api_ms = []
            for _ in range(args.steps):
                flush.zero_()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for qs in qcode_host:
                    qa.batch_ground_truth(corpus, qs, k, metric)
                api_ms.append((time.perf_counter() - t0) * 1e3)
            e2e_api = {"value": nq / (float(np.mean(api_ms)) / 1e3), "unit": "queries/s",
                       "h2d_bytes_per_step": int(nq * d),
                       "d2h_bytes_per_step": int(nq * keff * 4),
                       "ms_per_step": float(np.mean(api_ms)),
                       "path": "batch_ground_truth(DenseDataset int8 corpus, int8 query batch, "
                               "k, metric) per batch (host wall clock; corpus resident)"}

    # correctness spot check of the last result on a few queries (oracle);
    # outside every timed region
    parity = None
    if rank == 0 and world == 1:
        try:
            from oracle import qa_oracle as o

            torch.cuda.synchronize()
            s, ids = outs[0]  # batch 0 as the last timed (graph-replayed) step left it
            sub = min(8, qcodes[0].n)
            Xc = index.codes_in_input_order()
            Qc = qcodes[0].to_host()[:sub]
            osc, oids = o.scan_topk_i8(Xc, Qc, k, int(metric), o.norms_i8(Xc), o.norms_i8(Qc))
            parity = {"queries_checked": sub,
                      "ids_equal": bool(np.array_equal(ids[:sub].cpu().numpy(), oids)),
                      "scores_equal": bool(np.array_equal(s[:sub].cpu().numpy(), osc))}
        except Exception as exc:  # pragma: no cover
            parity = {"error": str(exc)[:200]}

    ms = float(np.mean(step_ms))
    value = nq / (ms / 1e3)
    # roofline of the dominant kernel (the fused tcgen05 filter pass):
    # algorithmic ops = 2 * nq * rows * d (unpadded d) per launch, divided by
    # the CUDA-event time of those launches on their stream, summed over the
    # step's batches
    peak_tops = 2.0 * float(peaks["bf16_tflops"])
    traffic, traffic_note = None, "no committed ncu capture for this workload"
    tfile = ROOT / "profiles" / f"r02_filter_traffic_cfg{args.config}.json"
    if tfile.exists() and args.n is None and args.nq is None and world == 1:
        tj = json.loads(tfile.read_text())
        traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
        traffic_note = (f"DRAM bytes per launch of the main filter pass ({tj['source']}); "
                        f"algorithmic bytes per launch {tj['algorithmic_bytes']}")
    achieved = (tot["filter_ops"] / (tot["filter_ms"] / 1e3) / 1e12) if tot["filter_ms"] > 0 else None
    roofline = {
        "bound": "tensor", "kernel": "filter_tc_kernel (tcgen05 kind::i8 + fused threshold epilogue)",
        "achieved": achieved, "peak": peak_tops, "unit": "TOP/s",
        "frac": (achieved / peak_tops) if achieved else None,
        "peak_source": f"2 x dense bf16 {peaks_src} (int8 dense = 2x bf16 on B200)",
        "frac_of_measured_kind_i8": (achieved / MMA_I8_TOPS) if achieved else None,
        "frac_of_spec_4500": (achieved / 4500.0) if achieved else None,
        "traffic": traffic,
        "traffic_note": traffic_note,
        "whole_step_tops": 2.0 * nq * (n / world) * d / (ms / 1e3) / 1e12,
        "filter_ms_per_step": tot["filter_ms"], "select_ms_per_step": tot["select_ms"],
        "filter_launches_per_step": tot["filter_launches"],
        "filter_share_of_step": tot["filter_ms"] / ms if ms else None,
        "scan_stats": {key: tot[key] for key in ("rounds", "launches", "retries", "candidates")},
    }
    line = {
        "metric": METRIC_NAME, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": f"synthetic (synth.py config {args.config}, seed {c['seed']}; "
                f"stand-in for the paper's dataset)",
        "config": {"workload": workload_desc(c, k), "n": n, "d": d, "nq": nq, "batch": B, "k": k,
                   "metric": metric.short_name, "calibration": c["calibration"],
                   "parallelism": (f"row-shard x{world}, queries replicated, NCCL all-gather of "
                                   f"top-k" if world > 1 else "single GPU"),
                   "l2": "flushed (256 MiB write) before every timed step"},
        "database_vectors_per_s": value * n,
        "roofline": roofline,
        "e2e": e2e,
        "e2e_reference_api": e2e_api,
        "gpu_launches": launches,
        "gpu_launches_per_step": launches_per_step,
        "timing": ("CUDA graph of the whole step (stream-ordered searches, no host round trip), "
                   "replayed per step" if graph is not None else "eager launches"),
        "clocks": clk,
        "parity_spot_check": parity,
        "impl": "b200",
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            v1, q1, s1 = measure_reference(c, X_shard, Q, k, 1, 6.0)
            vp, qp, sp = measure_reference(c, X_shard, Q, k, cores, 12.0)
            line["cpu_baseline"] = {
                "value": vp, "unit": "queries/s", "cores": cores, "kind": "reference",
                "sample": f"{qp} of the {nq} queries against the full {n}x{d} int8 db "
                          f"(reference quantann._core.scan_topk, {cores} forked workers)",
                "single_thread": {"value": v1, "queries": q1, "seconds": s1},
                "cpu_model": cpu_model()}
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"error": str(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """The reference arm: its own CPU kernel on this box's host cores.  Only
    rank 0 works (the path is host-only); other ranks exit at once."""
    import synth

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    c = workload(args)
    k = args.k
    X, Q = synth.rows(args.config, 0, c["n"]), synth.queries(args.config, c["nq"])
    cores = os.cpu_count() or 1
    ref = CpuReference(c, X, Q, k, cores)
    sample = reference_sample(c, cores, 6.0)
    for _ in range(args.warmup):
        ref.step(cores)
    done, secs = 0, 0.0
    for _ in range(args.steps):
        q, s = ref.step(sample)
        done += q
        secs += s
    ref.close()
    value = done / secs
    line = {
        "metric": METRIC_NAME, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int8",
        "data": f"synthetic (synth.py config {args.config}, seed {c['seed']}; "
                f"stand-in for the paper's dataset)",
        "config": {"workload": workload_desc(c, k), "n": c["n"], "d": c["d"], "nq": c["nq"],
                   "batch": c["batch"], "k": k, "metric": ("ip", "l2", "angular")[c["metric"]],
                   "calibration": c["calibration"],
                   "parallelism": f"{cores} host processes (forked workers over query slices)",
                   "l2": "flushed (256 MiB write) before every timed step"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "reference",
                         "sample": f"{sample} queries per step ({done} in {args.steps} steps) "
                                   f"against the full {c['n']}x{c['d']} int8 db "
                                   f"(reference quantann._core.scan_topk)",
                         "cpu_model": cpu_model()},
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
