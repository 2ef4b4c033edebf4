#!/usr/bin/env python3
"""Benchmark of the B200 enumeration-and-retrieval path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1|c2|c3|c4]

N = 1 (BASELINE.json configs[1], "c2"): a synthetic 10M-product CSL of the
config-1 shape (40 reactions, mixed 2/3-component), random-init
linear heads on a synthetic embedding cache (property heads calibrated), and
20 queries (dock_a..e minimize x {lipinski, veber, pfizer_3_75, astex_ro3},
k=1000) answered in ONE batched device pass.  A step = one such pass.

N > 1 (configs[2] / configs[3], one process per GPU, NCCL): STRONG scaling of
the config-3 query (dock_a minimize, Lipinski, k=1000) over the synthetic
1e9-product CSL — every rank scans its contiguous 1/N of the index space,
the per-rank top-k entries are all-gathered and merged exactly on every rank
(dist.sharded_batch, stream-ordered) — plus the config-4 query (5 property
windows, k=10,000) over the ~5e9-product CSL on the same N GPUs, and the same
two queries on rank 0's GPU alone (the N = 1 point of the strong-scaling
curve).

metric: products scored per second = (products in the range) x (queries)
per step / step time.  `value` times the device pipeline with the table
resident in HBM (CUDA events on the launching stream, L2 flushed between
steps); `e2e` times the public C-ABI call with host buffers (query
descriptors H2D every step, result rows D2H into caller-owned host arrays,
host sync); `api` times the reference-facing Python operator API
(engine.search_topk_many / search_topk_stream on CslLibrary / QuerySpec
objects, TopKResult construction included).

--impl reference: the reference algorithm's CPU path (oracle port of
engine.search_topk_stream, all host cores via exact index-range sharding) on
the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2510_24380_b200 import synth  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=["c1", "c2", "c3", "c4"],
                    help="default: c2 on one GPU, c3 (strong scaling) on several")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks, no baselines)")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (5e9-product) roofline and effective passes")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(config: str, world: int = 1):
    """Shape and queries of a config (the library is NOT scaled with the GPU
    count: N > 1 is strong scaling of the same library)."""
    base = "c1" if config in ("c1", "c2") else config
    shape = synth.make_shape(synth.SHAPES[base])
    if config == "c2":
        queries = synth.c2_queries()
    elif config == "c1":
        queries = [synth.c1_query()]
    elif config == "c3":
        queries = [synth.c3_query()]
    else:
        queries = [synth.c4_query()]
    return shape, queries


def n_tests(q) -> int:
    """Per-product compares of the enumeration kernel for a query: the
    admission compare + one per finite merged bound (capi.cu make_tests)."""
    lo, up = {}, {}
    for t, a, b in q["constraints"]:
        if math.isfinite(a):
            lo[t] = max(lo.get(t, -math.inf), a)
        if math.isfinite(b):
            up[t] = min(up.get(t, math.inf), b)
    return 1 + len(lo) + len(up)


def f_ops(queries) -> int:
    """SURVEY.md §8(d) algorithmic FP32 work per product of a batched pass:
    F = |union of the queries' distinct tasks| (one add each) + sum over
    queries of (finite bounds + 1 admission compare)."""
    tasks = set()
    total = 0
    for q in queries:
        tasks.add(q["objective"])
        for t, a, b in q["constraints"]:
            if math.isfinite(a) or math.isfinite(b):
                tasks.add(t)
        total += n_tests(q)
    return len(tasks) + total


def build_model(shape, seed=1):
    return synth.build_model(shape, seed=seed)


# ---------------------------------------------------------------------------
# clocks (NVML polled in a thread during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self.stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self.stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                break
            time.sleep(0.002)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv is not None:
            self.stop.set()
            self.t.join()

    def summary(self):
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples), "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------------
# CPU legs (oracle port of the reference algorithm; test/baseline infra only)
# ---------------------------------------------------------------------------

_CPU = {}


def _cpu_task(args):
    qi, a, b = args
    from oracle import scan_oracle as orc
    W = _CPU
    q = W["queries"][qi]
    s, g, ret, disc, scanned = orc.search_topk(W["values"], W["biases"], W["lib"], q, a, b)
    return qi, s, g


def cpu_pass(pool, procs, lib, queries, start, end, ranges=None):
    """Exact top-k of every query over [start, end) with `procs` processes
    (contiguous index-range shards + exact merge); with `ranges`,
    over the union of those sub-ranges instead (a bounded sample)."""
    if ranges is None:
        ranges = [(start + (end - start) * r // procs, start + (end - start) * (r + 1) // procs) for r in range(procs)]
    tasks = [(qi, a, b) for qi in range(len(queries)) for a, b in ranges]
    parts = {}
    for qi, s, g in pool.imap_unordered(_cpu_task, tasks):
        parts.setdefault(qi, []).append((s, g))
    out = []
    for qi, q in enumerate(queries):
        s = np.concatenate([p[0] for p in parts[qi]])
        g = np.concatenate([p[1] for p in parts[qi]])
        order = np.lexsort((g, -s))[: q.k]
        out.append((s[order], g[order]))
    return out


def sample_ranges(total: int, frac: float, pieces: int = 64):
    """`pieces` equal slices spread evenly over [0, total), `frac` of it in all."""
    span = int(total * frac) // pieces
    return [(total * i // pieces, total * i // pieces + span) for i in range(pieces)]


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_setup(shape, values, biases, queries_named, procs):
    from oracle import scan_oracle as orc
    lib = orc.Lib(shape.sizes, shape.pair_off)
    qs = []
    for qd in queries_named:
        nq = synth.to_native(qd, 0, lib.total)
        qs.append(orc.Query(nq["obj"], nq["maximize"], nq["cons"], nq["k"]))
    _CPU.update(values=values, biases=biases, lib=lib, queries=qs)
    ctx = mp.get_context("fork")
    pool = ctx.Pool(procs)
    return pool, lib, qs


def cpu_procs(args) -> int:
    return args.cpu_procs or len(os.sched_getaffinity(0))


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return 0
    shape, queries_named = workload(args.config, world)
    u, w, b = build_model(shape)
    values = synth.host_table(u, w)
    procs = cpu_procs(args)
    pool, lib, qs = cpu_setup(shape, values, b, queries_named, procs)
    # a step = the whole workload when it takes a second or two on the host,
    # else a bounded sample of it (evenly spread slices of the index space)
    frac = 1.0 if shape.total * len(qs) <= 4e8 else max(1e-3, 1.25e8 / (shape.total * len(qs)))
    ranges = None if frac >= 1.0 else sample_ranges(lib.total, frac)
    products = (shape.total if ranges is None else sum(b_ - a_ for a_, b_ in ranges)) * len(qs)
    for _ in range(args.warmup):
        cpu_pass(pool, procs, lib, qs, 0, lib.total, ranges)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_pass(pool, procs, lib, qs, 0, lib.total, ranges)
    dt = time.perf_counter() - t0
    pool.close()
    value = products * args.steps / dt
    sample = (f"full pass: {len(qs)} quer{'y' if len(qs) == 1 else 'ies'} x {shape.total} products per step"
              if ranges is None else
              f"bounded sample per step: {len(qs)} quer{'y' if len(qs) == 1 else 'ies'} x {products // len(qs)} "
              f"products ({frac:.4f} of the {shape.total}-product library, 64 evenly spread slices)")
    line = {
        "impl": "reference", "metric": "products scored/sec", "value": value, "unit": "products/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, shape, queries_named, world),
        "cpu_baseline": {"value": value, "unit": "products/s", "cores": procs, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": sample + " (oracle/scan_oracle.py restating engine.search_topk_stream)"},
        "e2e": {"value": value, "unit": "products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, shape, queries_named, world):
    nq = len(queries_named)
    return {
        "workload": f"{args.config}: synthetic {shape.total / 1e6:.1f}M-product CSL ({len(shape.sizes)} reactions, "
                    f"mixed 2/3-component), {nq} quer{'y' if nq == 1 else 'ies'} "
                    f"(k={queries_named[0]['k']}) in one batched pass"
                    + (f", index range strong-scaled over {world} GPUs" if world > 1 else ""),
        "products": shape.total, "queries": nq, "k": queries_named[0]["k"],
        "products_per_step": shape.total * nq, "pair_rows": shape.n_pairs,
        "parallelism": f"contiguous index-range shards x{world} + NCCL all-gather + exact merge" if world > 1
                       else "single GPU",
        "l2": "flushed between timed steps (256 MiB write)",
        "model": "random-init linear heads (11 tasks) on a synthetic N(0,1) 64-d pair-embedding cache, "
                 "property heads calibrated",
    }


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def reduce_max(x: float) -> float:
    """max over ranks of a host scalar (device tensor under NCCL)."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed_loop(stream, steps, fn, flush, sync_each=False):
    """K steps of fn() bracketed by CUDA events on `stream` (L2 flushed before
    each); returns (device ms per step, host wall ms per step, last result).
    sync_each: wait for each step's end event before the next flush (a
    synchronous call's natural rhythm; the flush then never queues behind it)."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    wall = 0.0
    out = None
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        t0 = time.perf_counter()
        out = fn()
        ev[i][1].record(stream)
        wall += time.perf_counter() - t0
        if sync_each:
            ev[i][1].synchronize()
    torch.cuda.synchronize()
    return sum(x.elapsed_time(y) for x, y in ev) / steps, wall * 1e3 / steps, out


def peaks_json():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    if args.config is None:
        args.config = "c2" if world == 1 else "c3"
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        return run_multi(args, rank, world)
    return run_single(args)


# ---------------------------------------------------------------------------
# N = 1: the batched config-2 pass (headline), rooflines, CPU baselines, API
# ---------------------------------------------------------------------------

def results_equal(a: dict, b: dict) -> bool:
    """Every result field, bit for bit."""
    keys = ("g", "objective", "constraint_values", "reaction", "digits")
    return all(np.array_equal(np.asarray(a[k]), np.asarray(b[k])) for k in keys) and \
        (a["n"], a["discarded"], a["scanned"]) == (b["n"], b["discarded"], b["scanned"])


def oracle_parity(values, biases, lib, q, res, s, g) -> bool:
    """A device result against oracle (s, g): indices, objective bits and
    constraint-value bits (apex_score order, oracle.materialize_arrays)."""
    from oracle import scan_oracle as orc

    if not np.array_equal(np.asarray(res["g"]).astype(np.int64), g):
        return False
    _, _, obj, cons = orc.materialize_arrays(values, biases, lib, q, s, g)
    if not np.array_equal(np.asarray(res["objective"]).view(np.uint64), obj.view(np.uint64)):
        return False
    return not q.cons or np.array_equal(np.asarray(res["constraint_values"]).view(np.uint64), cons.view(np.uint64))


def tie_rate(values, biases, shape, task: int) -> float:
    """Fraction of products whose fp64 score (reference order, bias last)
    equals another product's: 1 - distinct / N over the whole library."""
    vals = []
    for sizes, offs in zip(shape.sizes, shape.pair_off):
        acc = values[task, offs[0]:offs[0] + sizes[0]].astype(np.float64)
        for n, o in zip(sizes[1:], offs[1:]):
            acc = (acc[:, None] + values[task, o:o + n].astype(np.float64)[None, :]).reshape(-1)
        vals.append(acc + float(biases[task]))
    v = np.concatenate(vals)
    return 1.0 - len(np.unique(v)) / len(v)


def api_latencies(args, shape, values, biases, queries_named, lib_total):
    """The reference-facing operator API (engine.search_topk_many /
    search_topk_stream on mirror CslLibrary / ContributionTable / QuerySpec
    objects, TopKResult entries built), host wall clock per call."""
    from paper_2510_24380_b200 import engine

    library, table = synth.mirror_objects(shape, values, biases)
    qspecs = [synth.query_spec(q) for q in queries_named]
    t0 = time.perf_counter()
    engine.search_topk_many(library, table, qspecs)
    first = (time.perf_counter() - t0) * 1e3
    for _ in range(args.warmup):
        engine.search_topk_many(library, table, qspecs)
    ms = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = engine.search_topk_many(library, table, qspecs)
        ms.append((time.perf_counter() - t0) * 1e3)
    med = statistics.median(ms)
    res = {"e2e_api": {"value": lib_total * len(qspecs) / (med * 1e-3), "unit": "products/s", "ms_per_step": med,
                       "first_call_ms": first, "entries_per_step": sum(len(r.entries) for r in out),
                       "call": "engine.search_topk_many(library, table, 20 QuerySpecs) -> 20 TopKResult"}}
    # single-query latency of the config-1 query (distinct calls, same query)
    q1 = synth.query_spec(synth.c1_query())
    for _ in range(3):
        engine.search_topk_stream(library, table, q1)
    lat = []
    for _ in range(max(20, args.steps)):
        t0 = time.perf_counter()
        engine.search_topk_stream(library, table, q1)
        lat.append((time.perf_counter() - t0) * 1e3)
    res["c1_query_ms"] = {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                          "n": len(lat), "call": "engine.search_topk_stream (config-1 query, k=100)"}
    return res


def c5_latencies(local, stream, n=60):
    """Config 5 sample: n distinct random queries over the 1e9-product library
    through engine.search_topk_stream (table resident, descriptors and results
    through the host every call), p50/p99 wall ms."""
    from paper_2510_24380_b200 import engine

    shape = synth.make_shape(synth.SHAPES["c3"])
    u, w, b = build_model(shape)
    values = synth.host_table(u, w) if shape.n_pairs < 400_000 else None
    del u
    library, table = synth.mirror_objects(shape, values, b)
    allq = synth.c5_queries()
    qs = [synth.query_spec(q) for q in allq[:n]]
    t0 = time.perf_counter()
    engine.search_topk_stream(library, table, qs[0])
    first = (time.perf_counter() - t0) * 1e3
    # steady state: one untimed query of each k class (outside the timed
    # sample) sizes the per-k buffers once, as a long-running sweep would
    for kk in sorted({q.k for q in qs}):
        extra = next((synth.query_spec(q) for q in allq[n:] if synth.query_spec(q).k == kk), None)
        if extra is not None:
            engine.search_topk_stream(library, table, extra)
    # the interpreter's cyclic-GC pauses that land inside a call (a gen-2
    # sweep walks every live object of the process) are part of its latency;
    # record them so an outlier can be attributed
    import gc
    gc_t = {"t0": 0.0, "ms": 0.0}

    def gc_cb(phase, info):
        if phase == "start":
            gc_t["t0"] = time.perf_counter()
        else:
            gc_t["ms"] += (time.perf_counter() - gc_t["t0"]) * 1e3

    lat, by_k, rows = [], {}, []
    gc.callbacks.append(gc_cb)
    try:
        for i, q in enumerate(qs):
            gc_t["ms"] = 0.0
            t0 = time.perf_counter()
            engine.search_topk_stream(library, table, q)
            dt = (time.perf_counter() - t0) * 1e3
            lat.append(dt)
            by_k.setdefault(q.k, []).append(dt)
            rows.append({"i": i, "ms": round(dt, 3), "k": q.k, "gc_ms": round(gc_t["ms"], 3)})
    finally:
        gc.callbacks.remove(gc_cb)
    return {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)), "mean": float(np.mean(lat)),
            "n": len(lat), "first_call_ms": first,
            "p50_by_k": {str(k): float(np.median(v)) for k, v in sorted(by_k.items())},
            "slowest": sorted(rows, key=lambda r: -r["ms"])[:3],
            "call": "engine.search_topk_stream, first n synth.c5_queries() (config 5) over the c3 library, after one "
                    "untimed query per k class"}


def run_single(args):
    import torch

    torch.cuda.set_device(0)
    import __graft_entry__ as g
    g.build()
    from paper_2510_24380_b200 import _native

    shape, queries_named = workload(args.config, 1)
    u, w, b = build_model(shape)
    # a real (non-default) torch stream shared with the C-ABI context, so the
    # CUDA events below bracket exactly the work the library enqueues
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _native.DeviceContext(0, stream.cuda_stream)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    values = ctx.load_cache(u, w, b)
    nqueries = [synth.to_native(q, 0, shape.total) for q in queries_named]
    products = shape.total * len(nqueries)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    prepared_dev = ctx.prepare(nqueries)  # descriptors built once (device-resident pass)

    for _ in range(args.warmup):
        ctx.run_async(prepared_dev)
        ctx.query_fetch()
    torch.cuda.synchronize()

    # timed: device-resident pass
    launches = 0
    sampler = ClockSampler(0) if not args.profile else None

    def step_device():
        nonlocal launches
        launches += ctx.run_async(prepared_dev)["kernel_launches"]

    torch.cuda.synchronize()
    with (sampler if sampler else _Null()):
        ms_per_step, _, _ = timed_loop(stream, args.steps, step_device, flush)
    res_dev, st_dev = ctx.query_fetch()  # validates the last in-flight pass (overflow check)
    value = products / (ms_per_step * 1e-3)

    # e2e: public C-ABI call with host buffers, descriptors H2D every step;
    # results returned as views into the context's pinned host block (D2H in
    # the same device pass, no host-side copy): the C-ABI view mode
    ctx.set_option("force_upload", 1)
    prepared = ctx.prepare_views(nqueries)
    acc = {"scan": [], "h2d": 0, "d2h": 0}

    def step_e2e():
        # the bare C-ABI call: host descriptors in, every result row in pinned
        # host memory when it returns (numpy views are built after timing)
        r, st = ctx.run_views_raw(prepared)
        acc["h2d"] += st.h2d_bytes
        acc["d2h"] += st.d2h_bytes
        return r, st

    for _ in range(args.warmup):  # this call's own signature (copy-out) is captured on its second run
        ctx.run_views_raw(prepared)
    torch.cuda.synchronize()
    e2e_ms, e2e_wall, (res_raw, st_raw) = timed_loop(stream, args.steps, step_e2e, flush,
                                                      sync_each=os.environ.get("APEX_BENCH_E2E_SYNC", "1") == "1")
    res, _ = ctx.views_of(prepared, res_raw, st_raw)
    ctx.set_option("force_upload", 0)
    e2e_value = products / (e2e_ms * 1e-3)

    # per-stage device times and the enumeration kernel's own time: a separate
    # loop with the stage events on (option "stages": each event is a node on
    # the pass's critical path, so the timed loops above run without them)
    ctx.set_option("stages", 1)
    st_stages = []
    for _ in range(max(5, min(args.steps, 20))):
        flush.zero_()
        _, st_k = ctx.run_views(prepared)
        acc["scan"].append(st_k["scan_kernel_ms"])
        st_stages.append(st_k)
    st_dev = {k_: statistics.median(x[k_] for x in st_stages)
              for k_ in ("pack_ms", "seed_ms", "scan_ms", "select_ms", "finalize_ms", "d2h_ms", "total_ms",
                         "scan_kernel_ms")} | {"candidates": st_stages[-1]["candidates"]}

    # Rooflines: F = algorithmic FP32 ops per product of the
    # batched pass; peak P32 = SMs x 128 FP32 lanes x the SM clock sampled
    # under load.  The roofline claim uses a pass that evaluates every active
    # test on every product (the full-predicate kernel, mode 0); the default
    # sorted-column kernel skips products that cannot pass and is reported
    # as "effective" (F-equivalent rate of the same pass).
    peaks = peaks_json()
    sm_count = ctx.device_info()[0]
    clk = sampler.summary() if sampler else None
    clk_mhz = float((clk or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0))
    peak_tops = sm_count * 128 * clk_mhz * 1e6 / 1e12
    scanned = shape.total
    F = f_ops(queries_named)
    traffic = traffic_sorted = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            traffic, traffic_sorted = tj.get(args.config), tj.get(args.config + "_sorted")
        except Exception:
            traffic = None
    kern_ms = statistics.mean(acc["scan"]) if acc["scan"] else None
    effective = None
    if kern_ms:
        eq = scanned * F / (kern_ms * 1e-3) / 1e12
        effective = {"products_per_s": scanned * len(nqueries) / (kern_ms * 1e-3), "kernel_ms": kern_ms,
                     "F_equivalent_tops": eq, "frac_equivalent": eq / peak_tops,
                     "kernel": "scan_sorted_kernel (per-row threshold + most selective test's sorted range)",
                     "note": "pruned: products that cannot pass are never evaluated, so the F-equivalent "
                             "rate can exceed the FP32 peak"}
    roofline = None
    if not args.profile:
        ctx.set_option("mode", 0)
        full_ms = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            _, stf = ctx.query(nqueries)
            full_ms.append(stf["scan_kernel_ms"])
        ctx.set_option("mode", 3)
        fm = statistics.median(full_ms)
        fach = scanned * F / (fm * 1e-3) / 1e12
        roofline = {"bound": "fp32", "achieved": fach, "peak": peak_tops, "unit": "TFLOP/s", "frac": fach / peak_tops,
                    "traffic": traffic, "kernel": "scan_kernel<NT,1,0> (K3 full predicate: every test on every "
                                                  "product, FSETP chain), all launches of one pass",
                    "kernel_ms": fm, "F_per_product": F, "products": scanned,
                    "peak_basis": f"{sm_count} SMs x 128 FP32 lanes x {clk_mhz:.0f} MHz (median SM clock under load)"}

    ctx.set_option("stages", 0)

    # the SURVEY's roofline reference point: the C4 query over the ~5e9-product
    # library (F = 15 per product), full-predicate pass (mode 0) and the
    # default sorted-column pass, on a second context with that table resident
    roofline_c4 = effective_c4 = c4_single = None
    if not args.profile and not args.no_c4 and args.config != "c4":
        try:
            c4shape, c4q = workload("c4", 1)
            u4, w4, b4 = build_model(c4shape)
            ctx4 = _native.DeviceContext(0, stream.cuda_stream)
            ctx4.set_option("stages", 1)  # scan kernel times (stage events)
            ctx4.load_library(c4shape.sizes, c4shape.pair_off, c4shape.g_offsets(), c4shape.n_pairs)
            ctx4.load_cache(u4, w4, b4, want_values=False)
            del u4
            q4 = [synth.to_native(q, 0, c4shape.total) for q in c4q]
            F4 = f_ops(c4q)
            pb4 = ctx4.prepare_views(q4)
            times, totals = {}, {}
            for mode in (0, 3):
                ctx4.set_option("mode", mode)
                ctx4.run_views(pb4)
                ms4, tot4 = [], []
                for _ in range(3 if mode == 0 else 10):
                    flush.zero_()
                    t0 = time.perf_counter()
                    _, st4 = ctx4.run_views(pb4)
                    tot4.append((time.perf_counter() - t0) * 1e3)
                    ms4.append(st4["scan_kernel_ms"])
                times[mode] = statistics.median(ms4)
                totals[mode] = statistics.median(tot4)
            ach4 = c4shape.total * F4 / (times[0] * 1e-3) / 1e12
            tr4 = None
            try:
                tr4 = json.loads((ROOT / "profiles" / "traffic.json").read_text()).get("c4")
            except Exception:
                pass
            roofline_c4 = {"bound": "fp32", "achieved": ach4, "peak": peak_tops, "unit": "TFLOP/s",
                           "frac": ach4 / peak_tops, "traffic": tr4,
                           "kernel": "scan_kernel<NT,1,0> full predicate (mode 0)",
                           "kernel_ms": times[0], "F_per_product": F4, "products": c4shape.total,
                           "workload": "c4: one query (5 property windows, k=10000) over the synthetic "
                                       f"{c4shape.total / 1e9:.2f}e9-product CSL"}
            eq4 = c4shape.total * F4 / (times[3] * 1e-3) / 1e12
            effective_c4 = {"products_per_s": c4shape.total / (times[3] * 1e-3), "kernel_ms": times[3],
                            "F_equivalent_tops": eq4, "frac_equivalent": eq4 / peak_tops,
                            "kernel": "scan_sorted_kernel"}
            c4_single = {"query_ms_c_abi": totals[3], "products_per_s_c_abi": c4shape.total / (totals[3] * 1e-3),
                         "call": "apex_query (one C4 query, k=10000, result rows to host) on one GPU"}
            ctx4.close()
        except Exception as exc:  # noqa: BLE001 - reported, never fatal for the headline line
            roofline_c4 = {"error": str(exc)[:200]}

    # K1 precompute (HBM-bound) at the C4 table size: u fp64
    # [n_pairs, 64] generated on the device, one timed launch after warm-up;
    # algorithmic bytes = 8*d*n_pairs (u) + 8*n_tasks*d (heads) + 4*n_tasks*n_pairs (table)
    precompute = None
    if not args.profile:
        try:
            c4 = synth.make_shape(synth.SHAPES["c4"])
            n_p, d_, n_t = c4.n_pairs, 64, len(synth.TASKS)
            u_dev = torch.randn((n_p, d_), dtype=torch.float64, device="cuda")
            w_dev = torch.randn((n_t, d_), dtype=torch.float64, device="cuda") * 0.01
            v_dev = torch.empty((n_t, n_p), dtype=torch.float32, device="cuda")
            # the K1 kernel alone: CUDA events around its launch inside the call
            w_host = w_dev.cpu().numpy().copy()  # host heads: kernel parameters of the TMA form
            for _ in range(3):
                ctx.precompute_device(u_dev.data_ptr(), n_p, d_, w_host.ctypes.data, n_t, v_dev.data_ptr())
            kms = []
            for _ in range(10):
                flush.zero_()  # same stream: the GPU is busy when the kernel's start event is recorded
                ctx.precompute_device(u_dev.data_ptr(), n_p, d_, w_host.ctypes.data, n_t, v_dev.data_ptr())
                kms.append(ctx.precompute_time())
            torch.cuda.synchronize()
            pms = statistics.median(kms)
            pbytes = 8 * d_ * n_p + 8 * n_t * d_ + 4 * n_t * n_p
            hbm = float(peaks.get("hbm_gbs", 6550.7))
            precompute = {"kernel": "precompute_bulk_kernel<11,64> (K1: TMA bulk-copy ring of u tiles, heads as "
                                    "DFMA constant operands; fp64 dots, fp32 table)",
                          "n_pairs": n_p, "d": d_, "n_tasks": n_t, "ms": pms, "bytes": pbytes,
                          "achieved_GBps": pbytes / (pms * 1e-3) / 1e9, "peak_GBps": hbm,
                          "frac": pbytes / (pms * 1e-3) / 1e9 / hbm,
                          "peak_basis": "MEASURED_PEAKS hbm_gbs (copy bandwidth)"}
            del u_dev, w_dev, v_dev
        except Exception as exc:  # noqa: BLE001 - reported, never fatal for the headline line
            precompute = {"error": str(exc)[:200]}

    # the roofline object describes the dominant kernel of the headline step
    # (the sorted-column enumeration), with SURVEY §8(d)'s algorithmic work F
    # per product: achieved = products x F / its mean launch time in the timed
    # e2e loop (CUDA events on the launching stream); the full-predicate pass
    # (every test on every product, ALU-bound) is reported beside it
    roofline_dominant = None
    if effective is not None:
        roofline_dominant = {"bound": "fp32", "achieved": effective["F_equivalent_tops"], "peak": peak_tops,
                             "unit": "TFLOP/s", "frac": effective["frac_equivalent"], "traffic": traffic_sorted,
                             "kernel": "scan_sorted_kernel (default; per-row exact thresholds, most selective test's "
                                       "sorted range)", "kernel_ms": kern_ms, "F_per_product": F, "products": scanned,
                             "note": "F-equivalent: products the kernel proves cannot pass are never evaluated",
                             "peak_basis": f"{sm_count} SMs x 128 FP32 lanes x {clk_mhz:.0f} MHz"}
    line = {
        "metric": "products scored/sec", "value": value, "unit": "products/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded CSL shape, random-init heads, calibrated properties)",
        "config": config_dict(args, shape, queries_named, 1),
        "e2e": {"value": e2e_value, "unit": "products/s", "h2d_bytes_per_step": acc["h2d"] // max(args.steps, 1),
                "d2h_bytes_per_step": acc["d2h"] // max(args.steps, 1), "ms_per_step": e2e_ms,
                "host_wall_ms_per_step": e2e_wall,
                "call": "apex_query (C ABI) with host query descriptors and host result rows"},
        "gpu_launches": launches, "roofline": roofline_dominant or roofline, "roofline_full_predicate": roofline,
        "effective": effective, "roofline_c4": roofline_c4,
        "effective_c4": effective_c4, "c4_single_gpu": c4_single, "precompute": precompute,
        "clocks": sampler.summary() if sampler else None,
        "device_stages_ms": {k_: st_dev[k_] for k_ in ("pack_ms", "seed_ms", "scan_ms", "select_ms", "finalize_ms",
                                                       "d2h_ms", "total_ms", "scan_kernel_ms")},
        "candidates_per_step": st_dev["candidates"],
        "gpu_parity_device_vs_e2e": all(results_equal(x, y) for x, y in zip(res_dev, res)),
    }
    if not args.profile:
        try:
            line.update(api_latencies(args, shape, values, b, queries_named, shape.total))
        except Exception as exc:  # noqa: BLE001
            line["e2e_api"] = {"error": str(exc)[:200]}
        try:
            line["c5_query_ms"] = c5_latencies(0, stream)
        except Exception as exc:  # noqa: BLE001
            line["c5_query_ms"] = {"error": str(exc)[:200]}
        obj = synth.TASKS.index(queries_named[0]["objective"])
        line["exact_tie_rate"] = {"dock_a": tie_rate(values, b, shape, obj),
                                  "mw": tie_rate(values, b, shape, synth.TASKS.index("mw")),
                                  "definition": "1 - distinct fp64 scores / products, whole library"}
    if not args.no_cpu_baseline and not args.profile:
        from oracle import fast_oracle as fo
        from oracle import scan_oracle as orc

        procs = cpu_procs(args)
        pool, lib, qs = cpu_setup(shape, values, b, queries_named, procs)
        t0 = time.perf_counter()
        cpu_out = cpu_pass(pool, procs, lib, qs, 0, lib.total)
        dt = time.perf_counter() - t0
        # one core: the same port, a bounded sample (2 of the 20 queries)
        t1 = time.perf_counter()
        for q in qs[:2]:
            orc.search_topk(values, b, lib, q)
        dt1 = time.perf_counter() - t1
        pool.close()
        # the threaded C restatement of the same algorithm (the scale checker)
        prep = fo.Prepared(values, b, lib)
        t2 = time.perf_counter()
        c_out = [fo.search_topk(values, b, lib, q, prepared=prep) for q in qs]
        dt2 = time.perf_counter() - t2
        # parity of the benchmarked pass itself (same inputs): indices,
        # objective and constraint-value bits of all 20 queries
        ok = all(oracle_parity(values, b, lib, q, r, co[0], co[1]) for q, r, co in zip(qs, res, cpu_out))
        ok_c = all(np.array_equal(co[1], cc[1]) for co, cc in zip(cpu_out, c_out))
        line["cpu_baseline"] = {"value": products / dt, "unit": "products/s", "cores": procs, "kind": "port",
                                "cpu_model": cpu_model(),
                                "sample": f"full pass ({len(qs)} queries x {shape.total} products), "
                                          "oracle/scan_oracle.py (numpy restatement of engine.search_topk_stream)",
                                "one_core": {"value": 2 * shape.total / dt1, "unit": "products/s", "cores": 1,
                                             "sample": f"2 queries x {shape.total} products, one process"},
                                "c_restatement": {"value": products / dt2, "unit": "products/s", "cores": procs,
                                                  "sample": "full pass, oracle/scan_oracle.c (threaded C, "
                                                            "threshold-pruned)", "parity_with_port": ok_c},
                                "parity_with_gpu": ok,
                                "parity_fields": "g, objective bits, constraint-value bits, retained/discarded"}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# N > 1: strong scaling of the config-3 query (and config 4), one process per GPU
# ---------------------------------------------------------------------------

def run_multi(args, rank, world):
    import torch
    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", 0))
    backend = os.environ.get("APEX_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()  # shared-GPU logic test (not a timing mode)
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    import __graft_entry__ as g
    if rank == 0:
        g.build()
    dist.barrier()
    g.build()
    from paper_2510_24380_b200 import _native
    from paper_2510_24380_b200.dist import sharded_batch

    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sampler = ClockSampler(local) if rank == 0 and not args.profile else None

    def strong(config, steps, warmup):
        """One config's query strong-scaled over the ranks: device ms (max over
        ranks), host wall ms (max over ranks), launches, bytes, parity vs rank
        0's single-GPU result, and rank 0's single-GPU device ms."""
        shape, queries_named = workload(config, world)
        u, w, b = build_model(shape)
        ctx = _native.DeviceContext(local, stream.cuda_stream)
        ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
        ctx.load_cache(u, w, b, want_values=False)
        single = None
        if rank == 0:  # the N = 1 reference point of the same workload (rank 0's GPU alone)
            single = _native.DeviceContext(local, stream.cuda_stream)
            single.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
            single.load_cache(u, w, b, want_values=False)
        del u
        gq = [synth.to_native(q, 0, shape.total) for q in queries_named]
        k = max(q["k"] for q in gq)
        local_buf = torch.empty((len(gq) * k, 2), dtype=torch.int64, device="cuda")
        prepared = ctx.prepare(gq)
        ctx.set_option("force_upload", 1)  # descriptors H2D every step (end to end)
        info = {"launches": 0, "h2d": 0, "d2h": 0, "rounds": 0}

        def step():
            res, st = sharded_batch(ctx, gq, prepared=prepared, local=local_buf)
            info["launches"] += st["local"].get("kernel_launches", 0) + st["merge"].get("kernel_launches", 0)
            info["h2d"] += st["local"].get("h2d_bytes", 0) + st["merge"].get("h2d_bytes", 0)
            info["d2h"] += st["merge"].get("d2h_bytes", 0)
            info["rounds"] += st["gather_rounds"]
            return res

        for _ in range(warmup):
            step()
        info.update(launches=0, h2d=0, d2h=0, rounds=0)
        dist.barrier()
        torch.cuda.synchronize()
        dev_ms, wall_ms, res = timed_loop(stream, steps, step, flush)
        dev_ms, wall_ms = reduce_max(dev_ms), reduce_max(wall_ms)
        out = {"products": shape.total, "queries": len(gq), "k": k, "ms_per_step": dev_ms,
               "products_per_s": shape.total * len(gq) / (dev_ms * 1e-3),
               "e2e_ms_per_step": wall_ms, "e2e_products_per_s": shape.total * len(gq) / (wall_ms * 1e-3),
               "gpu_launches": info["launches"], "h2d_bytes_per_step": info["h2d"] // steps,
               "d2h_bytes_per_step": info["d2h"] // steps, "gather_rounds_per_step": info["rounds"] / steps}
        # N = 1 point of the same workload, and exact parity (rank 0's GPU alone)
        if single is not None:
            pb = single.prepare(gq)
            for _ in range(warmup):
                single.run_async(pb)
                single.query_fetch()

            def one():
                single.run_async(pb)

            ms1, _, _ = timed_loop(stream, steps, one, flush)
            glob, _ = single.query_fetch()
            single.close()
            out["single_gpu"] = {"ms_per_step": ms1, "products_per_s": shape.total * len(gq) / (ms1 * 1e-3),
                                 "call": "apex_query_async/fetch on rank 0's GPU, whole range"}
            out["multi_gpu_parity"] = all(results_equal(x, y) for x, y in zip(res, glob))
        dist.barrier()
        ctx.close()
        return shape, queries_named, out

    with (sampler if sampler else _Null()):
        shape, queries_named, c3 = strong(args.config, args.steps, args.warmup)
    c4 = None
    if not args.no_c4 and args.config != "c4" and not args.profile:
        try:
            _, _, c4 = strong("c4", max(3, args.steps // 2), 2)
            c4["workload"] = "c4: one query (5 property windows, k=10000) over the synthetic ~5e9-product CSL"
        except Exception as exc:  # noqa: BLE001
            c4 = {"error": str(exc)[:200]}
    if rank == 0:
        line = {
            "metric": "products scored/sec", "value": c3["products_per_s"], "unit": "products/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": c3["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded CSL shape, random-init heads, calibrated properties)",
            "config": config_dict(args, shape, queries_named, world),
            "e2e": {"value": c3["e2e_products_per_s"], "unit": "products/s",
                    "h2d_bytes_per_step": c3["h2d_bytes_per_step"], "d2h_bytes_per_step": c3["d2h_bytes_per_step"],
                    "ms_per_step": c3["e2e_ms_per_step"],
                    "call": "dist.sharded_batch: apex_query_local_async -> NCCL all-gather -> "
                            "apex_merge_finalize_batch (result rows to host) -> apex_query_local_finish"},
            "gpu_launches": c3["gpu_launches"], "single_gpu": c3.get("single_gpu"),
            "multi_gpu_parity": c3.get("multi_gpu_parity"), "gather_rounds_per_step": c3["gather_rounds_per_step"],
            "c4": c4, "clocks": sampler.summary() if sampler else None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    sys.exit(main())
