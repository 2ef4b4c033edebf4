#!/usr/bin/env python3
"""Benchmark of the B200 enumeration-and-retrieval path (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|c3|c4]

Workload (BASELINE.json configs[1], "c2"): a synthetic 10M-product CSL of the
config-1 shape (40 reactions, mixed 2/3-component), random-init
linear heads on a synthetic embedding cache (property heads calibrated), and
20 queries (dock_a..e minimize x {lipinski, veber, pfizer_3_75, astex_ro3},
k=1000) answered in ONE batched device pass.  A step = one such pass.  With
N GPUs the library is N x 10M products and each rank scans its contiguous
1/N of the index space (weak scaling), then the per-rank top-k entries are
all-gathered (NCCL) and merged exactly on every rank.

metric: products scored per second = (products in the library) x (queries)
per step / step time.  `value` times the device pipeline with the table
resident in HBM (apex_query_async, CUDA events on the launching stream, L2
flushed between steps); `e2e` times the public C-ABI call apex_query with host
buffers (query descriptors H2D every step, result rows D2H into caller-owned
host arrays that are allocated once and reused, host sync).

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
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-procs", type=int, default=0)
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no clocks, no baselines)")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (5e9-product) roofline and effective passes")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def workload(config: str, world: int):
    base = "c1" if config in ("c1", "c2") else config
    shape = synth.scaled_shape(base, world) if world > 1 else synth.make_shape(synth.SHAPES[base])
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


def cpu_pass(pool, procs, lib, queries, start, end):
    """Exact top-k of every query over [start, end) with `procs` processes
    (contiguous index-range shards + exact merge)."""
    tasks = [(qi, start + (end - start) * r // procs, start + (end - start) * (r + 1) // procs)
             for qi in range(len(queries)) for r in range(procs)]
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
    products = shape.total * len(qs)
    for _ in range(args.warmup):
        cpu_pass(pool, procs, lib, qs, 0, lib.total)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_pass(pool, procs, lib, qs, 0, lib.total)
    dt = time.perf_counter() - t0
    pool.close()
    value = products * args.steps / dt
    line = {
        "impl": "reference", "metric": "products scored/sec", "value": value, "unit": "products/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(args, shape, queries_named, world),
        "cpu_baseline": {"value": value, "unit": "products/s", "cores": procs, "kind": "port",
                         "sample": f"full pass: {len(qs)} queries x {shape.total} products per step "
                                   f"(oracle/scan_oracle.py restating engine.search_topk_stream)"},
        "e2e": {"value": value, "unit": "products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args, shape, queries_named, world):
    return {
        "workload": f"{args.config}: synthetic {shape.total / 1e6:.1f}M-product CSL ({len(shape.sizes)} reactions, "
                    f"mixed 2/3-component), {len(queries_named)} quer{'y' if len(queries_named) == 1 else 'ies'} "
                    f"(k={queries_named[0]['k']}) in one batched pass",
        "products": shape.total, "queries": len(queries_named), "k": queries_named[0]["k"],
        "products_per_step": shape.total * len(queries_named), "pair_rows": shape.n_pairs,
        "parallelism": f"index-range shards x{world}" if world > 1 else "single GPU",
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


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    if os.environ.get("APEX_BENCH_BACKEND", "nccl") != "nccl":
        local %= torch.cuda.device_count()  # shared-GPU logic test (not a timing mode)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink; APEX_BENCH_BACKEND=gloo only to exercise the
        # multi-rank logic when several ranks share one GPU (not a timing mode)
        backend = os.environ.get("APEX_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    import __graft_entry__ as g
    g.build()
    from paper_2510_24380_b200 import _native
    from paper_2510_24380_b200.dist import PAD, all_gather_entries, shard_range

    shape, queries_named = workload(args.config, world)
    u, w, b = build_model(shape)
    # a real (non-default) torch stream shared with the C-ABI context, so the
    # CUDA events below bracket exactly the work the library enqueues
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _native.DeviceContext(local, stream.cuda_stream)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    values = ctx.load_cache(u, w, b)
    a, e = shard_range(0, shape.total, rank, world)
    nqueries = [synth.to_native(q, a, e) for q in queries_named]
    products = shape.total * len(nqueries)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    k = nqueries[0]["k"]

    prepared_dev = ctx.prepare(nqueries) if world == 1 else None  # descriptors built once (device-resident pass)

    def step_device():
        return ctx.run_async(prepared_dev)

    gqueries = [dict(q, start=0, end=shape.total) for q in nqueries]
    merge_prepared = ctx.prepare(gqueries) if world > 1 else None  # caller-owned host result arrays, reused
    local_buf = torch.full((len(nqueries) * k, 2), PAD, dtype=torch.int64, device="cuda") if world > 1 else None

    def step_multi():
        # local scan of this rank's shard for the whole batch, ONE all-gather
        # of the [queries][k] entry buffers (NCCL), ONE batched exact merge
        local_buf.fill_(PAD)
        counts, st = ctx.query_local(nqueries, local_buf.data_ptr())
        gathered = all_gather_entries(local_buf)
        res, st2 = ctx.merge_finalize_batch(gqueries, gathered.data_ptr(), world, k, shape.total, merge_prepared)
        step_multi.h2d = st["h2d_bytes"]
        step_multi.scan_ms = st["scan_kernel_ms"]
        step_multi.d2h = st2["d2h_bytes"]
        return st["kernel_launches"] + st2["kernel_launches"], res

    # warmup
    for _ in range(args.warmup):
        if world == 1:
            step_device()
            ctx.query_fetch()
        else:
            step_multi()
    torch.cuda.synchronize()

    # timed: device-resident pass
    launches = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local) if not args.profile else None
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with (sampler if sampler else _Null()):
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            if world == 1:
                st = step_device()
                launches += st["kernel_launches"]
            else:
                n, _ = step_multi()
                launches += n
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    ms = sum(s.elapsed_time(t) for s, t in ev)
    if world > 1:
        ms = reduce_max(ms)
    if world == 1:
        res_dev, st_dev = ctx.query_fetch()  # validates the last in-flight pass (overflow check)
    ms_per_step = ms / args.steps
    value = products / (ms_per_step * 1e-3)

    # e2e: public C-ABI call with host buffers, descriptors H2D every step
    ctx.set_option("force_upload", 1)
    # results returned as views into the library's pinned host block (D2H in
    # the same device pass, no host-side copy): the C-ABI view mode
    prepared = ctx.prepare_views(nqueries) if world == 1 else None
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    scan_ms, h2d, d2h = [], 0, 0
    for i in range(args.steps):
        flush.zero_()
        e2e_ev[i][0].record(stream)
        t0 = time.perf_counter()
        if world == 1:
            res, st = ctx.run_views(prepared)
            scan_ms.append(st["scan_kernel_ms"])
            h2d += st["h2d_bytes"]
            d2h += st["d2h_bytes"]
        else:
            _, res_multi = step_multi()
            h2d += step_multi.h2d
            d2h += step_multi.d2h
            scan_ms.append(step_multi.scan_ms)
        e2e_ev[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = sum(s.elapsed_time(t) for s, t in e2e_ev)
    if world > 1:
        e2e_ms = reduce_max(e2e_ms)
    ctx.set_option("force_upload", 0)
    e2e_value = products / (e2e_ms / args.steps * 1e-3)

    # Rooflines.  F = algorithmic FP32 ops per product of the
    # batched pass; peak P32 = SMs x 128 FP32 lanes x the SM clock sampled
    # under load.  The roofline claim uses a pass that evaluates every active
    # test on every product (the full-predicate kernel, mode 0); the default
    # sorted-column kernel skips products that cannot pass and is reported
    # as "effective" (F-equivalent rate of the same pass).
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    sm_count = ctx.device_info()[0]
    clk = sampler.summary() if sampler else None
    clk_mhz = float((clk or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0))
    peak_tops = sm_count * 128 * clk_mhz * 1e6 / 1e12
    scanned = e - a
    F = f_ops(queries_named)
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(args.config)
        except Exception:
            traffic = None
    kern_ms = statistics.mean(scan_ms) if scan_ms else None
    effective = None
    if kern_ms:
        eq = scanned * F / (kern_ms * 1e-3) / 1e12
        effective = {"products_per_s": scanned * len(nqueries) / (kern_ms * 1e-3), "kernel_ms": kern_ms,
                     "F_equivalent_tops": eq, "frac_equivalent": eq / peak_tops,
                     "kernel": "scan_sorted_kernel (per-row threshold + most selective test's sorted range)",
                     "note": "pruned: products that cannot pass are never evaluated, so the F-equivalent "
                             "rate can exceed the FP32 peak"}
    roofline = None
    if world == 1 and not args.profile:
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

    # the SURVEY's roofline reference point: the C4 query over the ~5e9-product
    # library (F = 15 per product), full-predicate pass (mode 0) and the
    # default sorted-column pass, on a second context with that table resident
    roofline_c4 = effective_c4 = None
    if world == 1 and not args.profile and not args.no_c4 and args.config != "c4":
        try:
            c4shape, c4q = workload("c4", 1)
            u4, w4, b4 = build_model(c4shape)
            ctx4 = _native.DeviceContext(local, stream.cuda_stream)
            ctx4.load_library(c4shape.sizes, c4shape.pair_off, c4shape.g_offsets(), c4shape.n_pairs)
            ctx4.load_cache(u4, w4, b4, want_values=False)
            del u4
            q4 = [synth.to_native(q, 0, c4shape.total) for q in c4q]
            F4 = f_ops(c4q)
            pb4 = ctx4.prepare_views(q4)
            times = {}
            for mode in (0, 3):
                ctx4.set_option("mode", mode)
                ctx4.run_views(pb4)
                ms4 = []
                for _ in range(3):
                    flush.zero_()
                    _, st4 = ctx4.run_views(pb4)
                    ms4.append(st4["scan_kernel_ms"])
                times[mode] = statistics.median(ms4)
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
            ctx4.close()
        except Exception as exc:  # noqa: BLE001 - reported, never fatal for the headline line
            roofline_c4 = {"error": str(exc)[:200]}

    # K1 precompute (HBM-bound) at the C4 table size: u fp64
    # [n_pairs, 64] generated on the device, one timed launch after warm-up;
    # algorithmic bytes = 8*d*n_pairs (u) + 8*n_tasks*d (heads) + 4*n_tasks*n_pairs (table)
    precompute = None
    if world == 1 and not args.profile:
        try:
            c4 = synth.make_shape(synth.SHAPES["c4"])
            n_p, d_, n_t = c4.n_pairs, 64, len(synth.TASKS)
            u_dev = torch.randn((n_p, d_), dtype=torch.float64, device="cuda")
            w_dev = torch.randn((n_t, d_), dtype=torch.float64, device="cuda") * 0.01
            v_dev = torch.empty((n_t, n_p), dtype=torch.float32, device="cuda")
            for _ in range(3):
                ctx.precompute_device(u_dev.data_ptr(), n_p, d_, w_dev.data_ptr(), n_t, v_dev.data_ptr())
            pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for e0, e1 in pe:
                flush.zero_()
                e0.record(stream)
                ctx.precompute_device(u_dev.data_ptr(), n_p, d_, w_dev.data_ptr(), n_t, v_dev.data_ptr())
                e1.record(stream)
            torch.cuda.synchronize()
            pms = statistics.median(s_.elapsed_time(t_) for s_, t_ in pe)
            pbytes = 8 * d_ * n_p + 8 * n_t * d_ + 4 * n_t * n_p
            hbm = float(peaks.get("hbm_gbs", 6550.7))
            precompute = {"kernel": "precompute_rows_kernel<11,64> (K1, fp64 head x u dots, fp32 table)", "n_pairs": n_p, "d": d_,
                          "n_tasks": n_t, "ms": pms, "bytes": pbytes, "achieved_GBps": pbytes / (pms * 1e-3) / 1e9,
                          "peak_GBps": hbm, "frac": pbytes / (pms * 1e-3) / 1e9 / hbm,
                          "peak_basis": "MEASURED_PEAKS hbm_gbs (copy bandwidth)"}
            del u_dev, w_dev, v_dev
        except Exception as exc:  # noqa: BLE001 - reported, never fatal for the headline line
            precompute = {"error": str(exc)[:200]}

    line = {
        "metric": "products scored/sec", "value": value, "unit": "products/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded CSL shape, random-init heads, calibrated properties)",
        "config": config_dict(args, shape, queries_named, world),
        "e2e": {"value": e2e_value, "unit": "products/s", "h2d_bytes_per_step": h2d // max(args.steps, 1),
                "d2h_bytes_per_step": d2h // max(args.steps, 1), "ms_per_step": e2e_ms / args.steps},
        "gpu_launches": launches, "roofline": roofline, "effective": effective, "roofline_c4": roofline_c4,
        "effective_c4": effective_c4, "precompute": precompute,
        "clocks": sampler.summary() if sampler else None,
    }
    if world == 1:
        line["device_stages_ms"] = {k_: st_dev[k_] for k_ in ("pack_ms", "seed_ms", "scan_ms", "select_ms",
                                                              "finalize_ms", "d2h_ms", "total_ms",
                                                              "scan_kernel_ms")}
        line["candidates_per_step"] = st_dev["candidates"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile:
        procs = cpu_procs(args)
        pool, lib, qs = cpu_setup(shape, values, b, queries_named, procs)
        t0 = time.perf_counter()
        cpu_out = cpu_pass(pool, procs, lib, qs, 0, lib.total)
        dt = time.perf_counter() - t0
        pool.close()
        # parity of the benchmarked pass itself (same inputs, bit-exact)
        ok = all(np.array_equal(r["g"].astype(np.int64), co[1]) for r, co in zip(res, cpu_out))
        line["cpu_baseline"] = {"value": products / dt, "unit": "products/s", "cores": procs, "kind": "port",
                                "sample": f"full pass ({len(qs)} queries x {shape.total} products), "
                                          "oracle/scan_oracle.py", "parity_with_gpu": ok}
    if world > 1 and rank == 0:
        # the merged multi-rank result against one global pass on this GPU
        # (every rank holds the whole table; outside the timed regions)
        glob, _ = ctx.query(gqueries)
        line["multi_gpu_parity"] = all(
            np.array_equal(m["g"], gq["g"]) and np.array_equal(m["objective"], gq["objective"])
            for m, gq in zip(res_multi, glob))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


if __name__ == "__main__":
    sys.exit(main())
