#!/usr/bin/env python3
"""BASELINE config 5: amortised query sweep — 1,000 random objective /
constraint combinations over the 1B-product CSL, reusing the resident table.
Reports per-query latency p50/p99 (each query its own apex_query call, host
wall clock incl. result D2H), the batched throughput (all queries in one
pass), and a consistency check of a sample of batched results against the
single-query results.  Usage: python tools/c5_check.py [n_queries] [c3|c1]"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import _native, synth  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    lib = sys.argv[2] if len(sys.argv) > 2 else "c3"
    opts = dict(kv.split("=") for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 and sys.argv[3] != "-" else {}
    single = os.environ.get("C5_SINGLE", "1") == "1"
    shape = synth.make_shape(synth.SHAPES[lib])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    ctx = _native.DeviceContext(0)
    ctx.set_option("stages", 1)  # per-stage events (diagnostics)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b, want_values=False)
    for k_, v in opts.items():
        ctx.set_option(k_, int(v))
    qs = [synth.to_native(q, 0, shape.total) for q in synth.c5_queries(n)]
    # per-query latency (each query alone, prepared host buffers)
    pbs = [ctx.prepare([q]) for q in qs] if single else []
    for pb in pbs[:5]:
        ctx.run(pb)
    lat, single, full, kern, cand, tot = [], [], [], [], [], []
    detail = []
    for qi, pb in enumerate(pbs):
        t0 = time.perf_counter()
        r, st1 = ctx.run(pb)
        lat.append((time.perf_counter() - t0) * 1e3)
        detail.append({"i": qi, "ms": round(lat[-1], 3), "k": qs[qi]["k"], "n_cons": len(qs[qi].get("cons", [])),
                       "full": bool(r[0]["full_predicate"]), "cand": st1["candidates"], "admitted": st1.get("admitted"), "retries": st1["retries"],
                       "seed": round(st1["seed_ms"], 3), "scan": round(st1["scan_kernel_ms"], 3),
                       "select": round(st1["select_ms"], 3), "total": round(st1["total_ms"], 3)})
        single.append((r[0]["g"].copy(), r[0]["objective"].copy()))
        full.append(r[0]["full_predicate"])
        kern.append(st1["scan_kernel_ms"])
        tot.append(st1["total_ms"])
        cand.append(st1["candidates"])
    lat, full, kern = np.array(lat or [0.0]), np.array(full or [False], dtype=bool), np.array(kern or [0.0])
    tot = np.array(tot)
    # batched: all queries in one pass
    pb = ctx.prepare(qs)
    ctx.run(pb)
    t0 = time.perf_counter()
    res, st = ctx.run(pb)
    wall = time.perf_counter() - t0
    ok = all(np.array_equal(res[i]["g"], single[i][0]) and np.array_equal(res[i]["objective"], single[i][1])
             for i in range(len(single)))
    print(json.dumps({
        "config": f"c5: {len(qs)} random objective/constraint queries (k in 100/1000/10000) over {shape.total} products",
        "latency_ms": {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                       "mean": float(lat.mean()), "max": float(lat.max())},
        "single_query_products_per_s": shape.total * len(qs) / (lat.sum() * 1e-3),
        "batched": {"wall_ms": wall * 1e3, "products_per_s": shape.total * len(qs) / wall,
                    "scan_kernel_ms": st["scan_kernel_ms"], "seed_ms": st["seed_ms"], "select_ms": st["select_ms"],
                    "d2h_ms": st["d2h_ms"], "total_ms": st["total_ms"]},
        "batched_equals_single": bool(ok),
        "full_predicate_queries": int(full.sum()),
        "scan_kernel_ms_mean": {"admission": float(kern[~full].mean()) if (~full).any() else None,
                                "full": float(kern[full].mean()) if full.any() else None},
        "retries_batched": st["retries"], "candidates_mean": float(np.mean(cand)),
        "scan_kernel_ms_p50": float(np.percentile(kern, 50)), "scan_kernel_ms_p99": float(np.percentile(kern, 99)),
        "device_total_ms_p50": float(np.percentile(tot, 50)) if len(tot) else None,
        "host_ms_p50": float(np.percentile(lat - tot, 50)) if len(tot) == len(lat) else None,
        "slowest": sorted(detail, key=lambda d: -d["ms"])[:8]}))


if __name__ == "__main__":
    main()
