#!/usr/bin/env python3
"""Scan-kernel time of each config-2 query alone, of each preset group (the 5
objectives sharing a constraint set) and of the whole 20-query batch: where
the batched pass's enumeration time goes.  Usage: python tools/c2_per_query.py"""
import json
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import _native, synth  # noqa: E402


def med(ctx, qs, reps=7):
    ms, tot, cand = [], [], 0
    for _ in range(reps):
        _, st = ctx.query(qs)
        ms.append(st["scan_kernel_ms"])
        tot.append(st["total_ms"])
        cand = st["candidates"]
    return statistics.median(ms), statistics.median(tot), cand


shape = synth.make_shape(synth.SHAPES["c1"])
u, w, b = synth.build_model(shape)
ctx = _native.DeviceContext(0)
ctx.set_option("stages", 1)  # per-stage events (diagnostics)
# A/B knobs: APEX_OPTS="name=value,name=value" (apex_set_option)
for kv in filter(None, os.environ.get("APEX_OPTS", "").split(",")):
    name, val = kv.split("=")
    ctx.set_option(name, int(val))
ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
ctx.load_cache(u, w, b)
qs = synth.c2_queries()
nq = [synth.to_native(q, 0, shape.total) for q in qs]
out = {"batch": med(ctx, nq)}
for name in ("lipinski", "veber", "pfizer_3_75", "astex_ro3"):
    grp = [x for q, x in zip(qs, nq) if q["name"].endswith(name)]
    out["group/" + name] = med(ctx, grp)
for q, x in zip(qs, nq):
    out[q["name"]] = med(ctx, [x])
for k, v in out.items():
    print(json.dumps({"what": k, "scan_kernel_ms": v[0], "total_ms": v[1], "candidates": v[2]}))
