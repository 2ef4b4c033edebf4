#!/usr/bin/env python3
"""Device stage breakdown of the config-2 batched pass (stream events between
the pipeline stages, graph replay): init/pack, seed, scan (incl. waiting for the
constraint pre-pass), scan kernel alone, select, finalize.  Medians of 31
passes.  A/B knobs: APEX_OPTS="name=value,...", APEX_B200_LIB=<lib>.
Usage: python tools/c2_stages.py"""
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

shape = synth.make_shape(synth.SHAPES["c1"])
u, w, b = synth.build_model(shape)
ctx = _native.DeviceContext(0)
ctx.set_option("stages", 1)  # per-stage events (diagnostics)
for kv in filter(None, os.environ.get("APEX_OPTS", "").split(",")):
    name, val = kv.split("=")
    ctx.set_option(name, int(val))
ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
ctx.load_cache(u, w, b)
nq = [synth.to_native(q, 0, shape.total) for q in synth.c2_queries()]
keys = ("pack_ms", "seed_ms", "scan_ms", "scan_kernel_ms", "select_ms", "finalize_ms", "total_ms")
rows = []
for _ in range(31):
    _, st = ctx.query(nq)
    rows.append(st)
out = {k: round(statistics.median(r[k] for r in rows), 4) for k in keys}
out["device_ms"] = round(statistics.median(sum(r[k] for k in keys[:3] + keys[4:6]) for r in rows), 4)
out["lib"] = os.path.basename(os.environ.get("APEX_B200_LIB", "in-tree"))
out["opts"] = os.environ.get("APEX_OPTS", "")
print(json.dumps(out))
