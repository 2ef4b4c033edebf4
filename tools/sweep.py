#!/usr/bin/env python3
"""Option sweep of the device pipeline on a config shape (tuning aid; prints
per-stage device times).  Usage: python tools/sweep.py c3 [opt=v,...] ..."""

import json
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
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    variants = [dict(kv.split("=") for kv in a.split(",")) if a != "-" else {} for a in sys.argv[2:]] or [{}]
    base = "c1" if cfg in ("c2", "c5") else cfg
    shape = synth.make_shape(synth.SHAPES[base])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    ctx = _native.DeviceContext(0)
    ctx.set_option("stages", 1)  # per-stage events (diagnostics)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b, want_values=False)
    qs = {"c1": [synth.c1_query()], "c2": synth.c2_queries(), "c3": [synth.c3_query()],
          "c4": [synth.c4_query()], "c5": synth.c5_queries()}[cfg]
    nq = [synth.to_native(q, 0, shape.total) for q in qs]
    for v in variants:
        for k_, val in v.items():
            ctx.set_option(k_, int(val))
        ctx.query(nq)
        sts = []
        t0 = time.perf_counter()
        for _ in range(5):
            _, st = ctx.query(nq)
            sts.append(st)
        wall = (time.perf_counter() - t0) / 5
        keys = ("pack_ms", "seed_ms", "scan_ms", "select_ms", "finalize_ms", "d2h_ms", "total_ms", "scan_kernel_ms")
        med = {k_: float(np.median([s[k_] for s in sts])) for k_ in keys}
        med["candidates"] = sts[-1]["candidates"]
        med["admitted"] = sts[-1]["admitted"]
        med["wall_ms"] = wall * 1e3
        med["products_per_s_scan"] = shape.total * len(nq) / (med["scan_kernel_ms"] * 1e-3)
        print(json.dumps({"config": cfg, "opts": v, **{k_: round(x, 4) if isinstance(x, float) else x
                                                       for k_, x in med.items()}}), flush=True)


if __name__ == "__main__":
    main()
