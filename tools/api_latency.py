#!/usr/bin/env python3
"""End-to-end latency of the public drop-in API (engine.search_topk_stream on
mirror CslLibrary / ContributionTable / QuerySpec objects, results as
ScoredCompound entries) for a config shape: the process's CUDA start-up, the
binding of a (library, table) pair alone (descriptors, table upload, device
sort of the columns, corner lists), the first call (binding + query) and warm
calls.
Usage: python tools/api_latency.py c4 [repeats]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import csl, engine, synth  # noqa: E402


mirror_objects = synth.mirror_objects


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    shape = synth.make_shape(synth.SHAPES[cfg])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    values = synth.host_table(u, w)
    lib, table = mirror_objects(shape, values, np.asarray(b, dtype=np.float64))
    qd = {"c1": synth.c1_query(), "c3": synth.c3_query(), "c4": synth.c4_query()}[cfg]
    q = engine.QuerySpec(qd["objective"], qd["direction"],
                         tuple(engine.Constraint(t, lo, hi) for t, lo, hi in qd["constraints"]), qd["k"])
    # CUDA context + module load happen once per process, before any library
    # is bound: a server pays them at start-up, not per (library, table)
    t0 = time.perf_counter()
    from paper_2510_24380_b200 import _native
    _native.DeviceContext(engine.default_device_one(None)).close()
    process_init = time.perf_counter() - t0
    t0 = time.perf_counter()
    b = engine.bind(lib, table)
    bind_s = time.perf_counter() - t0
    engine._BOUND.clear()
    del b
    t0 = time.perf_counter()
    r = engine.search_topk_stream(lib, table, q)
    first = time.perf_counter() - t0
    warm = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = engine.search_topk_stream(lib, table, q)
        warm.append(time.perf_counter() - t0)
    print(json.dumps({"config": cfg, "products": shape.total, "k": q.k, "retained": r.retained,
                      "process_cuda_init_s": process_init, "bind_s": bind_s,
                      "first_call_s": first, "warm_call_ms_median": float(np.median(warm)) * 1e3,
                      "warm_call_ms_min": float(np.min(warm)) * 1e3,
                      "device_total_ms": r.timing.get("device_total_ms")}))


if __name__ == "__main__":
    main()
