#!/usr/bin/env python3
"""Config 5 through the drop-in operator API (engine.search_topk_stream), as
bench.py's c5_query_ms: per-query wall ms with k, and the slowest queries.
Usage: python tools/c5_api.py [n]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import __graft_entry__ as g  # noqa: E402

g.build()
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_2510_24380_b200 import engine, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
shape = synth.make_shape(synth.SHAPES["c3"])
u, w, b = bench.build_model(shape)
values = synth.host_table(u, w) if shape.n_pairs < 400_000 else None
del u
library, table = synth.mirror_objects(shape, values, b)
qs = [synth.query_spec(q) for q in synth.c5_queries()[:n]]
engine.search_topk_stream(library, table, qs[0])
rows = []
for i, q in enumerate(qs):
    t0 = time.perf_counter()
    r = engine.search_topk_stream(library, table, q)
    dt = (time.perf_counter() - t0) * 1e3
    rows.append({"i": i, "ms": round(dt, 3), "k": q.k, "n_cons": len(q.constraints), "retained": r.retained,
                 "timing": {k: round(v, 3) for k, v in (r.timing or {}).items()}})
lat = np.array([r["ms"] for r in rows])
print(json.dumps({"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)), "mean": float(lat.mean()),
                  "slowest": sorted(rows, key=lambda r: -r["ms"])[:6]}))
