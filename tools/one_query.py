#!/usr/bin/env python3
"""Profile helper: one config-5 query (index i) on a library shape, run a few
times (for ncu -k ... -s/-c).  Usage: python tools/one_query.py SHAPE I [opt=v,...]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import _native, synth  # noqa: E402


def main():
    lib, i = sys.argv[1], int(sys.argv[2])
    opts = dict(kv.split("=") for kv in sys.argv[3].split(",")) if len(sys.argv) > 3 and sys.argv[3] != "-" else {}
    shape = synth.make_shape(synth.SHAPES[lib])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    ctx = _native.DeviceContext(0)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b, want_values=False)
    for k, v in opts.items():
        ctx.set_option(k, int(v))
    q = synth.to_native(synth.c5_queries(max(i + 1, 1000))[i], 0, shape.total)
    pb = ctx.prepare([q])
    for _ in range(4):
        r, st = ctx.run(pb)
    print(synth.c5_queries(max(i + 1, 1000))[i], "full" if r[0]["full_predicate"] else "admission",
          {k_: round(v, 4) if isinstance(v, float) else v for k_, v in st.items()})


if __name__ == "__main__":
    main()
