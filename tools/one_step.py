#!/usr/bin/env python3
"""One profiled device pass of a config (for `ncu --profile-from-start off`):
warm-up passes, then cudaProfilerStart / one apex_query / cudaProfilerStop.
Usage: python tools/one_step.py c2 [opt=v,...]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import _native, synth  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    opts = dict(kv.split("=") for kv in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] != "-" else {}
    base = "c1" if cfg == "c2" else cfg
    shape = synth.make_shape(synth.SHAPES[base])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    ctx = _native.DeviceContext(0)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b, want_values=False)
    qs = {"c1": [synth.c1_query()], "c2": synth.c2_queries(), "c3": [synth.c3_query()],
          "c4": [synth.c4_query()]}[cfg]
    nq = [synth.to_native(q, 0, shape.total) for q in qs]
    for k, v in opts.items():
        ctx.set_option(k, int(v))
    pb = ctx.prepare(nq)
    for _ in range(3):
        ctx.run(pb)
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    _, st = ctx.run(pb)
    torch.cuda.profiler.stop()
    print(st)


if __name__ == "__main__":
    main()
