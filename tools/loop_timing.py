#!/usr/bin/env python3
"""Device time per batched pass in the bench's timed-loop form, three ways:
query_async (descriptors built per call), run_async (prepared descriptors),
and run_async without the L2 flush — to separate host, flush and device costs."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import __graft_entry__ as g  # noqa: E402

g.build()
import torch  # noqa: E402

from paper_2510_24380_b200 import _native, synth  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    base = "c1" if cfg == "c2" else cfg
    shape = synth.make_shape(synth.SHAPES[base])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _native.DeviceContext(0, stream.cuda_stream)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b, want_values=False)
    qs = {"c1": [synth.c1_query()], "c2": synth.c2_queries(), "c3": [synth.c3_query()],
          "c4": [synth.c4_query()]}[cfg]
    nq = [synth.to_native(q, 0, shape.total) for q in qs]
    pb = ctx.prepare(nq)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    sys.path.insert(0, str(ROOT))
    import bench
    for mode in ("query_async", "run_async", "run_async_noflush", "run_async_synced", "query_async_sampler",
                 "run_async_sampler"):
        sampler = bench.ClockSampler(0) if mode.endswith("sampler") else bench._Null()
        for _ in range(5):
            ctx.run_async(pb)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        sampler.__enter__()
        for i in range(20):
            if mode != "run_async_noflush":
                flush.zero_()
            if mode == "run_async_synced":
                torch.cuda.synchronize()
            ev[i][0].record(stream)
            if mode.startswith("query_async"):
                ctx.query_async(nq)
            else:
                ctx.run_async(pb)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        sampler.__exit__(None, None, None)
        ms = [s.elapsed_time(t) for s, t in ev]
        print(mode, "ms/step mean %.4f min %.4f" % (sum(ms) / len(ms), min(ms)))
        ctx.query_fetch()


if __name__ == "__main__":
    main()
