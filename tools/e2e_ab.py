#!/usr/bin/env python3
"""Same-process A/B of the C-ABI end-to-end call (apex_query, view mode:
descriptors H2D every call, rows in pinned host memory on return) on the C2
batch, as bench.py's e2e loop (256 MiB L2 flush before each call, CUDA events
on the context's stream).  Usage: python tools/e2e_ab.py "opt=v,..." "opt=v,..." ..."""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import __graft_entry__ as g  # noqa: E402

g.build()
import torch  # noqa: E402
from paper_2510_24380_b200 import _native, synth  # noqa: E402

shape = synth.make_shape(synth.SHAPES["c1"])
u, w, b = synth.build_model(shape)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = _native.DeviceContext(0, stream.cuda_stream)
ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
ctx.load_cache(u, w, b)
nq = [synth.to_native(q, 0, shape.total) for q in synth.c2_queries()]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for rnd in range(2):
    for arg in sys.argv[1:]:
        opts = dict(kv.split("=") for kv in arg.split(",") if kv)
        for k, v in opts.items():
            ctx.set_option(k, int(v))
        ctx.set_option("force_upload", 1)
        pb = ctx.prepare_views(nq)
        for _ in range(5):
            ctx.run_views_raw(pb)
        ms = []
        for _ in range(30):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r, st = ctx.run_views_raw(pb)
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        res, _ = ctx.views_of(pb, r, st)
        sig = [(x["g"].tobytes(), x["objective"].tobytes(), x["constraint_values"].tobytes(), x["digits"].tobytes())
               for x in res]
        if ref is None:
            ref = sig
        print(json.dumps({"opts": arg, "e2e_ms_p50": round(statistics.median(ms), 4),
                          "same_rows": sig == ref}))
        ctx.set_option("force_upload", 0)
        for k in opts:
            pass
