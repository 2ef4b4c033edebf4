import sys, time
sys.path.insert(0, "/root/repo")
import __graft_entry__ as g
g.build()
import torch
from paper_2510_24380_b200 import _native, synth
shape = synth.make_shape(synth.SHAPES["c1"])
u = synth.random_cache(shape.n_pairs, seed=1)
w, b = synth.random_heads(seed=1)
w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
ctx = _native.DeviceContext(0)
ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
ctx.load_cache(u, w, b, want_values=False)
nq = [synth.to_native(q, 0, shape.total) for q in synth.c2_queries()]
for _ in range(5):
    ctx.query_async(nq); ctx.query_fetch()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    t0 = time.perf_counter(); ctx.query_async(nq); t1 = time.perf_counter(); ts.append(t1 - t0)
    ctx.query_fetch()
print("query_async host us: median", sorted(ts)[10] * 1e6)
specs, keep = ctx._specs(nq)
t0 = time.perf_counter()
for _ in range(100): ctx._specs(nq)
print("_specs us", (time.perf_counter() - t0) / 100 * 1e6)
import ctypes as C
st = _native.Stats()
ts = []
for _ in range(20):
    t0 = time.perf_counter(); ctx.lib.apex_query_async(ctx._ctx, specs, len(nq), C.byref(st)); t1 = time.perf_counter(); ts.append(t1 - t0)
    ctx._inflight = nq; ctx.query_fetch()
print("apex_query_async C-only host us: median", sorted(ts)[10] * 1e6)
print("last stats: prepare us", st.host_prepare_us, "launch us", st.host_launch_us)
pb = ctx.prepare(nq)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); s2 = ctx.run_async(pb); t1 = time.perf_counter(); ts.append(t1 - t0)
    ctx.query_fetch()
print("run_async (prepared) host us: median", sorted(ts)[10] * 1e6, s2["host_prepare_us"], s2["host_launch_us"])

for name, fn, arg in (("run (copy)", ctx.run, ctx.prepare(nq)), ("run_views", ctx.run_views, ctx.prepare_views(nq))):
    for _ in range(3):
        fn(arg)
    ts = []
    for _ in range(20):
        t0 = time.perf_counter(); r, st = fn(arg); ts.append(time.perf_counter() - t0)
    print(name, "wall us median", sorted(ts)[10] * 1e6, "prep", st["host_prepare_us"], "launch", st["host_launch_us"],
          "d2h_ms", st["d2h_ms"], "total_ms", st["total_ms"])
