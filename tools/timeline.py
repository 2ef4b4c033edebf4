#!/usr/bin/env python3
"""Concurrent-kernel timeline of one device pass (CUPTI through torch.profiler):
every kernel of the pass with its stream, start offset from the pass's first
kernel and duration, plus idle gaps on the critical path.  Unlike the ncu
launch list (serialised, cold), this is the pass as it runs (graph replay,
side streams overlapping).
Usage: python tools/timeline.py [c2|c1|c3|c4] [opt=v,...]"""
import json
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
    opts = dict(kv.split("=") for kv in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] != "-" else {}
    base = "c1" if cfg == "c2" else cfg
    shape = synth.make_shape(synth.SHAPES[base])
    u, w, b = synth.build_model(shape)
    ctx = _native.DeviceContext(0)
    for k, v in opts.items():
        ctx.set_option(k, int(v))
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b)
    qs = {"c1": [synth.c1_query()], "c2": synth.c2_queries(), "c3": [synth.c3_query()],
          "c4": [synth.c4_query()]}[cfg]
    nq = [synth.to_native(q, 0, shape.total) for q in qs]
    for _ in range(5):
        ctx.query(nq)
    torch.cuda.synchronize()
    passes = 3
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(passes):
            ctx.query(nq)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = []
    for e in evs:
        ks.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", -1), e.name))
    ks.sort()
    # split into passes at the init_ctl kernel
    starts = [i for i, k in enumerate(ks) if "init_ctl" in k[3]]
    out = []
    for pi, s0 in enumerate(starts):
        s1 = starts[pi + 1] if pi + 1 < len(starts) else len(ks)
        grp = ks[s0:s1]
        t0 = grp[0][0]
        rows = []
        for st, en, sid, name in grp:
            short = name.split("(")[0].replace("void ", "").replace("apexb200::", "")
            rows.append({"k": short[:48], "stream": sid, "start_us": round(st - t0, 2), "dur_us": round(en - st, 2)})
        end = max(r["start_us"] + r["dur_us"] for r in rows)
        busy = 0.0
        cur_s = cur_e = None
        for r in sorted(rows, key=lambda r: r["start_us"]):
            s, e = r["start_us"], r["start_us"] + r["dur_us"]
            if cur_e is None or s > cur_e:
                if cur_e is not None:
                    busy += cur_e - cur_s
                cur_s, cur_e = s, e
            else:
                cur_e = max(cur_e, e)
        busy += cur_e - cur_s
        out.append({"pass": pi, "span_us": round(end, 2), "busy_us": round(busy, 2), "kernels": rows})
    for p in out:
        print(f"pass {p['pass']}: span {p['span_us']} us, GPU busy {p['busy_us']} us, {len(p['kernels'])} kernels")
        for r in p["kernels"]:
            print(f"   {r['start_us']:8.2f} +{r['dur_us']:7.2f}  s{r['stream']:<4} {r['k']}")
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"timeline_{cfg}.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
