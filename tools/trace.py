#!/usr/bin/env python3
"""Per-item timeline of the admission scan (tuning aid): which SMs finish
last and which work items are the long ones.  Usage: python tools/trace.py c4 [opt=v,...]"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import _native, synth  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    opts = dict(kv.split("=") for kv in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] != "-" else {}
    base = "c1" if cfg == "c2" else cfg
    shape = synth.make_shape(synth.SHAPES[base])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000, seed=1)
    ctx = _native.DeviceContext(0)
    ctx.set_option("stages", 1)  # per-stage events (diagnostics)
    ctx.load_library(shape.sizes, shape.pair_off, shape.g_offsets(), shape.n_pairs)
    ctx.load_cache(u, w, b, want_values=False)
    qs = {"c1": [synth.c1_query()], "c2": synth.c2_queries(), "c3": [synth.c3_query()],
          "c4": [synth.c4_query()]}[cfg]
    nq = [synth.to_native(q, 0, shape.total) for q in qs]
    cap = 1 << 24
    for k, v in opts.items():
        ctx.set_option(k, int(v))
    ctx.set_option("trace", cap)
    for _ in range(3):
        _, st = ctx.query(nq)
    tr = ctx.debug_trace(cap)
    tr = tr[tr[:, 1] > 0]
    t0 = tr[:, 0].min()
    s, e = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3
    dur = e - s
    sm = (tr[:, 2] & 0xff).astype(int)
    rare = ((tr[:, 2] >> 8) & 0xffffff).astype(int)
    ncols = ((tr[:, 3] >> 8) & 0xffffff).astype(int)
    nrows = (tr[:, 3] & 0xff).astype(int)
    rx = (tr[:, 3] >> 32).astype(int)
    cyc_rare, cyc_thr, cyc_stage, cand = (tr[:, 4] / 1e3, tr[:, 5] / 1e3, tr[:, 6] / 1e3, tr[:, 7].astype(int))
    print(f"items {len(tr)}  span {e.max():.1f} us  scan_kernel_ms {st['scan_kernel_ms']:.4f}")
    sm_end = np.zeros(sm.max() + 1)
    np.maximum.at(sm_end, sm, e)
    q = np.percentile(sm_end, [0, 10, 50, 90, 100])
    print("SM last-item end (us) min/p10/p50/p90/max:", np.round(q, 1))
    print("item duration (us) p50/p90/p99/max:", np.round(np.percentile(dur, [50, 90, 99, 100]), 2))
    prod = ncols * nrows
    print("ns per product (sum dur / sum products):", dur.sum() * 1e3 / prod.sum())
    order = np.argsort(-dur)[:15]
    print("longest items: dur_us start_us sm rare nrows ncols rx | kcyc rare thr stage | cands")
    for i in order:
        print(f"  {dur[i]:9.2f} {s[i]:9.1f} {sm[i]:4d} {rare[i]:6d} {nrows[i]:4d} {ncols[i]:6d} {rx[i]:5d} |"
              f" {cyc_rare[i]:8.1f} {cyc_thr[i]:7.1f} {cyc_stage[i]:7.1f} | {cand[i]:6d}")
    print("totals: rare entries %d  kcyc rare %.0f thr %.0f stage %.0f  cands %d" %
          (rare.sum(), cyc_rare.sum(), cyc_thr.sum(), cyc_stage.sum(), cand.sum()))
    late = np.argsort(-e)[:10]
    print("last-finishing items: end_us dur_us sm rare nrows ncols rx")
    for i in late:
        print(f"  {e[i]:9.1f} {dur[i]:9.2f} {sm[i]:4d} {rare[i]:6d} {nrows[i]:4d} {ncols[i]:6d} {rx[i]:5d}")
    # cost model: duration vs products and rare entries
    A = np.stack([np.ones_like(dur), prod / 1e3, rare, nrows], 1)
    coef, *_ = np.linalg.lstsq(A, dur, rcond=None)
    print("fit dur_us = %.3f + %.4f*kprod + %.4f*rare + %.4f*nrows" % tuple(coef))


if __name__ == "__main__":
    main()
