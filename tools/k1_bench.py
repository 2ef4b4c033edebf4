#!/usr/bin/env python3
"""K1 precompute at the C4 table size (device-generated u), for ncu / timing.
Usage: python tools/k1_bench.py [pre_rows form: 0|1|2]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import __graft_entry__ as g  # noqa: E402

g.build()
import torch  # noqa: E402

from paper_2510_24380_b200 import _native, synth  # noqa: E402


def main():
    form = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    c4 = synth.make_shape(synth.SHAPES["c4"])
    n_p, d, n_t = c4.n_pairs, 64, len(synth.TASKS)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = _native.DeviceContext(0, stream.cuda_stream)
    ctx.set_option("pre_rows", form)
    u = torch.randn((n_p, d), dtype=torch.float64, device="cuda")
    w = torch.randn((n_t, d), dtype=torch.float64, device="cuda") * 0.01
    v = torch.empty((n_t, n_p), dtype=torch.float32, device="cuda")
    for _ in range(3):
        ctx.precompute_device(u.data_ptr(), n_p, d, w.data_ptr(), n_t, v.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        ctx.precompute_device(u.data_ptr(), n_p, d, w.data_ptr(), n_t, v.data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    byt = 8 * d * n_p + 8 * n_t * d + 4 * n_t * n_p
    print(f"form {form}: {ms:.4f} ms, {byt / ms / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
