#!/usr/bin/env python3
"""K1 precompute forms at the C4 table size (1.23M pair rows x 64 x 11 tasks):
device ms and HBM fraction of each form (pre_rows 2 = TMA bulk ring, 1 = row
parallel, 0 = smem tiles), tables compared bit for bit.  Usage: python tools/k1_ab.py"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.build()
from paper_2510_24380_b200 import _native, synth  # noqa: E402

n_p, d, n_t = synth.make_shape(synth.SHAPES["c4"]).n_pairs, 64, 11
u = torch.randn((n_p, d), dtype=torch.float64, device="cuda")
w = torch.randn((n_t, d), dtype=torch.float64, device="cuda") * 0.01
w_host = w.cpu().numpy().copy()  # the TMA form takes host heads as kernel parameters (no device round trip)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
outs = {}
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
byt = 8 * d * n_p + 8 * n_t * d + 4 * n_t * n_p
for pre in (2, 1, 0):
    ctx = _native.DeviceContext(0, stream.cuda_stream)  # same stream as the L2 flush: no idle gap before the kernel
    ctx.set_option("pre_rows", pre)
    wp = w_host.ctypes.data if pre == 2 else w.data_ptr()
    v = torch.empty((n_t, n_p), dtype=torch.float32, device="cuda")
    for _ in range(3):
        ctx.precompute_device(u.data_ptr(), n_p, d, wp, n_t, v.data_ptr())
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
    ms = []
    for e0, e1 in ev:
        flush.zero_()
        ctx.precompute_device(u.data_ptr(), n_p, d, wp, n_t, v.data_ptr())
        kt = ctx.precompute_time()
        ms.append(kt)
    torch.cuda.synchronize()
    outs[pre] = v.cpu().numpy()
    med = float(np.median(ms))
    print(json.dumps({"pre_rows": pre, "kernel_ms": med, "GBps": byt / (med * 1e-3) / 1e9 if med > 0 else None}))
    ctx.close()
print(json.dumps({"bit_identical": all(np.array_equal(outs[2].view(np.uint32), outs[p].view(np.uint32)) for p in (1, 0))}))
