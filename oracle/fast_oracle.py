"""ctypes wrapper of oracle/scan_oracle.c — CPU ORACLE, TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module, as the checker; the product package never does.  The C library
restates engine.search_topk_stream (engine.py:169-313) with threads over
contiguous g sub-ranges and an exact merge, so the GPU path can be checked at
BASELINE scale (1e9 / 5e9 products) in seconds.  ``search_topk`` has the same
signature and return value as ``scan_oracle.search_topk``; both are pinned
against the reference's golden vectors (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from .scan_oracle import Lib, Query

HERE = Path(__file__).resolve().parent
SRC = HERE / "scan_oracle.c"
SO = HERE / "liboracle.so"
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread", "-std=c11"]
MAX_RG = 6

_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle (gcc) into oracle/liboracle.so."""
    if force or not SO.exists() or SO.stat().st_mtime < SRC.stat().st_mtime:
        tmp = SO.with_suffix(".so.tmp")
        subprocess.run([os.environ.get("CC", "gcc"), *CFLAGS, "-o", str(tmp), str(SRC)], check=True)
        os.replace(tmp, SO)
    return SO


def _load():
    global _lib
    if _lib is None:
        if not SO.exists():
            build()
        lib = C.CDLL(str(SO))
        vp = C.c_void_p
        lib.orc_search_topk.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int32, vp, vp, vp, vp, C.c_int32, C.c_int32,
                                        C.c_int32, vp, vp, vp, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32, vp, vp]
        lib.orc_search_topk.restype = C.c_int64
        _lib = lib
    return _lib


class Prepared:
    """Library arrays in the C layout, built once per (library, table)."""

    def __init__(self, values: np.ndarray, biases: np.ndarray, lib: Lib):
        self.values = np.ascontiguousarray(values, dtype=np.float32)
        self.biases = np.ascontiguousarray(biases, dtype=np.float64)
        n = len(lib.sizes)
        self.n_rg = np.array([len(s) for s in lib.sizes], dtype=np.int32)
        self.sizes = np.zeros((max(n, 1), MAX_RG), dtype=np.int64)
        self.pair_off = np.zeros((max(n, 1), MAX_RG), dtype=np.int64)
        for t, (s, p) in enumerate(zip(lib.sizes, lib.pair_off)):
            self.sizes[t, : len(s)] = s
            self.pair_off[t, : len(p)] = p
        self.g_off = np.asarray(lib.offsets, dtype=np.uint64)
        self.lib = lib


def search_topk(values, biases, lib: Lib, q: Query, start: int = 0, end: int | None = None, threads: int = 0,
                prepared: Prepared | None = None):
    """Exact top-k: (s, g) best-first, retained, discarded, scanned (same
    contract as scan_oracle.search_topk)."""
    end = lib.total if end is None else end
    if not 0 <= start <= end <= lib.total:
        raise ValueError(f"index range [{start}, {end}) invalid")
    P = prepared if prepared is not None else Prepared(values, biases, lib)
    k = int(q.k)
    if k <= 0 or end == start:
        return np.empty(0), np.empty(0, dtype=np.int64), 0, min(k, end - start) - 0 if k > 0 else 0, end - start
    nth = threads or len(os.sched_getaffinity(0))
    cons_task = np.array([c[0] for c in q.cons] or [0], dtype=np.int32)
    cons_lo = np.array([c[1] for c in q.cons] or [0.0], dtype=np.float64)
    cons_hi = np.array([c[2] for c in q.cons] or [0.0], dtype=np.float64)
    out_s = np.empty(k, dtype=np.float64)
    out_g = np.empty(k, dtype=np.uint64)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    n = _load().orc_search_topk(p(P.values), p(P.biases), P.values.shape[0], P.values.shape[1], len(lib.sizes),
                                p(P.n_rg), p(P.sizes), p(P.pair_off), p(P.g_off), int(q.obj), 1 if q.maximize else 0,
                                len(q.cons), p(cons_task), p(cons_lo), p(cons_hi), k, int(start), int(end), nth,
                                p(out_s), p(out_g))
    if n < 0:
        raise RuntimeError("orc_search_topk failed")
    s, g = out_s[:n].copy(), out_g[:n].astype(np.int64)
    return s, g, int(n), min(k, end - start) - int(n), end - start
