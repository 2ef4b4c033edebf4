#!/usr/bin/env python3
"""Debug aid: one golden case/query through the C ABI under option sets,
diffed against the CPU oracle.  Usage: python tools/dbg_golden.py CI QI [opt=v,...] ..."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import __graft_entry__ as g  # noqa: E402

g.build()
from conftest import golden_cases  # noqa: E402

from oracle import scan_oracle as orc  # noqa: E402
from paper_2510_24380_b200 import _native  # noqa: E402


def main():
    ci, qi = int(sys.argv[1]), int(sys.argv[2])
    variants = [dict(kv.split("=") for kv in a.split(",")) if a != "-" else {} for a in sys.argv[3:]] or [{}]
    case = golden_cases()[ci]
    qd = case.queries[qi]
    lib = case.lib_arrays()
    q = case.oracle_query(qd)
    rng = qd["query"]["index_range"]
    a, b = (rng[0], rng[1]) if rng else (0, lib.total)
    s, gg, ret, disc, scanned = orc.search_topk(case.values, case.biases, lib, q, a, b)
    print("case", case.name, "query", qd["query"], "total", lib.total)
    for v in variants:
        ctx = _native.DeviceContext(0)
        ctx.load_library(lib.sizes, lib.pair_off, lib.offsets[:-1], case.values.shape[1])
        ctx.load_table(case.values, case.biases)
        for k, val in v.items():
            ctx.set_option(k, int(val))
        res, st = ctx.query([{"obj": q.obj, "maximize": q.maximize, "cons": q.cons, "k": q.k, "start": a, "end": b}])
        r = res[0]
        got = r["g"].astype(np.int64)
        ok = np.array_equal(got, gg)
        print(v, "ok" if ok else "MISMATCH", "n", r["n"], ret, "dups", len(got) - len(set(got.tolist())),
              "missing", sorted(set(gg.tolist()) - set(got.tolist()))[:10],
              "extra", sorted(set(got.tolist()) - set(gg.tolist()))[:10], "cand", st["candidates"])


if __name__ == "__main__":
    main()
