#!/usr/bin/env python3
"""Randomized parity stress (test infrastructure, not the product): random
libraries (1e4-1e8 products, 2/3/4-component reactions, tie-heavy and
integer-valued tables), random batches of 1-20 queries (random constraints,
k, index ranges) and a random option per case, each result checked field by
field against the threaded C oracle (oracle/fast_oracle.py, pinned to the
numpy port) + the vectorized materialization.  Runs until the time budget.
Usage: python tools/stress.py [seconds] [first_seed]"""
import json
import math
import sys
import time
import traceback
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import __graft_entry__ as g  # noqa: E402

g.build()
import numpy as np  # noqa: E402

from oracle import fast_oracle as fo  # noqa: E402
from oracle import scan_oracle as orc  # noqa: E402
from paper_2510_24380_b200 import _native  # noqa: E402

OPTS = [{}, {}, {}, {}, {"mode": 0}, {"mode": 2}, {"sorted": 0}, {"rowp": 0}, {"packed16": 0}, {"fin_bucket": 0},
        {"cpre": 0}, {"cpre": 1}, {"bail": 0}, {"bail": 1000000000, "bail_min": 1}, {"lazy_hist": 0},
        {"cap": 1024, "samples": 16}, {"graph": 0}, {"heavy_first": 0}, {"tau_side": 0}, {"dense": 1}]


def make_case(rng):
    n_rx = int(rng.integers(1, 40))
    mu = float(rng.choice([2.5, 3.5, 4.5, 5.5]))
    sizes = []
    for _ in range(n_rx):
        r = rng.random()
        c = 2 if r < 0.45 else 3 if r < 0.93 else 4 if r < 0.97 else 1
        sizes.append([int(max(1, round(math.exp(rng.normal(mu - 0.4 * (c - 2), 0.6))))) for _ in range(c)])
    total = sum(math.prod(s) for s in sizes)
    while total > 1.2e8:  # keep the oracle to seconds
        t = int(np.argmax([math.prod(s) for s in sizes]))
        sizes[t] = [max(1, x // 2) for x in sizes[t]]
        total = sum(math.prod(s) for s in sizes)
    pair_off, p = [], 0
    for s in sizes:
        pair_off.append([p + sum(s[:j]) for j in range(len(s))])
        p += sum(s)
    n_tasks = int(rng.integers(2, 12))
    values = (rng.standard_normal((n_tasks, p)) * rng.uniform(0.05, 10, (n_tasks, 1))).astype(np.float32)
    kind = rng.random()
    if kind < 0.2:  # few distinct levels: exact ties everywhere
        values = np.round(values * 2) / 2
    elif kind < 0.3:
        values[:] = 0.0
    values[n_tasks - 1] = np.round(values[n_tasks - 1])
    biases = rng.standard_normal(n_tasks) * (0 if rng.random() < 0.3 else 1)
    return sizes, pair_off, p, values.astype(np.float32), biases


def make_queries(rng, values, total):
    n_tasks = values.shape[0]
    out = []
    for _ in range(int(rng.choice([1, 1, 2, 5, 20]))):
        cons = []
        for t in rng.choice(n_tasks, size=int(rng.integers(0, min(n_tasks, 6) + 1)), replace=False):
            v = values[t]
            lo = float(np.quantile(v, rng.uniform(0, 0.5)) * rng.uniform(1, 3)) if rng.random() < 0.6 else -np.inf
            hi = float(np.quantile(v, rng.uniform(0.5, 1.0)) * rng.uniform(1, 3)) if rng.random() < 0.7 else np.inf
            if t == n_tasks - 1:
                lo = math.floor(lo) if np.isfinite(lo) else lo
                hi = math.ceil(hi) if np.isfinite(hi) else hi
            if lo < hi:  # engine.py:112 rejects lower >= upper
                cons.append((int(t), lo, hi))
        k = int(rng.choice([0, 1, 7, 100, 1000, 5000, 10000]))
        a, b = 0, total
        if rng.random() < 0.25:
            a = int(rng.integers(0, total))
            b = int(rng.integers(a, total + 1))
        out.append({"obj": int(rng.integers(0, n_tasks)), "maximize": bool(rng.random() < 0.5), "cons": cons, "k": k,
                    "start": a, "end": b})
    return out


def check(res, values, biases, lib, prep, nq):
    q = orc.Query(nq["obj"], nq["maximize"], nq["cons"], nq["k"])
    s, g_, ret, disc, scanned = fo.search_topk(values, biases, lib, q, nq["start"], nq["end"], prepared=prep)
    assert (res["n"], res["discarded"], res["scanned"]) == (ret, disc, scanned), \
        ((res["n"], res["discarded"], res["scanned"]), (ret, disc, scanned))
    assert np.array_equal(res["g"].astype(np.int64), g_), "indices"
    if ret == 0:
        return
    t, dig, obj, cons = orc.materialize_arrays(values, biases, lib, q, s, g_)
    assert np.array_equal(res["objective"].view(np.uint64), obj.view(np.uint64)), "objective bits"
    if q.cons:
        assert np.array_equal(np.asarray(res["constraint_values"]).view(np.uint64), cons.view(np.uint64)), "cons"
    assert np.array_equal(res["reaction"].astype(np.int64), t), "reaction"
    for j in range(6):
        live = np.array([len(lib.sizes[x]) > j for x in t], dtype=bool)
        assert np.array_equal(res["digits"][live, j].astype(np.int64), dig[live, j]), "digits"


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    t_end = time.time() + budget
    stats = {"cases": 0, "queries": 0, "products": 0, "failures": []}
    while time.time() < t_end:
        rng = np.random.default_rng(seed)
        sizes, pair_off, n_pairs, values, biases = make_case(rng)
        opts = OPTS[int(rng.integers(0, len(OPTS)))]
        lib = orc.Lib(sizes, pair_off)
        qs = make_queries(rng, values, lib.total)
        try:
            ctx = _native.DeviceContext(0)
            ctx.load_library(sizes, pair_off, lib.offsets[:-1], n_pairs)
            ctx.load_table(values, biases)
            for k, v in opts.items():
                ctx.set_option(k, v)
            prep = fo.Prepared(values, biases, lib)
            for rep in range(2):  # the second run replays the captured graph
                res, _ = ctx.query(qs)
                for r, nq in zip(res, qs):
                    check(r, values, biases, lib, prep, nq)
            ctx.close()
        except Exception as exc:  # noqa: BLE001
            stats["failures"].append({"seed": seed, "opts": opts, "total": lib.total, "nq": len(qs),
                                      "err": f"{type(exc).__name__}: {exc}"[:300]})
            traceback.print_exc()
        stats["cases"] += 1
        stats["queries"] += len(qs)
        stats["products"] += lib.total * len(qs)
        seed += 1
    stats["last_seed"] = seed - 1
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
