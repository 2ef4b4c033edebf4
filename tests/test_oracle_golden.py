"""CPU: the oracle (oracle/scan_oracle.py) reproduces the reference's own
outputs recorded in tests/golden (make_golden.py), bit for bit."""

import numpy as np
import pytest

from conftest import golden_cases, golden_query_ids, unhex
from oracle import scan_oracle as orc


def _expected_rows(qd):
    return [(e[0], unhex(e[1]), unhex(e[2]), tuple(unhex(v) for v in e[3]), e[4], tuple(e[5])) for e in qd["entries"]]


@pytest.mark.parametrize("ci,qi", golden_query_ids())
def test_oracle_matches_reference(ci, qi):
    case = golden_cases()[ci]
    qd = case.queries[qi]
    lib = case.lib_arrays()
    library = case.library()
    q = case.oracle_query(qd)
    rng = qd["query"]["index_range"]
    start, end = rng if rng is not None else (0, lib.total)
    s, g, ret, disc, scanned = orc.search_topk(case.values, case.biases, lib, q, start, end)
    assert (ret, disc, scanned) == (qd["retained"], qd["discarded"], qd["scanned"])
    rows = orc.materialize(case.values, case.biases, lib, q, s, g)
    exp = _expected_rows(qd)
    assert len(rows) == len(exp)
    for (gi, t, dig, obj, cons), (eg, eobj, eviol, econs, erx, esids) in zip(rows, exp):
        assert gi == eg
        assert obj.hex() == eobj.hex()
        assert eviol == 0.0 and str(eviol) == "0.0"
        assert tuple(c.hex() for c in cons) == tuple(c.hex() for c in econs)
        rx = library.reactions[t]
        assert rx.reaction_id == erx
        assert tuple(rg.synthon_ids[d] for rg, d in zip(rx.rgroups, dig)) == esids


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_sharded_merge_is_exact(shards):
    """merging per-shard top-k over contiguous g ranges is exact."""
    for case in golden_cases():
        lib = case.lib_arrays()
        for qd in case.queries[:2]:
            q = case.oracle_query(qd)
            rng = qd["query"]["index_range"]
            start, end = rng if rng is not None else (0, lib.total)
            a = orc.search_topk(case.values, case.biases, lib, q, start, end)
            b = orc.search_topk_sharded(case.values, case.biases, lib, q, start, end, shards)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2:] == b[2:]


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_c_oracle_matches_reference(threads):
    """The threaded C restatement (oracle/scan_oracle.c, the scale checker)
    reproduces every golden query recorded from the reference, bit for bit."""
    from oracle import fast_oracle as fo

    fo.build()
    for case in golden_cases():
        lib = case.lib_arrays()
        for qd in case.queries:
            q = case.oracle_query(qd)
            rng = qd["query"]["index_range"]
            start, end = rng if rng is not None else (0, lib.total)
            s, g, ret, disc, scanned = fo.search_topk(case.values, case.biases, lib, q, start, end, threads=threads)
            assert (ret, disc, scanned) == (qd["retained"], qd["discarded"], qd["scanned"])
            assert [int(x) for x in g] == [e[0] for e in qd["entries"]]
            obj = s if q.maximize else -s
            assert [x.hex() for x in obj.tolist()] == [unhex(e[1]).hex() for e in qd["entries"]]


@pytest.mark.parametrize("seed", range(6))
def test_c_oracle_matches_numpy_port(seed):
    """C oracle == numpy oracle on random libraries (2/3/4-component reactions,
    ragged sub-ranges, constraints with both bounds, k past the feasible count)."""
    from oracle import fast_oracle as fo

    rng = np.random.default_rng(100 + seed)
    sizes, pair_off, p = [], [], 0
    for _ in range(int(rng.integers(3, 8))):
        c = int(rng.integers(1, 5))
        s = [int(x) for x in rng.integers(2, 30 if c > 2 else 200, size=c)]
        sizes.append(s)
        pair_off.append([p + sum(s[:j]) for j in range(c)])
        p += sum(s)
    values = rng.standard_normal((4, p)).astype(np.float32)
    if seed % 2:
        values = np.round(values * 2).astype(np.float32)  # integer-valued: exact ties and bounds hit exactly
    biases = rng.standard_normal(4)
    lib = orc.Lib(sizes, pair_off)
    for trial in range(6):
        a = int(rng.integers(0, lib.total // 3))
        b = int(rng.integers(2 * lib.total // 3, lib.total + 1))
        cons = [(int(rng.integers(0, 4)), float(rng.normal(-1, 0.5)), float(rng.normal(1, 0.5)))
                for _ in range(int(rng.integers(0, 3)))]
        cons = [c for c in cons if c[1] < c[2]]
        q = orc.Query(int(rng.integers(0, 4)), bool(rng.integers(0, 2)), cons, int(rng.integers(1, 400)))
        x = orc.search_topk(values, biases, lib, q, a, b)
        y = fo.search_topk(values, biases, lib, q, a, b, threads=int(rng.integers(1, 6)))
        assert np.array_equal(x[0].view(np.uint64), y[0].view(np.uint64)) and np.array_equal(x[1], y[1])
        assert x[2:] == y[2:]


def gt_cases():
    import json
    from pathlib import Path

    root = Path(__file__).resolve().parent / "golden"
    doc = json.loads((root / "gt_golden.json").read_text())
    arrays = dict(np.load(root / "gt_golden.npz"))
    return doc["cases"], arrays


def gt_oracle(case, arrays):
    """Mirror GroundTruthOracle of a golden case (paper_2510_24380_b200.evalkit types)."""
    from paper_2510_24380_b200 import evalkit

    tasks = [evalkit.TaskDef(t["name"], t["mode"], arrays[f"{case['name']}/latent/{i}"],
                             unhex(t["nonlinear_scale"]), unhex(t["nonlinear_alpha"]), unhex(t["pair_scale"]),
                             unhex(t["pair_density"])) for i, t in enumerate(case["tasks"])]
    return evalkit.GroundTruthOracle(tasks, case["seed"])


def test_gt_oracle_matches_reference():
    """oracle/gt_oracle.py (numpy restatement of props.oracle_block_values +
    evalkit.oracle_topk) reproduces the reference's recorded oracle top-j."""
    from oracle import gt_oracle as gto
    from paper_2510_24380_b200 import csl

    cases, arrays = gt_cases()
    n = 0
    for case in cases:
        lib = csl.deserialize_library(case["library"])
        oracle = gt_oracle(case, arrays)
        names = [t["name"] for t in case["tasks"]]
        for q in case["queries"]:
            cons = [(names.index(t), unhex(lo), unhex(hi)) for t, lo, hi in q["constraints"]]
            start, end = q["index_range"] if q["index_range"] else (0, None)
            g, o = gto.topk(lib, oracle, names.index(q["objective"]), q["direction"] == "maximize", cons, q["j"],
                            start, end)
            assert g.tolist() == q["g"], (case["name"], q["objective"])
            assert [x.hex() for x in o.tolist()] == q["objective_values"]
            n += 1
    assert n == 21
