"""GPU: BatchTrace accounting of the chain-of-batches variant on the device
 against the reference's own traces
(tests/golden/trace_golden.json, make_trace_golden.py): every batch size,
new and carried count, for chunk sizes 1..1e6, k past the feasible count and
infeasible-heavy queries (the chain's selections then hold violating rows);
and the chain invariants at the config-1 scale (10M products)."""

import json
from pathlib import Path

import numpy as np
import pytest

from conftest import golden_cases, unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    import __graft_entry__ as g

    g.build()
    from paper_2510_24380_b200 import _native

    return _native


def test_trace_matches_reference(native):
    from paper_2510_24380_b200 import engine

    recs = json.loads((Path(__file__).resolve().parent / "golden" / "trace_golden.json").read_text())["traces"]
    cases = {c.name: c for c in golden_cases()}
    objs = {}
    for r in recs:
        case = cases[r["case"]]
        if r["case"] not in objs:
            objs[r["case"]] = (case.library(), case.table())
        lib, table = objs[r["case"]]
        q = engine.QuerySpec(r["objective"], r["direction"],
                             tuple(engine.Constraint(t, unhex(lo), unhex(hi)) for t, lo, hi in r["constraints"]),
                             r["k"])
        trace = engine.BatchTrace([], [], [])
        rng = tuple(r["index_range"]) if r["index_range"] else None
        res = engine.search_topk_batched(lib, table, q, r["chunk"], index_range=rng, trace=trace)
        assert trace.batch_sizes == r["batch_sizes"], r
        assert trace.new_elements == r["new"], r
        assert trace.carried_elements == r["carried"], r
        assert res.retained <= q.k


def test_trace_invariants_c1_scale(native):
    """10M products, an infeasible-heavy query: batch sizes cover the range,
    new + carried == min(k, products so far), the first batch carries nothing."""
    from paper_2510_24380_b200 import engine, synth

    shape = synth.make_shape(synth.SHAPES["c1"])
    u, w, b = synth.build_model(shape)
    values = synth.host_table(u, w)
    lib, table = synth.mirror_objects(shape, values, b)
    q = synth.query_spec({"objective": "dock_a", "direction": "minimize",
                          "constraints": [("mw", 300.0, 300.5), ("tpsa", -np.inf, 40.0)], "k": 1000})
    trace = engine.BatchTrace([], [], [])
    engine.search_topk_batched(lib, table, q, 1 << 20, trace=trace)
    assert sum(trace.batch_sizes) == shape.total
    assert trace.carried_elements[0] == 0
    cum = np.cumsum(trace.batch_sizes)
    assert [n + c for n, c in zip(trace.new_elements, trace.carried_elements)] == [min(q.k, int(x)) for x in cum]
