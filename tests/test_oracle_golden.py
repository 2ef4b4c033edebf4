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
