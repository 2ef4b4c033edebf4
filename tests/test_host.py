"""CPU: host-side logic of the drop-in (no GPU calls)."""

import math

import numpy as np
import pytest

from conftest import golden_cases, import_reference, unhex
from paper_2510_24380_b200 import csl, engine, synth


def test_fingerprint_matches_reference_serialization():
    for case in golden_cases():
        lib = case.library()
        assert csl.library_fingerprint(lib, memo=False) == case.fingerprint
        assert csl.serialize_library(lib) == case.library_text


def test_fingerprint_memoized_per_object():
    lib = golden_cases()[0].library()
    a = csl.library_fingerprint(lib)
    assert csl.library_fingerprint(lib) is a


def test_decode_index_roundtrip():
    lib = golden_cases()[0].library()
    total = csl.product_count(lib)
    for g in range(0, total, 7):
        chi = csl.decode_index(lib, g)
        t = chi.reaction_id
        idx = 0
        for rg, (rid, sid) in zip(lib.reactions[t].rgroups, chi.assignment):
            idx = idx * len(rg.synthon_ids) + rg.synthon_ids.index(sid)
        assert lib.reaction_offset(t) + idx == g


def test_errors_before_device():
    case = golden_cases()[0]
    lib, table = case.library(), case.table()
    Q, C = engine.QuerySpec, engine.Constraint
    with pytest.raises(engine.EngineError, match="unknown task"):
        engine.search_topk_stream(lib, table, Q("nope", "maximize", (), k=3))
    with pytest.raises(engine.EngineError, match="unknown task"):
        engine.search_topk_stream(lib, table, Q("obj", "maximize", (C("nope"),), k=3))
    with pytest.raises(engine.EngineError, match="index range"):
        engine.search_topk_stream(lib, table, Q("obj", "maximize", (), k=1), index_range=(10, 5))
    with pytest.raises(engine.EngineError, match="chunk size"):
        engine.search_topk_batched(lib, table, Q("obj", "maximize", (), k=1), 0)
    other = golden_cases()[3].library()
    with pytest.raises(engine.EngineError, match="fingerprint"):
        engine.search_topk_stream(other, table, Q("obj", "maximize", (), k=1))
    with pytest.raises(engine.EngineError, match="lower < upper"):
        C("a", 1.0, 1.0)
    with pytest.raises(engine.EngineError, match="direction"):
        Q("obj", "up")
    with pytest.raises(engine.EngineError, match="k"):
        Q("obj", "maximize", k=-1)


@pytest.mark.parametrize("native", [True, False])
def test_save_result_matches_reference_tsv(tmp_path, native, monkeypatch):
    """The mirror's TSV writer (native formatter, csrc/rowbuild.c, and the
    Python one) reproduces the reference's bytes from the same entries."""
    import __graft_entry__ as gr

    gr._build_rowbuild()
    if not native:
        monkeypatch.setattr(engine, "_rowbuild", None)
    else:
        assert engine._rowbuild is not None
    for case in golden_cases():
        lib = case.library()
        for qi, qd in enumerate(case.queries):
            q = case.mirror_query(qd)
            entries = []
            for g, obj, viol, cons, rid, sids in qd["entries"]:
                rx = lib.reactions[rid]
                chi = csl.MultiIndex(rid, tuple((rg.rgroup_id, s) for rg, s in zip(rx.rgroups, sids)))
                entries.append(engine.ScoredCompound(g, chi, unhex(obj), unhex(viol), tuple(unhex(v) for v in cons)))
            res = engine.TopKResult(entries, qd["scanned"], qd["retained"], qd["discarded"], {})
            p = tmp_path / f"{case.name}_{qi}.tsv"
            engine.save_result(res, q, p)
            assert p.read_text() == qd["tsv"]


def test_reference_objects_duck_typed():
    rcsl, rengine = import_reference()
    case = golden_cases()[0]
    rlib = rcsl.deserialize_library(case.library_text)
    assert csl.library_fingerprint(rlib, memo=False) == case.fingerprint
    mi, sc, tk = engine._types_for(rlib, rengine.QuerySpec("obj", "maximize"))
    assert mi is rcsl.MultiIndex and sc is rengine.ScoredCompound and tk is rengine.TopKResult


@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
def test_synthetic_shapes_hit_targets(name):
    cfg = synth.SHAPES[name]
    shape = synth.make_shape(cfg)
    assert abs(shape.total / cfg.target - 1) < 0.002
    assert len(shape.sizes) == cfg.n_reactions
    assert all(2 <= n <= 200_000 for s in shape.sizes for n in s)
    assert shape.pair_off[0][0] == 0
    # pair rows are R-group-major in declaration order
    flat = [p for po in shape.pair_off for p in po]
    assert flat == sorted(flat) and shape.n_pairs == sum(sum(s) for s in shape.sizes)


def test_c5_queries_are_valid():
    qs = synth.c5_queries(200)
    assert len(qs) == 200
    for q in qs:
        for t, lo, hi in q["constraints"]:
            assert lo < hi and t in synth.PROPERTY_TASKS
        assert q["k"] in (100, 1000, 10_000)


def test_score_key_is_order_preserving():
    from paper_2510_24380_b200.dist import score_key
    rng = np.random.default_rng(0)
    s = np.concatenate([rng.standard_normal(1000) * 10.0 ** rng.integers(-30, 30, 1000), [0.0, -0.0, 1e308, -1e308]])
    k = score_key(s)
    order_s = np.argsort(s, kind="stable")
    assert np.all(k[order_s][1:] >= k[order_s][:-1])
    assert score_key(np.array([0.0]))[0] == score_key(np.array([-0.0]))[0]


def test_shard_ranges_partition():
    from paper_2510_24380_b200.dist import shard_range
    for world in (1, 2, 3, 8):
        for start, end in ((0, 0), (0, 10), (5, 5_000_000_007), (3, 4)):
            parts = [shard_range(start, end, r, world) for r in range(world)]
            assert parts[0][0] == start and parts[-1][1] == end
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))


def _fake_rows(library, n, m, seed=0):
    from paper_2510_24380_b200 import csl

    rng = np.random.default_rng(seed)
    total = csl.product_count(library)
    g = np.sort(rng.choice(total, size=n, replace=False)).astype(np.uint64)
    offs = np.asarray(csl.reaction_offsets(library), dtype=np.uint64)
    t = (np.searchsorted(offs, g, side="right") - 1).astype(np.int32)
    dig = np.zeros((n, 6), dtype=np.int32)
    for i, (gi, ti) in enumerate(zip(g.tolist(), t.tolist())):
        rem = gi - int(offs[ti])
        rgs = library.reactions[ti].rgroups
        for j in range(len(rgs) - 1, -1, -1):
            rem, dig[i, j] = divmod(rem, len(rgs[j].synthon_ids))
    return {"n": n, "g": g, "objective": rng.standard_normal(n), "constraint_values": rng.standard_normal((n, m)),
            "reaction": t, "digits": dig, "scanned": total, "discarded": 0}


@pytest.mark.parametrize("use_reference", [False, True])
def test_native_row_builder_equals_python(use_reference, monkeypatch):
    """csrc/rowbuild.c builds the same ScoredCompound / MultiIndex rows as the
    Python builder (mirror classes, and the reference's own classes)."""
    import __graft_entry__ as gr

    gr._build_rowbuild()
    from conftest import golden_cases
    from paper_2510_24380_b200 import engine

    assert engine._rowbuild is not None
    case = golden_cases()[0]
    if use_reference:
        rcsl, rengine = import_reference()
        library = rcsl.deserialize_library(case.library_text)
        query = rengine.QuerySpec("obj" if "obj" in case.task_names else case.task_names[0], "maximize",
                                  tuple(rengine.Constraint(t) for t in case.task_names[:2]), 10)
    else:
        library = case.library()
        query = engine.QuerySpec(case.task_names[0], "maximize",
                                 tuple(engine.Constraint(t) for t in case.task_names[:2]), 10)
    rows = _fake_rows(library, 25, len(query.constraints))
    fast = engine._build_result(library, query, rows, {"x": 1.0})
    monkeypatch.setattr(engine, "_rowbuild", None)
    slow = engine._build_result(library, query, rows, {"x": 1.0})
    assert type(fast) is type(slow)
    assert fast.entries == slow.entries
    assert [type(e) for e in fast.entries] == [type(e) for e in slow.entries]
    assert [e.violation.hex() for e in fast.entries] == ["0x0.0p+0"] * 25
    assert (fast.scanned, fast.retained, fast.discarded_for_violation) == (slow.scanned, slow.retained,
                                                                           slow.discarded_for_violation)


def test_native_row_builder_caches():
    """The builder's shared objects: a repeated query (same spec, range and
    first row) reuses the MultiIndex instances of its first result, a distinct
    one does not fill the cache; (rgroup_id, synthon_id) tuples are shared per
    library and digit; every result still equals the Python builder's."""
    import __graft_entry__ as gr

    gr._build_rowbuild()
    from conftest import golden_cases
    from paper_2510_24380_b200 import engine

    case = golden_cases()[0]
    library = case.library()
    query = engine.QuerySpec(case.task_names[0], "maximize", tuple(engine.Constraint(t) for t in case.task_names[:2]),
                             10)
    rows = _fake_rows(library, 40, len(query.constraints))
    first = engine._build_result(library, query, rows, {})
    second = engine._build_result(library, query, rows, {})   # repeated: fills the cache
    third = engine._build_result(library, query, rows, {})    # served from it
    assert first.entries == second.entries == third.entries
    assert all(a.chi is b.chi for a, b in zip(second.entries, third.entries))
    # pair tuples shared between rows with the same (R-group, synthon)
    pairs = {}
    for e in third.entries:
        for pr in e.chi.assignment:
            assert pairs.setdefault(pr, pr) is pr
    other = engine.QuerySpec(case.task_names[0], "minimize", (), 10)
    rows2 = _fake_rows(library, 40, 0)
    before = len(engine._chi_cache(library, type(first.entries[0].chi)))
    engine._build_result(library, other, rows2, {})
    assert len(engine._chi_cache(library, type(first.entries[0].chi))) == before  # a first-time query adds nothing


@pytest.mark.parametrize("mmap", [True, False])
def test_table_file_roundtrip_and_reference_bytes(tmp_path, mmap):
    """save_table writes the reference's apexblob1 bytes; load_table (memory
    mapped or copied) returns the same arrays, bit for bit."""
    case = golden_cases()[0]
    table = case.table()
    p = tmp_path / "t.blob"
    engine.save_table(table, p)
    back = engine.load_table(p, mmap=mmap)
    for name in ("values", "biases", "member_ids", "rg_offsets", "rg_ids"):
        a, b = np.asarray(getattr(table, name)), np.asarray(getattr(back, name))
        assert a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes(), name
    assert back.task_names == list(table.task_names) and back.fingerprint == table.fingerprint
    if mmap:
        assert isinstance(back.values, np.memmap) and not back.values.flags.writeable
    rcsl, rengine = import_reference()
    rt = rengine.ContributionTable(values=table.values, biases=table.biases, task_names=list(table.task_names),
                                   member_ids=table.member_ids, rg_offsets=table.rg_offsets, rg_ids=table.rg_ids,
                                   fingerprint=table.fingerprint)
    q = tmp_path / "r.blob"
    rengine.save_table(rt, q)
    assert q.read_bytes() == p.read_bytes()
    ref_back = rengine.load_table(p)
    assert ref_back.values.tobytes() == np.asarray(back.values).tobytes()


def test_operator_calls_pause_gc_and_restore_it():
    """engine._gc_paused: the cyclic GC is off inside an operator call and
    restored after it, on return and on error; a caller that had it off
    keeps it off."""
    import gc

    from paper_2510_24380_b200 import engine

    seen = []

    @engine._gc_paused
    def op(fail=False):
        seen.append(gc.isenabled())
        if fail:
            raise ValueError("x")
        return 7

    assert gc.isenabled()
    assert op() == 7 and seen == [False] and gc.isenabled()
    with pytest.raises(ValueError):
        op(fail=True)
    assert gc.isenabled()
    gc.disable()
    try:
        op()
        assert not gc.isenabled()
    finally:
        gc.enable()
    for f in (engine.search_topk_stream, engine.search_topk_many, engine.search_topk_batched):
        assert f.__wrapped__ is not None
