"""GPU parity: the C-ABI path (libapexb200.so on a B200) against the reference's
own outputs (tests/golden) and the CPU oracle, bit-exact (integer indices,
fp64 objective and constraint values, counts, TSV bytes)."""

import math

import numpy as np
import pytest

from conftest import golden_arrays, golden_cases, golden_query_ids, unhex

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def native():
    import __graft_entry__ as g

    g.build()
    from paper_2510_24380_b200 import _native

    return _native


def _ctx(native, lib_sizes, pair_off, n_pairs, values, biases, **opts):
    from oracle import scan_oracle as orc

    ctx = native.DeviceContext(0)
    lib = orc.Lib(lib_sizes, pair_off)
    ctx.load_library(lib_sizes, pair_off, lib.offsets[:-1], n_pairs)
    ctx.load_table(values, biases)
    for k, v in opts.items():
        ctx.set_option(k, v)
    return ctx, lib


def _check_against_oracle(res, values, biases, lib, q, start, end):
    from oracle import scan_oracle as orc

    s, g, ret, disc, scanned = orc.search_topk(values, biases, lib, q, start, end)
    assert (res["n"], res["discarded"], res["scanned"]) == (ret, disc, scanned)
    assert np.array_equal(res["g"].astype(np.int64), g)
    obj = s if q.maximize else -s
    assert np.array_equal(res["objective"].view(np.uint64), np.asarray(obj, dtype=np.float64).view(np.uint64))
    rows = orc.materialize(values, biases, lib, q, s, g)
    if q.cons and rows:
        cons = np.array([r[4] for r in rows], dtype=np.float64)
        assert np.array_equal(res["constraint_values"].view(np.uint64), cons.view(np.uint64))
    for i, (gi, t, dig, _, _) in enumerate(rows):
        assert res["reaction"][i] == t
        assert tuple(res["digits"][i][: len(dig)]) == dig


def test_graft_smoke():
    import __graft_entry__ as g

    g.build()
    g.smoke()


@pytest.mark.parametrize("ci,qi", golden_query_ids())
def test_golden_through_public_api(native, ci, qi, tmp_path):
    """Reference outputs (make_golden.py) reproduced through the drop-in API."""
    from paper_2510_24380_b200 import engine

    case = golden_cases()[ci]
    qd = case.queries[qi]
    lib, table = case.library(), case.table()
    q = case.mirror_query(qd)
    rng = qd["query"]["index_range"]
    res = engine.search_topk_stream(lib, table, q, index_range=tuple(rng) if rng else None)
    assert (res.retained, res.discarded_for_violation, res.scanned) == (qd["retained"], qd["discarded"],
                                                                        qd["scanned"])
    assert len(res.entries) == len(qd["entries"])
    for e, (g, obj, viol, cons, rid, sids) in zip(res.entries, qd["entries"]):
        assert e.global_index == g
        assert e.objective.hex() == unhex(obj).hex()
        assert repr(e.violation) == repr(unhex(viol)) == "0.0"
        assert tuple(v.hex() for v in e.constraint_values) == tuple(unhex(v).hex() for v in cons)
        assert e.chi.reaction_id == rid and tuple(e.chi.synthon_ids()) == tuple(sids)
    p = tmp_path / "r.tsv"
    engine.save_result(res, q, p)
    assert p.read_text() == qd["tsv"]
    # the batched variant is the same operator (test_engine.py:138-145)
    if rng is None:
        rb = engine.search_topk_batched(lib, table, q, 7)
        assert [e.global_index for e in rb.entries] == [e.global_index for e in res.entries]


def test_golden_batch_equals_single(native):
    """Many queries in one device pass == one call per query."""
    from paper_2510_24380_b200 import engine

    case = next(c for c in golden_cases() if c.name == "preset")
    lib, table = case.library(), case.table()
    qs = [case.mirror_query(qd) for qd in case.queries if qd["query"]["index_range"] is None]
    many = engine.search_topk_many(lib, table, qs)
    for q, r in zip(qs, many):
        one = engine.search_topk_stream(lib, table, q)
        assert [e.global_index for e in r.entries] == [e.global_index for e in one.entries]
        assert [e.objective for e in r.entries] == [e.objective for e in one.entries]


@pytest.mark.parametrize("pre_rows", [2, 1, 0])
def test_precompute_matches_reference_table(native, pre_rows):
    """K1 (fp64 head_w @ u^T, fp32 rounding) == reference precompute_contributions,
    for every kernel form (TMA bulk ring, row-parallel, shared-memory tiles)."""
    arr = golden_arrays()
    ctx = native.DeviceContext(0)
    ctx.set_option("pre_rows", pre_rows)
    got = ctx.load_cache(arr["model/u"], arr["model/head_w"], arr["model/head_b"])
    ref = arr["model/values"]
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("n_pairs,d,n_tasks", [(1, 16, 1), (300, 64, 11), (1000, 32, 16), (257, 48, 5), (5000, 64, 17),
                                               (1, 64, 11), (100_003, 64, 11), (1_231_528, 64, 11)])
def test_precompute_forms_agree_with_numpy_order(native, n_pairs, d, n_tasks):
    """Every K1 form gives the same fp32 table (same per-entry FMA order) on odd
    sizes: partial row blocks and tiles, d not 64, > 16 tasks (tile form only),
    and the C4 table size through the TMA bulk ring (11 x 64)."""
    import torch

    rng = np.random.default_rng(n_pairs + d)
    u = rng.standard_normal((n_pairs, d))
    w = rng.standard_normal((n_tasks, d)) * 0.01
    outs = []
    for pre in (2, 1, 0):
        ctx = native.DeviceContext(0)
        ctx.set_option("pre_rows", pre)
        ud = torch.tensor(u, device="cuda")
        wd = torch.tensor(w, device="cuda")
        vd = torch.empty((n_tasks, n_pairs), dtype=torch.float32, device="cuda")
        ctx.precompute_device(ud.data_ptr(), n_pairs, d, wd.data_ptr(), n_tasks, vd.data_ptr())
        torch.cuda.synchronize()
        outs.append(vd.cpu().numpy())
        ctx.close()
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
    assert np.array_equal(outs[0].view(np.uint32), outs[2].view(np.uint32))
    # and close to the plain fp64 product (the exact order is pinned by the golden test above)
    assert np.allclose(outs[0], (w @ u.T).astype(np.float32), rtol=1e-6, atol=1e-6)


def _brute_upper(p, b, beta, x):
    return ((p + np.float64(x)) + b) <= beta


def test_thresholds_exact(native):
    """The per-row fp32 thresholds are exact: f(U) <= beta < f(nextup(U)) and
    f(L) >= beta > f(nextdown(L)), including degenerate magnitudes."""
    rng = np.random.default_rng(1)
    n = 20000
    p = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)
    b = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)
    beta = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 5, n)
    # degenerate cases: huge prefix absorbs x, exact ties, zeros
    p[:100] = 1e30
    b[100:200] = -1e25
    beta[200:300] = p[200:300] + b[200:300]
    p[300:310] = 0.0
    b[300:310] = 0.0
    beta[300:310] = 0.0
    ctx = native.DeviceContext(0)
    up, lo = ctx.debug_thresholds(p, b, beta)
    fmax = np.float32(3.4028234663852886e38)
    for i in range(n):
        f = lambda x: (p[i] + np.float64(np.float32(x))) + b[i]
        u = up[i]
        if np.isnan(u):
            assert not f(-fmax) <= beta[i]
        elif np.isinf(u):
            assert u > 0 and f(fmax) <= beta[i]
        else:
            assert f(u) <= beta[i]
            assert not f(np.nextafter(u, np.float32(np.inf))) <= beta[i]
        l_ = lo[i]
        if np.isnan(l_):
            assert not f(fmax) >= beta[i]
        elif np.isinf(l_):
            assert l_ < 0 and f(-fmax) >= beta[i]
        else:
            assert f(l_) >= beta[i]
            assert not f(np.nextafter(l_, np.float32(-np.inf))) >= beta[i]


def _random_case(seed, n_rx=6, mu=3.0, sigma=0.7, n_tasks=4, c3=0.5, max_c=3):
    rng = np.random.default_rng(seed)
    sizes = []
    for _ in range(n_rx):
        c = 3 if rng.random() < c3 else 2
        if max_c > 3 and rng.random() < 0.2:
            c = max_c
        sizes.append([int(max(1, round(math.exp(rng.normal(mu, sigma))))) for _ in range(c)])
    pair_off, p = [], 0
    for s in sizes:
        pair_off.append([p + sum(s[:j]) for j in range(len(s))])
        p += sum(s)
    values = (rng.standard_normal((n_tasks, p)) * rng.uniform(0.1, 10, (n_tasks, 1))).astype(np.float32)
    # integer-valued task so bounds are hit exactly
    values[n_tasks - 1] = np.round(values[n_tasks - 1])
    biases = rng.standard_normal(n_tasks)
    return sizes, pair_off, p, values, biases, rng


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("opts", [{}, {"rl": 2, "mode": 2}, {"mode": 0}, {"mode": 0, "cb": 8},
                                  {"mode": 0, "chunk_min": 1000, "tile_products": 64},
                                  {"chunk_min": 1000, "tile_products": 64, "cb_admit": 64},
                                  {"cap": 1024, "samples": 16}, {"refresh": 256, "samples": 64}, {"graph": 0},
                                  {"mode": 2, "dense": 1}, {"mode": 2, "dense": 5, "rl": 2}, {"mode": 2, "dense": 3}, {"mode": 2, "dense": 1, "rl": 2, "tile_products": 8192}, {"mode": 2, "dense": 2},
                                  {"sorted": 0}, {"sorted": 0, "dense": 1}, {"sorted": 0, "rl": 2, "mode": 2},
                                  {"mode": 2, "dense": 0}, {"packed16": 0}, {"rowp": 0}, {"packed16": 0, "rowp": 0},
                                  {"fin_bucket": 0}, {"fin_bucket": 2}, {"cpre": 0}, {"stages": 1},
                                  {"bail": 1000000000, "bail_min": 1}, {"bail": 1000000000, "bail_min": 64},
                                  {"bail": 0}, {"cpre": 1}, {"cpre": 2}, {"lazy_hist": 0}, {"cpre_fused": 0}])
def test_random_libraries_vs_oracle(native, seed, opts):
    from oracle import scan_oracle as orc

    sizes, pair_off, n_pairs, values, biases, rng = _random_case(seed)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases, **opts)
    qs = []
    for qi in range(6):
        obj = int(rng.integers(0, 4))
        cons = []
        for t in rng.choice(4, size=int(rng.integers(0, 4)), replace=False):
            v = values[t]
            lo = float(np.quantile(v, rng.uniform(0, 0.4)) * 2) if rng.random() < 0.6 else -np.inf
            hi = float(np.quantile(v, rng.uniform(0.6, 1.0)) * 2) if rng.random() < 0.7 else np.inf
            if t == 3:  # integer task: integer bounds, hit exactly
                lo = math.floor(lo) if np.isfinite(lo) else lo
                hi = math.ceil(hi) if np.isfinite(hi) else hi
            if lo < hi:
                cons.append((int(t), lo, hi))
        k = int(rng.choice([1, 5, 64, 500, 3000]))
        a, b = 0, lib.total
        if qi % 3 == 2:
            a = int(rng.integers(0, lib.total // 2))
            b = int(rng.integers(a, lib.total + 1))
        qs.append((orc.Query(obj, bool(rng.random() < 0.5), cons, k), a, b))
    res, _ = ctx.query([{"obj": q.obj, "maximize": q.maximize, "cons": q.cons, "k": q.k, "start": a, "end": b}
                        for q, a, b in qs])
    for r, (q, a, b) in zip(res, qs):
        _check_against_oracle(r, values, biases, lib, q, a, b)
    ctx.close()


@pytest.mark.parametrize("opts", [{}, {"dense": 1}, {"dense": 3}, {"cb_admit": 64}, {"mode": 2}, {"sorted": 0},
                                  {"sorted": 0, "mode": 2}, {"refresh": 256}])
@pytest.mark.parametrize("seed", [21, 22, 23])
def test_shared_objective_batches_vs_oracle(native, seed, opts):
    """Batches whose queries share objective columns (same task and
    direction, different constraints and k) against the oracle, query by
    query."""
    from oracle import scan_oracle as orc

    sizes, pair_off, n_pairs, values, biases, rng = _random_case(seed)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases, **opts)
    qs = []
    for obj in (0, 2):
        for maximize in (False, True):
            for ci in range(3):
                cons = []
                for t in rng.choice(4, size=int(rng.integers(0, 4)), replace=False):
                    v = values[t]
                    lo = float(np.quantile(v, rng.uniform(0, 0.3)) * 2) if rng.random() < 0.5 else -np.inf
                    hi = float(np.quantile(v, rng.uniform(0.7, 1.0)) * 2) if rng.random() < 0.7 else np.inf
                    if lo < hi:
                        cons.append((int(t), lo, hi))
                qs.append(orc.Query(obj, maximize, cons, int(rng.choice([1, 20, 300, 2000]))))
    res, _ = ctx.query([{"obj": q.obj, "maximize": q.maximize, "cons": q.cons, "k": q.k, "start": 0,
                         "end": lib.total} for q in qs])
    for r, q in zip(res, qs):
        _check_against_oracle(r, values, biases, lib, q, 0, lib.total)
    ctx.close()


def test_four_and_one_component_reactions(native):
    from oracle import scan_oracle as orc

    sizes = [[7, 5, 3, 4], [11], [6, 9], [3, 4, 5, 2, 3]]
    pair_off, p = [], 0
    for s in sizes:
        pair_off.append([p + sum(s[:j]) for j in range(len(s))])
        p += sum(s)
    rng = np.random.default_rng(3)
    values = rng.standard_normal((2, p)).astype(np.float32)
    biases = rng.standard_normal(2)
    ctx, lib = _ctx(native, sizes, pair_off, p, values, biases)
    for q in (orc.Query(0, True, [], 50), orc.Query(1, False, [(0, -0.5, 1.0)], 40)):
        res, _ = ctx.query([{"obj": q.obj, "maximize": q.maximize, "cons": q.cons, "k": q.k, "start": 0,
                             "end": lib.total}])
        _check_against_oracle(res[0], values, biases, lib, q, 0, lib.total)


def test_all_ties_large_k_exceeds_buffer(native):
    """Massive exact ties (all-zero table) with a small buffer: overflow + re-run,
    ties broken to the lowest global indices."""
    sizes = [[300, 200], [40, 30, 20]]
    pair_off = [[0, 300], [500, 540, 570]]
    values = np.zeros((1, 590), dtype=np.float32)
    biases = np.zeros(1)
    ctx, lib = _ctx(native, sizes, pair_off, 590, values, biases, cap=1024, samples=64)
    res, st = ctx.query([{"obj": 0, "maximize": True, "cons": [], "k": 700, "start": 0, "end": lib.total}])
    assert res[0]["n"] == 700
    assert np.array_equal(res[0]["g"], np.arange(700, dtype=np.uint64))


@pytest.mark.parametrize("k", [8193, 12000, 30000])
def test_large_k_sorted_in_chunks_vs_oracle(native, k):
    """k past the one-CTA sort: radix select, chunk sort + merge rank, and
    materialization equal the oracle (several chunks, a ragged last one)."""
    from oracle import scan_oracle as orc

    sizes, pair_off, n_pairs, values, biases, rng = _random_case(21, n_rx=10, mu=3.8)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases)
    assert lib.total > 2 * k
    for q in (orc.Query(1, False, [(0, -3.0, 3.0)], k), orc.Query(3, True, [], k)):
        res, _ = ctx.query([{"obj": q.obj, "maximize": q.maximize, "cons": q.cons, "k": q.k, "start": 0,
                             "end": lib.total}])
        _check_against_oracle(res[0], values, biases, lib, q, 0, lib.total)


def test_large_k_all_ties_order(native):
    """All-equal objective with k past the one-CTA sort: the chunked order
    breaks ties by ascending global index, as the reference does."""
    sizes = [[300, 200], [40, 30, 20]]
    pair_off = [[0, 300], [500, 540, 570]]
    values = np.zeros((1, 590), dtype=np.float32)
    biases = np.zeros(1)
    ctx, lib = _ctx(native, sizes, pair_off, 590, values, biases)
    res, _ = ctx.query([{"obj": 0, "maximize": True, "cons": [], "k": 10000, "start": 0, "end": lib.total}])
    assert res[0]["n"] == 10000
    assert np.array_equal(res[0]["g"], np.arange(10000, dtype=np.uint64))


def test_local_plus_merge_equals_global(native):
    """Multi-GPU protocol on one device: two range shards -> local top-k ->
    gathered buffer -> merge kernel == one global query."""
    import torch

    from paper_2510_24380_b200.dist import PAD, shard_range

    sizes, pair_off, n_pairs, values, biases, rng = _random_case(11, n_rx=10, mu=3.5)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases)
    q = {"obj": 1, "maximize": False, "cons": [(0, -3.0, 3.0), (2, -np.inf, 2.0)], "k": 300, "start": 0,
         "end": lib.total}
    full, _ = ctx.query([q])
    world = 3
    buf = torch.full((world * q["k"], 2), PAD, dtype=torch.int64, device="cuda")
    for r in range(world):
        a, b = shard_range(0, lib.total, r, world)
        part = buf[r * q["k"]:(r + 1) * q["k"]]
        counts, _ = ctx.query_local([dict(q, start=a, end=b)], part.data_ptr())
        torch.cuda.synchronize()
    merged, _ = ctx.merge_finalize(q, buf.data_ptr(), buf.shape[0], lib.total)
    for key in ("g", "objective", "constraint_values", "reaction", "digits"):
        assert np.array_equal(merged[key], full[0][key]), key
    assert (merged["n"], merged["discarded"], merged["scanned"]) == (full[0]["n"], full[0]["discarded"],
                                                                     full[0]["scanned"])


@pytest.mark.parametrize("k", [1, 50, 3000])
def test_local_plus_batched_merge_equals_global(native, k):
    """Batched multi-GPU protocol on one device: every shard runs the whole
    batch locally (apex_query_local), the [shard][query][k] buffers are
    stacked as an all-gather would, and ONE apex_merge_finalize_batch equals
    the global batch query for every query (k up to well past the small-sort
    path, and k exceeding some queries' feasible counts)."""
    import torch

    from paper_2510_24380_b200.dist import PAD, shard_range

    sizes, pair_off, n_pairs, values, biases, rng = _random_case(12, n_rx=12, mu=3.5)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases)
    qs = [{"obj": 1, "maximize": False, "cons": [(0, -3.0, 3.0), (2, -np.inf, 2.0)], "k": k},
          {"obj": 2, "maximize": True, "cons": [], "k": k},
          {"obj": 0, "maximize": False, "cons": [(1, -0.5, 0.5), (2, -0.5, 0.5), (3, -0.5, 0.5)], "k": k},
          {"obj": 3, "maximize": True, "cons": [(1, -1.0, np.inf)], "k": k}]
    qs = [dict(q, start=0, end=lib.total) for q in qs]
    full, _ = ctx.query(qs)
    world, nq = 3, len(qs)
    buf = torch.full((world * nq * k, 2), PAD, dtype=torch.int64, device="cuda")
    for r in range(world):
        a, b = shard_range(0, lib.total, r, world)
        part = buf[r * nq * k:(r + 1) * nq * k]
        ctx.query_local([dict(q, start=a, end=b) for q in qs], part.data_ptr())
        torch.cuda.synchronize()
    merged, _ = ctx.merge_finalize_batch(qs, buf.data_ptr(), world, k, lib.total)
    for qi in range(nq):
        for key in ("g", "objective", "constraint_values", "reaction", "digits"):
            assert np.array_equal(merged[qi][key], full[qi][key]), (qi, key)
        assert (merged[qi]["n"], merged[qi]["discarded"], merged[qi]["scanned"]) == (
            full[qi]["n"], full[qi]["discarded"], full[qi]["scanned"])


def test_result_views_equal_copies(native):
    """View mode (null output arrays: rows returned as views into the
    context's pinned block) equals the copying call, query by query."""
    sizes, pair_off, n_pairs, values, biases, rng = _random_case(13, n_rx=9, mu=3.5)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases)
    qs = [{"obj": 1, "maximize": False, "cons": [(0, -3.0, 3.0)], "k": 200},
          {"obj": 2, "maximize": True, "cons": [], "k": 7},
          {"obj": 0, "maximize": False, "cons": [(1, -0.5, 0.5), (2, -0.5, 0.5)], "k": 50}]
    qs = [dict(q, start=3, end=lib.total - 5) for q in qs]
    ref, _ = ctx.query(qs)
    pb = ctx.prepare_views(qs)
    for _ in range(2):
        got, _ = ctx.run_views(pb)
        for a, b in zip(got, ref):
            for key in ("g", "objective", "constraint_values", "reaction", "digits"):
                assert np.array_equal(a[key], b[key]), key
            assert (a["n"], a["discarded"], a["scanned"]) == (b["n"], b["discarded"], b["scanned"])
    with pytest.raises(native.NativeError):
        ctx.run_views(ctx.prepare_views([qs[0], dict(qs[1], start=0)]))


@pytest.mark.parametrize("seed", [31, 32])
def test_repeated_batches_identical(native, seed):
    """A batch signature runs directly, then is captured as a graph, then
    replayed (and, when no query needed the full predicate, without those
    launches): every run returns the oracle's result."""
    from oracle import scan_oracle as orc

    sizes, pair_off, n_pairs, values, biases, rng = _random_case(seed)
    ctx, lib = _ctx(native, sizes, pair_off, n_pairs, values, biases)
    qs = [orc.Query(1, False, [(0, -1.0, 1.0)], 50), orc.Query(2, True, [], 20),
          orc.Query(0, False, [(2, -0.3, 0.3), (3, -2.0, 2.0)], 300), orc.Query(3, True, [], 10 ** 6)]
    spec = [{"obj": q.obj, "maximize": q.maximize, "cons": q.cons, "k": q.k, "start": 0, "end": lib.total} for q in qs]
    for _ in range(4):
        res, _ = ctx.query(spec)
        for r, q in zip(res, qs):
            _check_against_oracle(r, values, biases, lib, q, 0, lib.total)
    ctx.close()


def test_c1_shape_vs_oracle(native):
    """Config-1 shape (10M products, random-init heads, calibrated properties)
    against the oracle for the config-1 query and one preset query."""
    from oracle import scan_oracle as orc
    from paper_2510_24380_b200 import synth

    shape = synth.make_shape(synth.SHAPES["c1"])
    u = synth.random_cache(shape.n_pairs, seed=1)
    w, b = synth.random_heads(seed=1)
    w, b = synth.calibrate_heads(shape, u, w, b, n_sample=20000)
    ctx = native.DeviceContext(0)
    lib = orc.Lib(shape.sizes, shape.pair_off)
    ctx.load_library(shape.sizes, shape.pair_off, lib.offsets[:-1], shape.n_pairs)
    values = ctx.load_cache(u, w, b)
    assert np.array_equal(values.view(np.uint32), synth.host_table(u, w).view(np.uint32))
    for qd in (synth.c1_query(), synth.c2_queries()[5]):
        nq = synth.to_native(qd, 0, lib.total)
        res, _ = ctx.query([nq])
        q = orc.Query(nq["obj"], nq["maximize"], nq["cons"], nq["k"])
        _check_against_oracle(res[0], values, b, lib, q, 0, lib.total)
