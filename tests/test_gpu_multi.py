"""GPU: the multi-GPU paths on one device (this pool has one B200 per box).

  * apex_multi (one process, one host thread, N shards): shard contexts whose
    device ids repeat, so the local steps, the merge context's cross-stream
    waits and the fused peer-pointer merge all run on cuda:0 — results must
    equal one single-device apex_query, field for field;
  * one process per GPU: two ranks (torch.multiprocessing, gloo for the
    host-side all-gather) each driving cuda:0 through the stream-ordered
    dist.sharded_batch (apex_query_local_async -> all-gather ->
    apex_merge_finalize_batch -> apex_query_local_finish) — the merged result
    on every rank equals the single-range query; a forced local overflow
    (tiny candidate capacity) exercises the stale-marker re-gather.
No kernel waits on another rank's kernel (the exchange goes through the host).
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("g", "objective", "constraint_values", "reaction", "digits")


@pytest.fixture(scope="module")
def native():
    import __graft_entry__ as g

    g.build()
    from paper_2510_24380_b200 import _native

    return _native


def _case(seed, n_rx=10, mu=3.6):
    rng = np.random.default_rng(seed)
    sizes, pair_off, p = [], [], 0
    for _ in range(n_rx):
        c = int(rng.integers(2, 4))
        s = [int(max(2, round(np.exp(rng.normal(mu if c == 2 else mu * 0.66, 0.6))))) for _ in range(c)]
        sizes.append(s)
        pair_off.append([p + sum(s[:j]) for j in range(c)])
        p += sum(s)
    values = rng.standard_normal((4, p)).astype(np.float32)
    biases = rng.standard_normal(4)
    return sizes, pair_off, p, values, biases


def _queries(total):
    qs = [{"obj": 1, "maximize": False, "cons": [(0, -3.0, 3.0), (2, -np.inf, 2.0)], "k": 300},
          {"obj": 2, "maximize": True, "cons": [], "k": 50},
          {"obj": 0, "maximize": False, "cons": [(1, -0.5, 0.5), (3, -0.5, 0.5)], "k": 1000},
          {"obj": 3, "maximize": True, "cons": [(1, -1.0, np.inf)], "k": 7}]
    return [dict(q, start=0, end=total) for q in qs]


@pytest.mark.parametrize("n_shards", [2, 3, 8])
@pytest.mark.parametrize("seed", [41, 42])
def test_multi_context_equals_single(native, n_shards, seed):
    from oracle import scan_oracle as orc

    sizes, pair_off, p, values, biases = _case(seed)
    lib = orc.Lib(sizes, pair_off)
    single = native.DeviceContext(0)
    single.load_library(sizes, pair_off, lib.offsets[:-1], p)
    single.load_table(values, biases)
    multi = native.MultiDeviceContext([0] * n_shards)
    multi.load_library(sizes, pair_off, lib.offsets[:-1], p)
    multi.load_table(values, biases)
    assert multi.info() == (n_shards, True)
    qs = _queries(lib.total)
    # whole range, a ragged sub-range (shards cut rows mid-way), a tiny range
    # (some shards empty), and k = 0
    for sub in (qs, [dict(q, start=17, end=lib.total - 23) for q in qs], [dict(q, start=5, end=9) for q in qs],
                [dict(qs[0], k=0)]):
        want, _ = single.query(sub)
        got, st = multi.query(sub)
        for a, b in zip(got, want):
            for key in FIELDS:
                assert np.array_equal(a[key], b[key]), key
            assert (a["n"], a["discarded"], a["scanned"]) == (b["n"], b["discarded"], b["scanned"])
    multi.close()
    single.close()


def test_multi_context_overflow_rerun(native):
    """A shard whose candidate buffer overflows re-runs exactly and the merge
    is repeated (massive exact ties, tiny capacity)."""
    sizes = [[300, 200], [40, 30, 20]]
    p = 590
    pair_off = [[0, 300], [500, 540, 570]]
    values = np.zeros((1, p), dtype=np.float32)
    multi = native.MultiDeviceContext([0, 0, 0])
    multi.load_library(sizes, pair_off, [0, 60000], p)
    multi.load_table(values, np.zeros(1))
    multi.set_option("cap", 1024)
    multi.set_option("samples", 64)
    res, st = multi.query([{"obj": 0, "maximize": True, "cons": [], "k": 700, "start": 0, "end": 84000}])
    assert res[0]["n"] == 700
    assert np.array_equal(res[0]["g"], np.arange(700, dtype=np.uint64))
    multi.close()


def test_engine_api_on_several_devices(native, monkeypatch):
    """The drop-in operator API with APEX_B200_DEVICES (one process, N shards)."""
    from conftest import golden_cases
    from paper_2510_24380_b200 import engine

    case = next(c for c in golden_cases() if c.name == "preset")
    lib, table = case.library(), case.table()
    qs = [case.mirror_query(qd) for qd in case.queries if qd["query"]["index_range"] is None]
    one = [engine.search_topk_stream(lib, table, q, device=0) for q in qs]
    monkeypatch.setenv("APEX_B200_DEVICES", "0,0,0,0")
    many = [engine.search_topk_stream(lib, table, q) for q in qs]
    for a, b in zip(one, many):
        assert [(e.global_index, e.objective.hex(), e.constraint_values) for e in a.entries] == \
               [(e.global_index, e.objective.hex(), e.constraint_values) for e in b.entries]
        assert (a.retained, a.discarded_for_violation, a.scanned) == (b.retained, b.discarded_for_violation,
                                                                      b.scanned)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, seed, ties, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__ as g

    g.build()
    from oracle import scan_oracle as orc
    from paper_2510_24380_b200 import _native
    from paper_2510_24380_b200.dist import sharded_batch

    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if ties is True:  # all-zero table: every local candidate set overflows the minimum capacity
        sizes, pair_off, p = [[300, 200], [40, 30, 20]], [[0, 300], [500, 540, 570]], 590
        values, biases = np.zeros((1, p), dtype=np.float32), np.zeros(1)
    else:
        sizes, pair_off, p, values, biases = _case(seed)
    lib = orc.Lib(sizes, pair_off)
    ctx = _native.DeviceContext(0, stream.cuda_stream)
    ctx.load_library(sizes, pair_off, lib.offsets[:-1], p)
    ctx.load_table(values, biases)
    if ties is True:
        qs = [{"obj": 0, "maximize": True, "cons": [], "k": 700, "start": 0, "end": lib.total}]
        if rank == 1:  # only rank 1 overflows: the ranks must still agree on the re-gather
            ctx.set_option("cap", 1024)
            ctx.set_option("samples", 16)
    else:
        qs = [q for q in _queries(lib.total) if q["k"] > 0]
        if ties == "bail" and rank == 1:
            # only rank 1's sorted-column kernel gives its queries up (a
            # one-pair budget): its exports are marked stale and re-gathered
            ctx.set_option("bail", 1_000_000_000)
            ctx.set_option("bail_min", 1)
    res, info = sharded_batch(ctx, qs)
    ref = _native.DeviceContext(0)
    ref.load_library(sizes, pair_off, lib.offsets[:-1], p)
    ref.load_table(values, biases)
    glob, _ = ref.query(qs)
    ok = all(all(np.array_equal(a[k], b[k]) for k in FIELDS) and a["n"] == b["n"] and
             a["discarded"] == b["discarded"] for a, b in zip(res, glob))
    out[rank] = (ok, info["gather_rounds"])
    dist.destroy_process_group()


@pytest.mark.parametrize("ties", [False, True, "bail"])
def test_two_ranks_stream_ordered_protocol(native, ties):
    import torch.multiprocessing as mp

    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_rank_main, args=(2, _free_port(), 43, ties, out), nprocs=2, join=True)
    assert out[0][0] and out[1][0]
    assert out[0][1] == out[1][1]  # every rank agreed on the number of gather rounds
    if ties:
        assert out[0][1] >= 2  # the overflowed / given-up local results were marked stale and gathered again
