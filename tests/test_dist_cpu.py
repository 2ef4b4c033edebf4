"""CPU, world_size 2 over gloo: the multi-GPU protocol's host side — contiguous
g-range shards, order-preserving keys, all-gather of padded (key, g) entries —
reproduces the single-range result exactly.  The per-rank local
top-k is computed with the CPU oracle here (the GPU runs apex_query_local)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import golden_cases
    from oracle import scan_oracle as orc
    from paper_2510_24380_b200.dist import PAD, all_gather_entries, score_key, shard_range

    results = []
    for case in golden_cases():
        lib = case.lib_arrays()
        for qd in case.queries:
            q = case.oracle_query(qd)
            if q.k == 0:
                continue
            rng = qd["query"]["index_range"]
            start, end = rng if rng is not None else (0, lib.total)
            a, b = shard_range(start, end, rank, world)
            s, g, *_ = orc.search_topk(case.values, case.biases, lib, q, a, b)
            local = torch.full((q.k, 2), PAD, dtype=torch.int64)
            if len(s):
                local[: len(s), 0] = torch.from_numpy(score_key(s).view(np.int64))
                local[: len(s), 1] = torch.from_numpy(g.astype(np.int64))
            gathered = all_gather_entries(local).numpy()
            keys = gathered[:, 0].view(np.uint64)
            gs = gathered[:, 1].view(np.uint64)
            valid = gs != np.uint64(0xFFFFFFFFFFFFFFFF)
            keys, gs = keys[valid], gs[valid]
            order = np.lexsort((gs, ~keys))[: q.k]  # key desc, g asc
            results.append((gs[order].astype(np.int64).tolist(), min(q.k, end - start) - len(order)))
    if rank == 0:
        out.extend(results)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_merge_matches_single_range(world):
    from conftest import golden_cases
    from oracle import scan_oracle as orc

    manager = mp.Manager()
    out = manager.list()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    expected = []
    for case in golden_cases():
        lib = case.lib_arrays()
        for qd in case.queries:
            q = case.oracle_query(qd)
            if q.k == 0:
                continue
            rng = qd["query"]["index_range"]
            start, end = rng if rng is not None else (0, lib.total)
            s, g, ret, disc, _ = orc.search_topk(case.values, case.biases, lib, q, start, end)
            expected.append((g.tolist(), disc))
    assert list(out) == expected
