"""Multi-GPU sharding, one process per GPU.

The product index space [start, end) is cut into contiguous g ranges, one per
rank; every rank computes its exact local top-min(k, feasible) on its GPU, the
per-rank (key, g) entries (16 B each, padded to k) are all-gathered with NCCL
over NVLink, and every rank runs the exact merge (apex_merge_finalize_batch:
one device pass for a whole batch) on the gathered buffer.  Exactness: the
global top-k is contained in the union of the local top-k's, and the (key, g)
order is global.  ``sharded_batch`` is the stream-ordered form (local step,
all-gather and merge enqueued back to back; one host sync).  The one-process
form driving several GPUs is ``_native.MultiDeviceContext`` (apex_multi_*),
whose merge reads the shards' entries over NVLink peer pointers directly.
"""

from __future__ import annotations

import numpy as np

PAD = -1  # int64 view of UINT64_MAX: key 0xff..ff / g 0xff..ff marks an empty slot


def shard_range(start: int, end: int, rank: int, world: int) -> tuple[int, int]:
    span = end - start
    return start + span * rank // world, start + span * (rank + 1) // world


def score_key(s: np.ndarray) -> np.ndarray:
    """Host restatement of the device's order-preserving key (common.cuh skey):
    +-0 canonicalized, larger score -> larger uint64."""
    s = np.where(np.asarray(s, dtype=np.float64) == 0.0, 0.0, s).astype(np.float64)
    u = s.view(np.uint64)
    neg = (u >> np.uint64(63)) == np.uint64(1)
    return np.where(neg, ~u, u | np.uint64(0x8000000000000000))


def all_gather_entries(local, group=None):
    """all-gather a [k, 2] int64 tensor of (key, g) entries from every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world * local.shape[0], 2), dtype=local.dtype, device=local.device)
    if local.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    elif local.is_cuda:
        # non-NCCL group (tests): gather through host memory
        return all_gather_entries(local.cpu(), group).to(local.device)
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous(), group=group)
        out = torch.cat(parts, 0)
    return out


def sharded_query(ctx, query: dict, group=None, stream_sync=True):
    """Run one native query dict (task indices, start/end = global range) on
    this rank's shard and return the merged global result (every rank)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    a, b = shard_range(query["start"], query["end"], rank, world)
    k = int(query["k"])
    local = torch.full((max(k, 1), 2), PAD, dtype=torch.int64, device="cuda")
    q = dict(query, start=a, end=b)
    counts, st_local = ctx.query_local([q], local.data_ptr())
    gathered = all_gather_entries(local, group)
    torch.cuda.current_stream().synchronize()
    res, st_merge = ctx.merge_finalize(query, gathered.data_ptr(), gathered.shape[0], query["end"] - query["start"])
    return res, {"local": st_local, "merge": st_merge, "local_count": counts[0]}


def sharded_batch(ctx, queries: list[dict], group=None, prepared=None, local=None):
    """A batch of native queries sharing one global range [start, end): every
    rank scans its shard for all of them, ONE all-gather of the [n_queries][k]
    entry buffers, and one batched exact merge — stream-ordered on the
    context's stream (which must be torch's current stream): the local step
    and its padded export (apex_query_local_async), the NCCL all-gather and
    the merge are enqueued back to back, and the only host sync is the merge's
    result copy.  A local candidate-buffer overflow is resolved exactly: the
    overflowed rank exports a stale marker, every rank's merge sees it in the
    same gathered data (so all ranks agree without another collective), the
    overflowed rank re-runs in apex_query_local_finish, and all ranks gather
    and merge again."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    start, end = queries[0]["start"], queries[0]["end"]
    if any(q["start"] != start or q["end"] != end for q in queries):
        raise ValueError("sharded_batch: all queries must share one index range")
    k = max(max(int(q["k"]) for q in queries), 1)
    a, b = shard_range(start, end, rank, world)
    if local is None:
        local = torch.empty((len(queries) * k, 2), dtype=torch.int64, device="cuda")
    live = b > a
    if live:
        st_local = ctx.query_local_async([dict(q, start=a, end=b) for q in queries], local.data_ptr(), k)
    else:  # an empty shard contributes padding only
        local.fill_(PAD)
        st_local = {}
    gathered = all_gather_entries(local, group)
    res, st_merge = ctx.merge_finalize_batch(queries, gathered.data_ptr(), world, k, end - start, prepared)
    counts, st_fin = [0] * len(queries), {}
    if live:
        counts, _, st_fin = ctx.query_local_finish()
    rounds = 1
    while st_merge.get("stale_sources", 0):
        gathered = all_gather_entries(local, group)
        res, st_merge = ctx.merge_finalize_batch(queries, gathered.data_ptr(), world, k, end - start, prepared)
        rounds += 1
    return res, {"local": st_local, "local_finish": st_fin, "merge": st_merge, "local_counts": counts,
                 "gather_rounds": rounds}
