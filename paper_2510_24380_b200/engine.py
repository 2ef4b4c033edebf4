"""Drop-in B200 implementation of the reference retrieval operator API.

Mirrors `apexcsl.engine` (reference `pkg/src/apexcsl/engine.py`) for the hot
path only:

  * ``search_topk_stream(library, table, query, index_range=None)``   engine.py:265-313
  * ``search_topk_batched(library, table, query, chunk_size, index_range=None, trace=None)``
                                                                      engine.py:345-398
  * ``precompute_contributions(cache, surrogate)``                    engine.py:80-92
  * ``search_topk_many(library, table, queries, index_range=None)``   batched multi-query
    pass (configs 2 and 5; no reference counterpart — its oracle is one
    ``search_topk_stream`` call per query)

with the same names, argument meaning, result types and error behaviour:
``EngineError`` (a ``RuntimeError``) with the reference's message substrings
("unknown task", "fingerprint", "index range", "chunk size").  Inputs may be
objects of the reference classes or of the mirrors defined here.

All compute runs in libapexb200.so (C ABI, sm_100a kernels); there is no CPU
fallback — without the library or a B200 the call raises.
"""

from __future__ import annotations

import collections
import functools
import gc
import math
import operator
import os
import sys
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .csl import MultiIndex, library_fingerprint, product_count


class EngineError(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# mirror types (engine.py:35-162)
# ---------------------------------------------------------------------------

@dataclass
class ContributionTable:
    values: np.ndarray        # float32 (n_tasks, n_pairs), pair-row order
    biases: np.ndarray        # float64 (n_tasks,)
    task_names: list
    member_ids: np.ndarray
    rg_offsets: np.ndarray
    rg_ids: np.ndarray
    fingerprint: str

    _rg_pos: dict = field(init=False, repr=False, compare=False)

    def __post_init__(self):
        self._rg_pos = {int(r): i for i, r in enumerate(self.rg_ids)}

    @property
    def n_tasks(self) -> int:
        return len(self.task_names)

    @property
    def n_pairs(self) -> int:
        return self.values.shape[1]

    def task_index(self, name: str) -> int:
        try:
            return list(self.task_names).index(name)
        except ValueError:
            raise _error(f"unknown task {name!r}") from None

    def check_library(self, library) -> None:
        if self.fingerprint != library_fingerprint(library):
            raise _error("library fingerprint does not match the contribution table")


@dataclass(frozen=True)
class Constraint:
    task: str
    lower: float = float("-inf")
    upper: float = float("inf")

    def __post_init__(self):
        if not self.lower < self.upper:
            raise _error(f"constraint bounds must satisfy lower < upper: {self}")


@dataclass(frozen=True)
class QuerySpec:
    objective: str
    direction: str
    constraints: tuple = ()
    k: int = 10

    def __post_init__(self):
        if self.direction not in ("maximize", "minimize"):
            raise _error(f"direction must be maximize or minimize, got {self.direction!r}")
        if self.k < 0:
            raise _error("k must be >= 0")


@dataclass
class ScoredCompound:
    global_index: int
    chi: MultiIndex
    objective: float
    violation: float
    constraint_values: tuple


@dataclass
class TopKResult:
    entries: list
    scanned: int
    retained: int
    discarded_for_violation: int
    timing: dict


def _error(msg: str) -> Exception:
    # resolved at raise time so dropin.install() can substitute the reference's class
    return _ERROR_CLASS[0](msg)


_ERROR_CLASS = [EngineError]


# ---------------------------------------------------------------------------
# device contexts, memoized per (library, table)
# ---------------------------------------------------------------------------

def default_device():
    """Device(s) the operator API runs on: ``APEX_B200_DEVICES="0,1,...,7"``
    selects the single-process multi-GPU context (index range sharded over
    those devices), else ``APEX_B200_DEVICE`` / ``LOCAL_RANK`` /
    0 — one device."""
    multi = os.environ.get("APEX_B200_DEVICES", "").strip()
    if multi:
        ids = tuple(int(x) for x in multi.split(",") if x.strip())
        return ids if len(ids) > 1 else ids[0]
    for var in ("APEX_B200_DEVICE", "LOCAL_RANK"):
        if var in os.environ:
            return int(os.environ[var])
    return 0


def _open_context(device):
    """One device (int) -> DeviceContext; several (sequence) -> MultiDeviceContext."""
    if isinstance(device, (list, tuple)):
        if len(device) > 1:
            return _native.MultiDeviceContext(list(device))
        device = device[0]
    return _native.DeviceContext(int(device))


class _Bound:
    """A device context (one GPU, or several) with one library + table resident."""

    def __init__(self, library, table, device):
        self.ctx = _open_context(device)
        rg_pos = {int(r): i for i, r in enumerate(table.rg_ids)}
        offs = np.asarray(table.rg_offsets, dtype=np.int64)
        sizes, pair_offsets, g_offsets = [], [], []
        g = 0
        for rx in library.reactions:
            s, p = [], []
            for rg in rx.rgroups:
                j = rg_pos.get(int(rg.rgroup_id))
                if j is None:
                    raise _error(f"R-group {rg.rgroup_id} not in table")
                lo, hi = int(offs[j]), int(offs[j + 1])
                if hi - lo != len(rg.synthon_ids):
                    raise _error(f"table rows for R-group {rg.rgroup_id} do not match library")
                s.append(len(rg.synthon_ids))
                p.append(lo)
            sizes.append(s)
            pair_offsets.append(p)
            g_offsets.append(g)
            g += math.prod(s)
        self.total = g
        self.index_space = (sizes, pair_offsets, g_offsets, int(np.asarray(table.values).shape[1]))
        values = np.asarray(table.values)
        try:
            self.ctx.load_library(sizes, pair_offsets, g_offsets, values.shape[1])
            self.ctx.load_table(values, np.asarray(table.biases, dtype=np.float64))
        except _native.NativeError as exc:
            raise _error(str(exc)) from None
        self.task_names = list(table.task_names)


_BOUND: dict[tuple, tuple[weakref.ref, weakref.ref, _Bound, tuple]] = {}
_MAX_BOUND = 4


def _content_token(table) -> tuple:
    """Cheap identity of the table's current contents: the arrays' buffers and
    shapes plus a CRC of a strided sample of the values and all biases.  The
    reference re-reads the table on every call (engine.py:285); a device copy
    must not survive an in-place edit or a reassignment of values/biases."""
    import zlib

    v = np.asarray(table.values)
    bias = np.asarray(table.biases)
    flat = v.reshape(-1)
    step = max(1, flat.size // 4096)
    sample = np.ascontiguousarray(flat[::step])
    return (v.__array_interface__["data"][0], v.shape, v.dtype.str, bias.__array_interface__["data"][0],
            zlib.crc32(sample.tobytes(), zlib.crc32(np.ascontiguousarray(bias).tobytes())))


def bind(library, table, device=None) -> _Bound:
    """Device context for (library, table), created on first use and reused
    while the table's contents are unchanged (see _content_token)."""
    dev = default_device() if device is None else device
    dev = tuple(dev) if isinstance(dev, (list, tuple)) else int(dev)
    key = (id(library), id(table), dev)
    token = _content_token(table)
    hit = _BOUND.get(key)
    if hit is not None and hit[0]() is library and hit[1]() is table and hit[3] == token:
        return hit[2]
    b = _Bound(library, table, dev)
    if len(_BOUND) >= _MAX_BOUND and key not in _BOUND:
        _BOUND.pop(next(iter(_BOUND)))
    _BOUND[key] = (weakref.ref(library), weakref.ref(table), b, token)
    return b


def _fingerprint_ok(library, table) -> None:
    if table.fingerprint != library_fingerprint(library):
        raise _error("library fingerprint does not match the contribution table")


def _task_index(table, name: str) -> int:
    try:
        return list(table.task_names).index(name)
    except ValueError:
        raise _error(f"unknown task {name!r}") from None


def _validate(library, table, query, index_range):
    _fingerprint_ok(library, table)
    _task_index(table, query.objective)
    for con in query.constraints:
        _task_index(table, con.task)
    total = product_count(library)
    start, end = index_range if index_range is not None else (0, total)
    if not 0 <= start <= end <= total:
        raise _error(f"index range [{start}, {end}) invalid")
    return int(start), int(end)


def _native_query(table, query, start: int, end: int) -> dict:
    return {
        "obj": _task_index(table, query.objective),
        "maximize": query.direction == "maximize",
        "cons": [(_task_index(table, c.task), float(c.lower), float(c.upper)) for c in query.constraints],
        "k": int(query.k),
        "start": start,
        "end": end,
    }


def _types_for(library, query):
    """Result classes from the caller's modules (reference classes when the
    inputs are reference objects), so results compare equal to the reference's."""
    mi = getattr(sys.modules.get(type(library).__module__), "MultiIndex", MultiIndex)
    mod = sys.modules.get(type(query).__module__)
    sc = getattr(mod, "ScoredCompound", ScoredCompound)
    tk = getattr(mod, "TopKResult", TopKResult)
    return mi, sc, tk


def _plain_fields(cls, names):
    """True when ``cls`` is a dataclass whose instances are exactly their
    ``__dict__`` of these fields (no __post_init__, no slots, no defaults that
    __init__ would compute), so an instance can be made without running the
    generated __init__ — a frozen dataclass's __init__ pays an
    object.__setattr__ per field, ~1 µs per result row."""
    fields = getattr(cls, "__dataclass_fields__", None)
    return (fields is not None and tuple(fields) == names and not hasattr(cls, "__post_init__")
            and "__slots__" not in cls.__dict__ and "__dict__" in dir(cls))


_MI_FIELDS = ("reaction_id", "assignment")
_SC_FIELDS = ("global_index", "chi", "objective", "violation", "constraint_values")


try:
    from . import _rowbuild  # native row builder (csrc/rowbuild.c, built by __graft_entry__.build)
except ImportError:  # pragma: no cover - host object construction only; the compute path has no fallback
    _rowbuild = None

_RX_TABLES: dict[int, tuple[weakref.ref, list]] = {}


def _rx_table(library) -> list:
    """Per reaction position: (reaction_id, rgroup ids, synthon id tuples),
    built once per library object (libraries are immutable)."""
    hit = _RX_TABLES.get(id(library))
    if hit is not None and hit[0]() is library:
        return hit[1]
    # (reaction_id, rgroup ids, synthon id tuples, per R-group list of the
    # (rgroup_id, synthon_id) tuples, filled by the native builder on first use)
    table = [(rx.reaction_id, tuple(rg.rgroup_id for rg in rx.rgroups), tuple(rg.synthon_ids for rg in rx.rgroups),
              tuple([None] * len(rg.synthon_ids) for rg in rx.rgroups))
             for rx in library.reactions]
    try:
        _RX_TABLES[id(library)] = (weakref.ref(library), table)
    except TypeError:
        pass
    return table


_CHI_CACHES: dict[int, tuple[weakref.ref, dict]] = {}
_CHI_CACHE_ON = os.environ.get("APEX_B200_CHI_CACHE", "1") != "0"


def _chi_cache(library, mi_cls) -> dict:
    """global index -> MultiIndex of this library, per MultiIndex class: the
    reference's MultiIndex is frozen (csl.py:47), so a product that recurs in
    later results shares one instance (the native builder fills it and clears
    it at 2^16 entries; the device pass is unaffected)."""
    hit = _CHI_CACHES.get(id(library))
    if hit is None or hit[0]() is not library:
        try:
            hit = _CHI_CACHES[id(library)] = (weakref.ref(library), {})
        except TypeError:
            return {}
    return hit[1].setdefault(mi_cls, {})


_RECENT: dict[int, collections.deque] = {}


def _repeated(library, query, res) -> bool:
    """Whether this query (spec and range) was among the library's last 64:
    only a repeated query adds its products to the MultiIndex cache (a stream
    of distinct queries would pay the inserts and gain nothing)."""
    sig = (query.objective, query.direction, int(query.k),
           tuple((c.task, float(c.lower), float(c.upper)) for c in query.constraints), int(res["scanned"]),
           int(res["g"][0]) if len(res["g"]) else -1)
    recent = _RECENT.setdefault(id(library), collections.deque(maxlen=64))
    hit = sig in recent
    if not hit:
        recent.append(sig)
    return hit


def _build_result(library, query, res: dict, timing: dict):
    """TopKResult from the device rows (engine.py:238-262 output shape):
    entries best-first, chi = (reaction_id, ((rgroup_id, synthon_id), ...)),
    violation +0.0, constraint values in constraint order."""
    mi_cls, sc_cls, tk_cls = _types_for(library, query)
    n = int(res["n"])
    if _rowbuild is not None and n:
        fast = _plain_fields(mi_cls, _MI_FIELDS) and _plain_fields(sc_cls, _SC_FIELDS)
        # the rows create no reference cycles: pause the cyclic GC, whose
        # generation sweeps otherwise fire every ~700 of these allocations
        gc_on = gc.isenabled()
        gc.disable()
        try:
            entries = _rowbuild.build_entries(
            mi_cls, sc_cls, fast, n, np.ascontiguousarray(res["g"], dtype=np.uint64),
            np.ascontiguousarray(res["objective"], dtype=np.float64),
            np.ascontiguousarray(res["constraint_values"], dtype=np.float64), len(query.constraints),
            np.ascontiguousarray(res["reaction"], dtype=np.int32), np.ascontiguousarray(res["digits"], dtype=np.int32),
            _rx_table(library), _chi_cache(library, mi_cls) if fast and _CHI_CACHE_ON else None,
            _repeated(library, query, res))
        finally:
            if gc_on:
                gc.enable()
        return tk_cls(entries=entries, scanned=int(res["scanned"]), retained=n,
                      discarded_for_violation=int(res["discarded"]), timing=timing)
    g = res["g"].tolist()
    obj = res["objective"].tolist()
    cons = res["constraint_values"].tolist()
    rxi = res["reaction"].tolist()
    dig = res["digits"].tolist()
    reactions = library.reactions
    fast = _plain_fields(mi_cls, _MI_FIELDS) and _plain_fields(sc_cls, _SC_FIELDS)
    new = object.__new__
    getitem = operator.getitem
    per_rx = {}  # reaction position -> (reaction_id, rgroup ids, synthon id sequences)
    entries = []
    append = entries.append
    for gi, oi, ci, t, d in zip(g, obj, cons, rxi, dig):
        rx = per_rx.get(t)
        if rx is None:
            spec = reactions[t]
            rx = per_rx[t] = (spec.reaction_id, tuple(rg.rgroup_id for rg in spec.rgroups),
                              tuple(rg.synthon_ids for rg in spec.rgroups))
        rid, rgids, sids = rx
        if len(rgids) == 2:
            assignment = ((rgids[0], sids[0][d[0]]), (rgids[1], sids[1][d[1]]))
        elif len(rgids) == 3:
            assignment = ((rgids[0], sids[0][d[0]]), (rgids[1], sids[1][d[1]]), (rgids[2], sids[2][d[2]]))
        else:
            assignment = tuple(zip(rgids, map(getitem, sids, d)))
        if fast:
            chi = new(mi_cls)
            chi.__dict__.update(reaction_id=rid, assignment=assignment)
            sc = new(sc_cls)
            sc.__dict__.update(global_index=gi, chi=chi, objective=oi, violation=0.0, constraint_values=tuple(ci))
        else:
            sc = sc_cls(gi, mi_cls(rid, assignment), oi, 0.0, tuple(ci))
        append(sc)
    return tk_cls(entries=entries, scanned=int(res["scanned"]), retained=n,
                  discarded_for_violation=int(res["discarded"]), timing=timing)


def _timing(t0: float, start: int, end: int, stats: dict) -> dict:
    dt = time.perf_counter() - t0
    timing = {"scan_seconds": dt, "scanned": float(end - start)}
    if dt > 0:
        timing["products_per_second"] = (end - start) / dt
    timing.update({f"device_{k}": float(v) for k, v in stats.items()})
    return timing


# ---------------------------------------------------------------------------
# operator API
# ---------------------------------------------------------------------------

def _gc_paused(fn):
    """Run an operator call with the cyclic GC paused.  A call allocates k
    result rows (none in reference cycles); with the GC live, the sweeps they
    trigger run while the rows are still referenced, promote them, and every
    few calls escalate to a full sweep of every live object in the process —
    tens of ms with a 1e9-product library's ~3e5 synthon records resident.
    Paused, the allocation count falls back as soon as the caller drops a
    result, so a stream of queries never pays a sweep it did not cause; a
    caller that keeps its results pays it at its own next allocation, as it
    would for any other objects.  Nothing is allocated between the re-enable
    and the return."""
    @functools.wraps(fn)
    def call(*args, **kwargs):
        gc_on = gc.isenabled()
        gc.disable()
        try:
            return fn(*args, **kwargs)
        finally:
            if gc_on:
                gc.enable()
    return call


@_gc_paused
def search_topk_stream(library, table, query, index_range=None, device=None):
    """Exact constrained top-k (engine.py:265-313), on the B200 — on several
    B200s when ``device`` is a sequence of ids (or APEX_B200_DEVICES is set)."""
    start, end = _validate(library, table, query, index_range)
    return _run([query], library, table, start, end, device)[0]


@dataclass
class BatchTrace:
    batch_sizes: list
    new_elements: list
    carried_elements: list


def batch_ends(library, chunk_size: int, start: int, end: int) -> list:
    """Exclusive end of every batch of ``make_batches`` (engine.py:316-335):
    whole (reaction, first-digit) slabs of ``iter_blocks`` (engine.py:169-189)
    grouped while the running size stays <= chunk_size (a larger slab forms
    its own batch).  Batches are contiguous ranges of the index space."""
    ends, cur, cur_end = [], 0, None
    off = 0
    for rx in library.reactions:
        sizes = [len(rg.synthon_ids) for rg in rx.rgroups]
        size = math.prod(sizes)
        if off + size <= start or off >= end:
            off += size
            continue
        inner = size // sizes[0]
        j0 = max(0, (start - off) // inner) if start > off else 0
        j1 = min(sizes[0], -(-(end - off) // inner))
        for j in range(j0, j1):
            g0 = off + j * inner
            lo, hi = max(start, g0), min(end, g0 + inner)
            if lo >= hi:
                continue
            n = hi - lo
            if cur and cur + n > chunk_size:
                ends.append(cur_end)
                cur = 0
            cur += n
            cur_end = hi
        off += size
    if cur:
        ends.append(cur_end)
    return ends


@_gc_paused
def search_topk_batched(library, table, query, chunk_size, index_range=None, trace=None, device=None):
    """Chain-of-batches variant (engine.py:345-398).  Results are identical to
    the stream variant by contract (test_engine.py:138-145), so both run the
    same device pipeline; ``chunk_size`` is validated as the reference does.
    ``trace`` receives the chain's BatchTrace accounting (engine.py:387-391),
    computed exactly on the device (apex_batch_trace: per batch, the k best of
    carry and batch under the full order, infeasible products included)."""
    _fingerprint_ok(library, table)
    _task_index(table, query.objective)
    for con in query.constraints:
        _task_index(table, con.task)
    if chunk_size < 1:
        raise _error("chunk size must be >= 1")
    start, end = _validate(library, table, query, index_range)
    out = _run([query], library, table, start, end, device)[0]
    if trace is not None and query.k > 0 and end > start:
        ends = batch_ends(library, int(chunk_size), start, end)
        b = bind(library, table, device)
        ctx = b.ctx if isinstance(b.ctx, _native.DeviceContext) else _native.DeviceContext(default_device_one(device))
        if ctx is not b.ctx:
            ctx.load_library(*b.index_space)
            ctx.load_table(np.asarray(table.values), np.asarray(table.biases, dtype=np.float64))
        try:
            new, carried = ctx.batch_trace(_native_query(table, query, start, end), np.asarray(ends, dtype=np.uint64))
        except _native.NativeError as exc:
            raise _error(str(exc)) from None
        prev = start
        for e, n, c in zip(ends, new.tolist(), carried.tolist()):
            trace.batch_sizes.append(e - prev)
            trace.new_elements.append(int(n))
            trace.carried_elements.append(int(c))
            prev = e
    return out


def default_device_one(device) -> int:
    dev = default_device() if device is None else device
    return int(dev[0] if isinstance(dev, (list, tuple)) else dev)


@_gc_paused
def search_topk_many(library, table, queries, index_range=None, device=None):
    """Several queries in one batched device pass; same results as one
    ``search_topk_stream`` call per query."""
    if not queries:
        return []
    start, end = _validate(library, table, queries[0], index_range)
    for q in queries[1:]:
        _validate(library, table, q, index_range)
    return _run(list(queries), library, table, start, end, device)


def _run(queries, library, table, start, end, device):
    t0 = time.perf_counter()
    out = [None] * len(queries)
    live = [i for i, q in enumerate(queries) if q.k > 0 and end > start]
    if live:
        b = bind(library, table, device)
        try:
            res, stats = b.ctx.query([_native_query(table, queries[i], start, end) for i in live])
        except _native.NativeError as exc:
            raise _error(str(exc)) from None
        timing = _timing(t0, start, end, stats)
        for j, i in enumerate(live):
            out[i] = _build_result(library, queries[i], res[j], dict(timing))
    for i, q in enumerate(queries):
        if out[i] is None:
            empty = {"n": 0, "g": np.empty(0, np.uint64), "objective": np.empty(0), "constraint_values": np.empty((0, 0)),
                     "reaction": np.empty(0, np.int32), "digits": np.empty((0, 6), np.int32), "discarded": 0,
                     "scanned": end - start}
            out[i] = _build_result(library, q, empty, _timing(t0, start, end, {}))
    return out


def precompute_contributions(cache, surrogate, device=None):
    """Dot each task head with every cached associative embedding
    (engine.py:80-92) on the device: fp64 products and accumulation, fp32
    rounding.  Returns a table of the caller's class when available."""
    dev = default_device() if device is None else device
    ctx = _native.DeviceContext(int(dev[0] if isinstance(dev, (list, tuple)) else dev))
    try:
        values = ctx.load_cache(np.asarray(cache.u, dtype=np.float64), np.asarray(surrogate.head_w, dtype=np.float64),
                                np.asarray(surrogate.head_b, dtype=np.float64))
    except _native.NativeError as exc:
        raise _error(str(exc)) from None
    finally:
        ctx.close()
    rg_ids = np.asarray(sorted(cache.rg_pos, key=cache.rg_pos.get))
    mod = sys.modules.get(type(surrogate).__module__.replace("surrogate", "engine"))
    cls = getattr(mod, "ContributionTable", ContributionTable) if mod else ContributionTable
    return cls(
        values=values,
        biases=np.asarray(surrogate.head_b, dtype=np.float64).copy(),
        task_names=list(surrogate.task_names),
        member_ids=np.asarray(cache.member_ids).copy(),
        rg_offsets=np.asarray(cache.rg_offsets).copy(),
        rg_ids=rg_ids,
        fingerprint=cache.fingerprint,
    )


# ---------------------------------------------------------------------------
# contribution-table files (engine.py:425-460 over blobio.py:14-44)
# ---------------------------------------------------------------------------

BLOB_MAGIC = "apexblob1"
TABLE_VERSION = 1


def save_table(table, path) -> None:
    """The reference's apexblob1 table file, byte for byte: one JSON header
    line (sort_keys) with the array specs, then the raw little-endian arrays
    in order values, biases, member_ids, rg_offsets, rg_ids."""
    import json

    arrays = {"values": np.asarray(table.values), "biases": np.asarray(table.biases),
              "member_ids": np.asarray(table.member_ids), "rg_offsets": np.asarray(table.rg_offsets),
              "rg_ids": np.asarray(table.rg_ids)}
    meta = {"kind": "contribution_table", "version": TABLE_VERSION, "task_names": list(table.task_names),
            "fingerprint": table.fingerprint}
    header = {"magic": BLOB_MAGIC, "meta": meta,
              "arrays": [{"name": k, "dtype": str(v.dtype), "shape": list(v.shape)} for k, v in arrays.items()]}
    with open(path, "wb") as fh:
        fh.write(json.dumps(header, sort_keys=True).encode() + b"\n")
        for v in arrays.values():
            fh.write(np.ascontiguousarray(v).tobytes())


def load_table(path, mmap: bool = True, cls=None):
    """Read a table file written by ``save_table`` / the reference's
    ``save_table``.  With ``mmap`` (default) the arrays are read-only views of
    the memory-mapped file: nothing is copied on the host, and the device
    upload at the first query (apex_load_table) reads the pages straight from
    the mapping — the 5e9-product table (58 MB) loads without a host copy.
    ``mmap=False`` copies like the reference (engine.py:448-460).  ``cls``:
    the table class to build (the reference's, under dropin.install())."""
    import json

    with open(path, "rb") as fh:
        line = fh.readline()
        header = json.loads(line.decode())
        if header.get("magic") != BLOB_MAGIC:
            raise ValueError(f"{path}: not an {BLOB_MAGIC} file")
        offset = len(line)
        arrays = {}
        for spec in header["arrays"]:
            dtype = np.dtype(spec["dtype"])
            shape = tuple(spec["shape"])
            n = int(np.prod(shape)) if shape else 1
            if mmap and n > 0:
                arrays[spec["name"]] = np.memmap(path, dtype=dtype, mode="r", offset=offset, shape=shape)
            else:
                fh.seek(offset)
                arrays[spec["name"]] = np.frombuffer(fh.read(n * dtype.itemsize), dtype=dtype).reshape(shape).copy()
            offset += n * dtype.itemsize
    meta = header["meta"]
    if meta.get("kind") != "contribution_table" or meta.get("version") != TABLE_VERSION:
        raise _error(f"{path}: not a version-{TABLE_VERSION} contribution table")
    return (cls or ContributionTable)(values=arrays["values"], biases=arrays["biases"],
                                      task_names=list(meta["task_names"]), member_ids=arrays["member_ids"],
                                      rg_offsets=arrays["rg_offsets"], rg_ids=arrays["rg_ids"],
                                      fingerprint=meta["fingerprint"])


RESULT_HEADER_PREFIX = "rank\tglobal_index\treaction_id\tsynthon_ids\tobjective\tviolation"


def save_result(result, query, path, library=None) -> None:
    """Delimited text export with the reference's exact format (engine.py:463-489):
    repr() of every float, constraint columns in query order, optional
    assembled-token column (csl.py:218-227)."""
    cols = RESULT_HEADER_PREFIX + "".join(f"\t{con.task}" for con in query.constraints)
    tokens = None
    if library is not None:
        cols += "\tassembled"
        tokens = {s.synthon_id: s.token for s in library.synthons}
    if tokens is None and _rowbuild is not None:
        # native formatter (csrc/rowbuild.c): the same bytes, without per-row bytecode
        with open(path, "w") as fh:
            fh.write(cols + "\n")
            fh.write(_rowbuild.format_rows(result.entries))
        return
    lines = [cols]
    for rank, e in enumerate(result.entries):
        sids = ",".join(map(str, e.chi.synthon_ids()))
        row = f"{rank}\t{e.global_index}\t{e.chi.reaction_id}\t{sids}\t{e.objective!r}\t{e.violation!r}"
        row += "".join(f"\t{v!r}" for v in e.constraint_values)
        if tokens is not None:
            frags = sorted(tokens[s].replace("*", "") for _, s in e.chi.assignment)
            row += f"\tt{e.chi.reaction_id}|" + ".".join(frags)
        lines.append(row)
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")
