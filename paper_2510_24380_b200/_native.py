"""ctypes binding of the C ABI in ``include/apex_b200.h`` (libapexb200.so).

This is the only way the Python mirror reaches the GPU: there is no CPU
fallback.  If the shared library is missing, or no sm_100 device is present,
every entry point raises ``NativeError`` (mapped to ``EngineError`` by
``engine.py``) instead of silently computing on the host.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

MAX_RGROUPS = 6

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("APEX_B200_LIB", _PKG / "libapexb200.so"))

# status codes (apex_b200.h)
APEX_OK, APEX_EINVAL, APEX_ERANGE, APEX_ETASK, APEX_ECUDA, APEX_ESTATE, APEX_ENOMEM, APEX_ELIMIT = range(8)

EXPORTED = (
    "apex_last_error", "apex_version", "apex_ctx_create", "apex_ctx_destroy", "apex_set_stream",
    "apex_load_library", "apex_load_table", "apex_load_cache", "apex_precompute_device", "apex_query",
    "apex_query_async", "apex_query_fetch", "apex_query_local", "apex_merge_finalize", "apex_merge_finalize_batch",
    "apex_set_option", "apex_get_device_info",
    "apex_debug_thresholds", "apex_debug_trace",
    "apex_query_local_async", "apex_query_local_finish", "apex_precompute_time", "apex_gt_load", "apex_gt_topk",
    "apex_encode_hierarchy", "apex_precompute_resident", "apex_batch_trace",
    "apex_multi_create", "apex_multi_destroy", "apex_multi_load_library", "apex_multi_load_table",
    "apex_multi_load_cache", "apex_multi_set_option", "apex_multi_query", "apex_multi_info",
)


class PreparedBatch:
    """A query batch with its C descriptors and result arrays (DeviceContext.prepare)."""

    def __init__(self, queries, specs, keep, results, bufs):
        self.queries, self.specs, self.keep, self.results, self.bufs = queries, specs, keep, results, bufs


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class Reaction(C.Structure):
    _fields_ = [
        ("n_rgroups", C.c_int32),
        ("_pad", C.c_int32),
        ("sizes", C.c_int64 * MAX_RGROUPS),
        ("pair_offset", C.c_int64 * MAX_RGROUPS),
        ("g_offset", C.c_uint64),
    ]


class ConstraintC(C.Structure):
    _fields_ = [("task", C.c_int32), ("_pad", C.c_int32), ("lower", C.c_double), ("upper", C.c_double)]


class QuerySpecC(C.Structure):
    _fields_ = [
        ("objective_task", C.c_int32),
        ("maximize", C.c_int32),
        ("n_constraints", C.c_int32),
        ("_pad", C.c_int32),
        ("constraints", C.POINTER(ConstraintC)),
        ("k", C.c_int64),
        ("start", C.c_uint64),
        ("end", C.c_uint64),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("pack_ms", C.c_double),
        ("seed_ms", C.c_double),
        ("scan_ms", C.c_double),
        ("select_ms", C.c_double),
        ("finalize_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("total_ms", C.c_double),
        ("scan_kernel_ms", C.c_double),
        ("candidates", C.c_int64),
        ("scan_launches", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("retries", C.c_int64),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("admitted", C.c_int64),
        ("host_prepare_us", C.c_double),
        ("host_launch_us", C.c_double),
        ("stale_sources", C.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class ResultC(C.Structure):
    _fields_ = [
        ("global_index", C.POINTER(C.c_uint64)),
        ("objective", C.POINTER(C.c_double)),
        ("constraint_values", C.POINTER(C.c_double)),
        ("reaction", C.POINTER(C.c_int32)),
        ("digits", C.POINTER(C.c_int32)),
        ("n", C.c_int64),
        ("discarded", C.c_int64),
        ("scanned", C.c_uint64),
        ("candidates", C.c_int64),
        ("admitted", C.c_int64),
        ("full_predicate", C.c_int32),
        ("_pad", C.c_int32),
    ]


class GtTaskC(C.Structure):
    _fields_ = [("flags", C.c_int32), ("salt", C.c_uint32), ("nonlinear_scale", C.c_double),
                ("nonlinear_alpha", C.c_double), ("pair_scale", C.c_double), ("pair_density", C.c_double)]


class MlpShapeC(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("dims", C.c_int32 * 7)]


class EntryC(C.Structure):
    _fields_ = [("key", C.c_uint64), ("g", C.c_uint64)]


_lib = None


def load_library(path: Path | None = None):
    """Load libapexb200.so (once).  Raises NativeError if it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else LIB_PATH
    if not p.exists():
        raise NativeError(APEX_ESTATE, f"{p} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    vp = C.c_void_p
    sig = {
        "apex_last_error": ([], C.c_char_p),
        "apex_version": ([], C.c_char_p),
        "apex_ctx_create": ([C.c_int32, vp, C.POINTER(vp)], C.c_int),
        "apex_ctx_destroy": ([vp], None),
        "apex_set_stream": ([vp, vp], C.c_int),
        "apex_load_library": ([vp, C.POINTER(Reaction), C.c_int32, C.c_int64], C.c_int),
        "apex_load_table": ([vp, vp, vp, C.c_int32, C.c_int64], C.c_int),
        "apex_load_cache": ([vp, vp, C.c_int64, C.c_int32, vp, vp, C.c_int32, vp], C.c_int),
        "apex_precompute_device": ([vp, vp, C.c_int64, C.c_int32, vp, C.c_int32, vp], C.c_int),
        "apex_query": ([vp, C.POINTER(QuerySpecC), C.c_int32, C.POINTER(ResultC), C.POINTER(Stats)], C.c_int),
        "apex_query_async": ([vp, C.POINTER(QuerySpecC), C.c_int32, C.POINTER(Stats)], C.c_int),
        "apex_query_fetch": ([vp, C.POINTER(ResultC), C.POINTER(Stats)], C.c_int),
        "apex_query_local": ([vp, C.POINTER(QuerySpecC), C.c_int32, vp, C.POINTER(C.c_int64), C.POINTER(Stats)],
                             C.c_int),
        "apex_merge_finalize": ([vp, C.POINTER(QuerySpecC), vp, C.c_int64, C.c_uint64, C.POINTER(ResultC),
                                 C.POINTER(Stats)], C.c_int),
        "apex_merge_finalize_batch": ([vp, C.POINTER(QuerySpecC), C.c_int32, vp, C.c_int32, C.c_int64, C.c_uint64,
                                       C.POINTER(ResultC), C.POINTER(Stats)], C.c_int),
        "apex_precompute_time": ([vp, C.POINTER(C.c_double)], C.c_int),
        "apex_gt_load": ([vp, vp, C.c_int64, vp, C.c_int64, vp, C.c_int32], C.c_int),
        "apex_encode_hierarchy": ([vp, vp, vp, C.c_int64, vp, vp, C.c_int64, vp, C.c_int32, C.c_int32, C.c_double, vp,
                                   C.c_int64, vp, C.c_int32, vp, vp, C.c_int32, C.c_int32, C.c_int32, vp, vp, vp, vp,
                                   vp], C.c_int),
        "apex_precompute_resident": ([vp, vp, vp, C.c_int32, vp], C.c_int),
        "apex_batch_trace": ([vp, C.POINTER(QuerySpecC), vp, C.c_int32, vp, vp], C.c_int),
        "apex_gt_topk": ([vp, C.POINTER(QuerySpecC), C.POINTER(ResultC), C.POINTER(Stats)], C.c_int),
        "apex_query_local_async": ([vp, C.POINTER(QuerySpecC), C.c_int32, vp, C.c_int64, C.POINTER(Stats)], C.c_int),
        "apex_query_local_finish": ([vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(Stats)], C.c_int),
        "apex_multi_create": ([C.c_int32, C.POINTER(C.c_int32), C.POINTER(vp)], C.c_int),
        "apex_multi_destroy": ([vp], None),
        "apex_multi_load_library": ([vp, C.POINTER(Reaction), C.c_int32, C.c_int64], C.c_int),
        "apex_multi_load_table": ([vp, vp, vp, C.c_int32, C.c_int64], C.c_int),
        "apex_multi_load_cache": ([vp, vp, C.c_int64, C.c_int32, vp, vp, C.c_int32, vp], C.c_int),
        "apex_multi_set_option": ([vp, C.c_char_p, C.c_int64], C.c_int),
        "apex_multi_query": ([vp, C.POINTER(QuerySpecC), C.c_int32, C.POINTER(ResultC), C.POINTER(Stats)], C.c_int),
        "apex_multi_info": ([vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
        "apex_set_option": ([vp, C.c_char_p, C.c_int64], C.c_int),
        "apex_get_device_info": ([vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32)], C.c_int),
        "apex_debug_thresholds": ([vp, vp, vp, vp, C.c_int64, vp, vp], C.c_int),
        "apex_debug_trace": ([vp, vp, C.c_int64, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        if (name.startswith("apex_debug_") or "APEX_B200_LIB" in os.environ) and not hasattr(lib, name):
            continue  # profiling hooks are optional; A/B runs may load older builds
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc != APEX_OK:
        msg = load_library().apex_last_error().decode(errors="replace")
        raise NativeError(rc, msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class DeviceContext:
    """Owns one apex_ctx (one GPU): resident library descriptors and table."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self.lib = load_library()
        self._ctx = C.c_void_p()
        _check(self.lib.apex_ctx_create(int(device), C.c_void_p(stream) if stream else None, C.byref(self._ctx)))
        self.device = device

    def close(self) -> None:
        if self._ctx:
            self.lib.apex_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int | None) -> None:
        _check(self.lib.apex_set_stream(self._ctx, C.c_void_p(stream) if stream else None))

    def set_option(self, name: str, value: int) -> None:
        _check(self.lib.apex_set_option(self._ctx, name.encode(), int(value)))

    def device_info(self) -> tuple[int, int, int]:
        a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
        _check(self.lib.apex_get_device_info(self._ctx, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    # -- library / table ---------------------------------------------------
    def load_library(self, sizes: list[list[int]], pair_offsets: list[list[int]], g_offsets: list[int],
                     n_pairs: int) -> None:
        n = len(sizes)
        arr = (Reaction * max(n, 1))()
        for t in range(n):
            c = len(sizes[t])
            if c > MAX_RGROUPS:
                raise NativeError(APEX_ELIMIT, f"reaction {t} has {c} R-groups (max {MAX_RGROUPS})")
            arr[t].n_rgroups = c
            for j in range(c):
                arr[t].sizes[j] = int(sizes[t][j])
                arr[t].pair_offset[j] = int(pair_offsets[t][j])
            arr[t].g_offset = int(g_offsets[t])
        _check(self.lib.apex_load_library(self._ctx, arr, n, int(n_pairs)))

    def load_table(self, values: np.ndarray, biases: np.ndarray) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32)
        b = np.ascontiguousarray(biases, dtype=np.float64)
        _check(self.lib.apex_load_table(self._ctx, _ptr(v), _ptr(b), v.shape[0], v.shape[1]))

    def load_cache(self, u: np.ndarray, head_w: np.ndarray, head_b: np.ndarray, want_values: bool = True):
        u = np.ascontiguousarray(u, dtype=np.float64)
        w = np.ascontiguousarray(head_w, dtype=np.float64)
        b = np.ascontiguousarray(head_b, dtype=np.float64)
        out = np.empty((w.shape[0], u.shape[0]), dtype=np.float32) if want_values else None
        _check(self.lib.apex_load_cache(self._ctx, _ptr(u), u.shape[0], u.shape[1], _ptr(w), _ptr(b), w.shape[0],
                                        _ptr(out) if out is not None else None))
        return out

    def precompute_time(self) -> float:
        """Device ms of the last K1 kernel (events around the launch), -1 if untimed."""
        ms = C.c_double(-1.0)
        _check(self.lib.apex_precompute_time(self._ctx, C.byref(ms)))
        return ms.value

    def precompute_device(self, u_ptr: int, n_pairs: int, d: int, w_ptr: int, n_tasks: int, out_ptr: int) -> None:
        _check(self.lib.apex_precompute_device(self._ctx, C.c_void_p(u_ptr), n_pairs, d, C.c_void_p(w_ptr), n_tasks,
                                               C.c_void_p(out_ptr)))

    # -- queries -------------------------------------------------------------
    @staticmethod
    def _specs(queries):
        """queries: list of dicts {obj, maximize, cons: [(task, lo, hi)], k, start, end}."""
        specs = (QuerySpecC * len(queries))()
        keep = []
        for i, q in enumerate(queries):
            cons = q.get("cons", [])
            carr = (ConstraintC * max(len(cons), 1))()
            for j, (t, lo, hi) in enumerate(cons):
                carr[j].task = int(t)
                carr[j].lower = float(lo)
                carr[j].upper = float(hi)
            keep.append(carr)
            specs[i].objective_task = int(q["obj"])
            specs[i].maximize = 1 if q["maximize"] else 0
            specs[i].n_constraints = len(cons)
            specs[i].constraints = C.cast(carr, C.POINTER(ConstraintC))
            specs[i].k = int(q["k"])
            specs[i].start = int(q["start"])
            specs[i].end = int(q["end"])
        return specs, keep

    @staticmethod
    def _result_buffers(queries):
        results = (ResultC * len(queries))()
        bufs = []
        for i, q in enumerate(queries):
            k = max(int(q["k"]), 1)
            m = len(q.get("cons", []))
            b = {
                "g": np.empty(k, dtype=np.uint64),
                "objective": np.empty(k, dtype=np.float64),
                "constraint_values": np.empty((k, m), dtype=np.float64),
                "reaction": np.empty(k, dtype=np.int32),
                "digits": np.empty((k, MAX_RGROUPS), dtype=np.int32),
            }
            bufs.append(b)
            results[i].global_index = b["g"].ctypes.data_as(C.POINTER(C.c_uint64))
            results[i].objective = b["objective"].ctypes.data_as(C.POINTER(C.c_double))
            results[i].constraint_values = b["constraint_values"].ctypes.data_as(C.POINTER(C.c_double))
            results[i].reaction = b["reaction"].ctypes.data_as(C.POINTER(C.c_int32))
            results[i].digits = b["digits"].ctypes.data_as(C.POINTER(C.c_int32))
        return results, bufs

    @staticmethod
    def _unpack(results, bufs):
        out = []
        for i, b in enumerate(bufs):
            n = results[i].n
            out.append({
                "g": b["g"][:n],
                "objective": b["objective"][:n],
                "constraint_values": b["constraint_values"][:n],
                "reaction": b["reaction"][:n],
                "digits": b["digits"][:n],
                "n": n,
                "discarded": results[i].discarded,
                "scanned": results[i].scanned,
                "candidates": results[i].candidates,
                "admitted": results[i].admitted,
                "full_predicate": results[i].full_predicate,
            })
        return out

    def query(self, queries: list[dict]) -> tuple[list[dict], dict]:
        """Run a batch; returns per-query numpy result arrays and the stats."""
        specs, keep = self._specs(queries)
        results, bufs = self._result_buffers(queries)
        st = Stats()
        _check(self.lib.apex_query(self._ctx, specs, len(queries), results, C.byref(st)))
        del keep
        return self._unpack(results, bufs), st.as_dict()

    def prepare(self, queries: list[dict]) -> "PreparedBatch":
        """Descriptors and caller-owned result arrays built once, for callers
        that run the same batch shape repeatedly (the C-ABI usage pattern:
        host buffers allocated by the caller and reused)."""
        specs, keep = self._specs(queries)
        results, bufs = self._result_buffers(queries)
        for b in bufs:  # touch the pages once so no call pays first-touch faults
            for a in b.values():
                a.fill(0)
        return PreparedBatch(queries, specs, keep, results, bufs)

    def prepare_views(self, queries: list[dict]) -> "PreparedBatch":
        """Descriptors built once; results come back as views into the
        context's pinned host block (no host copy; valid until the next call)."""
        specs, keep = self._specs(queries)
        return PreparedBatch(queries, specs, keep, None, None)

    def run_views_raw(self, pb: "PreparedBatch"):
        """The bare C-ABI call in view mode: apex_query with NULL result
        arrays, so every result row lands in the context's pinned host block
        (device pass + D2H inside the call).  Returns the apex_result array
        and the stats; views_of() turns them into numpy views."""
        results = (ResultC * len(pb.queries))()  # all arrays NULL: view mode
        st = Stats()
        _check(self.lib.apex_query(self._ctx, pb.specs, len(pb.queries), results, C.byref(st)))
        return results, st

    def run_views(self, pb: "PreparedBatch") -> tuple[list[dict], dict]:
        results, st = self.run_views_raw(pb)
        return self.views_of(pb, results, st)

    def views_of(self, pb: "PreparedBatch", results, st) -> tuple[list[dict], dict]:
        # one numpy view over the pinned block, sliced per query
        addr = [C.cast(results[i].global_index, C.c_void_p).value or 0 for i in range(len(pb.queries))]
        base = min(a for a in addr if a) if any(addr) else 0
        end = 0
        for i, q in enumerate(pb.queries):
            if addr[i]:
                kk = max(int(q["k"]), 1)
                end = max(end, addr[i] + kk * (8 + 8 + 8 * len(q.get("cons", [])) + 4 + 4 * MAX_RGROUPS))
        block = np.frombuffer((C.c_uint8 * (end - base)).from_address(base), dtype=np.uint8) if base else None
        out = []
        u64, f64, i32 = np.uint64, np.float64, np.int32
        for i, q in enumerate(pb.queries):
            r = results[i]
            n, m = r.n, len(q.get("cons", []))
            kk = max(int(q["k"]), 1)
            o = addr[i] - base
            if n and block is not None and addr[i]:
                cv = (np.frombuffer(block, f64, n * m, o + 16 * kk).reshape(n, m) if m
                      else np.empty((n, 0), f64))
                d = {"g": np.frombuffer(block, u64, n, o), "objective": np.frombuffer(block, f64, n, o + 8 * kk),
                     "constraint_values": cv, "reaction": np.frombuffer(block, i32, n, o + (16 + 8 * m) * kk),
                     "digits": np.frombuffer(block, i32, n * MAX_RGROUPS,
                                             o + (20 + 8 * m) * kk).reshape(n, MAX_RGROUPS)}
            else:
                d = {"g": np.empty(0, u64), "objective": np.empty(0, f64), "constraint_values": np.empty((0, m), f64),
                     "reaction": np.empty(0, i32), "digits": np.empty((0, MAX_RGROUPS), i32)}
            d.update(n=n, discarded=r.discarded, scanned=r.scanned, candidates=r.candidates, admitted=r.admitted,
                     full_predicate=r.full_predicate)
            out.append(d)
        return out, st.as_dict()

    def run(self, pb: "PreparedBatch") -> tuple[list[dict], dict]:
        """apex_query on a prepared batch; the returned arrays are views of the
        batch's buffers (overwritten by the next run of the same batch)."""
        st = Stats()
        _check(self.lib.apex_query(self._ctx, pb.specs, len(pb.queries), pb.results, C.byref(st)))
        return self._unpack(pb.results, pb.bufs), st.as_dict()

    def run_async(self, pb: "PreparedBatch") -> dict:
        """apex_query_async on a prepared batch (descriptors built once)."""
        st = Stats()
        _check(self.lib.apex_query_async(self._ctx, pb.specs, len(pb.queries), C.byref(st)))
        self._inflight = pb.queries
        return st.as_dict()

    def query_async(self, queries: list[dict]) -> dict:
        """Enqueue a batch (one shared range, k >= 1) without a host sync."""
        specs, keep = self._specs(queries)
        st = Stats()
        _check(self.lib.apex_query_async(self._ctx, specs, len(queries), C.byref(st)))
        self._inflight = queries
        del keep
        return st.as_dict()

    def query_fetch(self) -> tuple[list[dict], dict]:
        queries = self._inflight
        results, bufs = self._result_buffers(queries)
        st = Stats()
        _check(self.lib.apex_query_fetch(self._ctx, results, C.byref(st)))
        return self._unpack(results, bufs), st.as_dict()

    def query_local(self, queries: list[dict], out_dev_ptr: int) -> tuple[list[int], dict]:
        specs, keep = self._specs(queries)
        counts = (C.c_int64 * len(queries))()
        st = Stats()
        _check(self.lib.apex_query_local(self._ctx, specs, len(queries), C.c_void_p(out_dev_ptr), counts, C.byref(st)))
        del keep
        return [counts[i] for i in range(len(queries))], st.as_dict()

    def query_local_async(self, queries: list[dict], out_dev_ptr: int, stride: int) -> dict:
        """Enqueue the local step + padded export ([query][stride] entries at
        out_dev_ptr) on the context stream; no host sync (apex_query_local_async)."""
        specs, keep = self._specs(queries)
        st = Stats()
        _check(self.lib.apex_query_local_async(self._ctx, specs, len(queries), C.c_void_p(out_dev_ptr), int(stride),
                                               C.byref(st)))
        self._local_n = len(queries)
        del keep
        return st.as_dict()

    def query_local_finish(self) -> tuple[list[int], bool, dict]:
        """Validate the local step in flight: (counts, rerun, stats); rerun is
        True when an overflow forced an exact re-run (gather + merge again)."""
        counts = (C.c_int64 * self._local_n)()
        rerun = C.c_int32(0)
        st = Stats()
        _check(self.lib.apex_query_local_finish(self._ctx, counts, C.byref(rerun), C.byref(st)))
        return [counts[i] for i in range(self._local_n)], bool(rerun.value), st.as_dict()

    def merge_finalize_batch(self, queries: list[dict], entries_dev_ptr: int, n_src: int, stride: int,
                             total_scanned: int, prepared: "PreparedBatch | None" = None):
        """Global top-k of every query from all-gathered local entries laid out
        [n_src][len(queries)][stride] (apex_merge_finalize_batch)."""
        pb = prepared if prepared is not None else self.prepare(queries)
        st = Stats()
        _check(self.lib.apex_merge_finalize_batch(self._ctx, pb.specs, len(queries), C.c_void_p(entries_dev_ptr),
                                                  int(n_src), int(stride), int(total_scanned), pb.results,
                                                  C.byref(st)))
        return self._unpack(pb.results, pb.bufs), st.as_dict()

    def merge_finalize(self, query: dict, entries_dev_ptr: int, n_entries: int, total_scanned: int):
        specs, keep = self._specs([query])
        k = max(int(query["k"]), 1)
        m = len(query.get("cons", []))
        b = {
            "g": np.empty(k, dtype=np.uint64),
            "objective": np.empty(k, dtype=np.float64),
            "constraint_values": np.empty((k, m), dtype=np.float64),
            "reaction": np.empty(k, dtype=np.int32),
            "digits": np.empty((k, MAX_RGROUPS), dtype=np.int32),
        }
        res = ResultC()
        res.global_index = b["g"].ctypes.data_as(C.POINTER(C.c_uint64))
        res.objective = b["objective"].ctypes.data_as(C.POINTER(C.c_double))
        res.constraint_values = b["constraint_values"].ctypes.data_as(C.POINTER(C.c_double))
        res.reaction = b["reaction"].ctypes.data_as(C.POINTER(C.c_int32))
        res.digits = b["digits"].ctypes.data_as(C.POINTER(C.c_int32))
        st = Stats()
        _check(self.lib.apex_merge_finalize(self._ctx, specs, C.c_void_p(entries_dev_ptr), int(n_entries),
                                            int(total_scanned), C.byref(res), C.byref(st)))
        n = res.n
        del keep
        return {
            "g": b["g"][:n], "objective": b["objective"][:n], "constraint_values": b["constraint_values"][:n],
            "reaction": b["reaction"][:n], "digits": b["digits"][:n], "n": n, "discarded": res.discarded,
            "scanned": res.scanned,
        }, st.as_dict()

    def batch_trace(self, query: dict, batch_end: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
        """BatchTrace new / carried counts of the chain of batches ending at
        batch_end (apex_batch_trace)."""
        specs, keep = self._specs([query])
        ends = np.ascontiguousarray(batch_end, dtype=np.uint64)
        new = np.zeros(len(ends), dtype=np.int64)
        carried = np.zeros(len(ends), dtype=np.int64)
        _check(self.lib.apex_batch_trace(self._ctx, specs, _ptr(ends), len(ends), _ptr(new), _ptr(carried)))
        del keep
        return new, carried

    def gt_load(self, member_ids: np.ndarray, latents: np.ndarray, tasks: list[dict]) -> None:
        """Ground-truth oracle tables (apex_gt_load): member_ids [n_pairs],
        latents [n_tasks][n_synthons], per task {flags, salt, nonlinear_scale,
        nonlinear_alpha, pair_scale, pair_density}."""
        m = np.ascontiguousarray(member_ids, dtype=np.int64)
        lat = np.ascontiguousarray(latents, dtype=np.float64)
        arr = (GtTaskC * len(tasks))()
        for i, t in enumerate(tasks):
            for k, v in t.items():
                setattr(arr[i], k, v)
        _check(self.lib.apex_gt_load(self._ctx, _ptr(m), len(m), _ptr(lat), lat.shape[1], arr, len(tasks)))

    def gt_topk(self, query: dict) -> tuple[dict, dict]:
        """Oracle top-j of one query dict {obj, maximize, cons, k=j, start, end}."""
        specs, keep = self._specs([query])
        results, bufs = self._result_buffers([query])
        st = Stats()
        _check(self.lib.apex_gt_topk(self._ctx, specs, results, C.byref(st)))
        del keep
        return self._unpack(results, bufs)[0], st.as_dict()

    def encode_hierarchy(self, shapes: list[list[int]], params: np.ndarray, token_bytes: np.ndarray,
                         token_off: np.ndarray, salt: bytes, p: int, scale: float, member_ids: np.ndarray,
                         rg_offsets: np.ndarray, rg_parent: np.ndarray, rx_offsets: np.ndarray, d: int, d_u: int,
                         want=("u", "h_s", "h_r", "h_t", "features")) -> dict:
        """K8 (apex_encode_hierarchy); returns the requested host copies.  The
        pair matrix u stays resident for precompute_resident."""
        nets = (MlpShapeC * 7)()
        for k, dims in enumerate(shapes):
            nets[k].n_layers = len(dims) - 1
            for i, x in enumerate(dims):
                nets[k].dims[i] = int(x)
        params = np.ascontiguousarray(params, dtype=np.float64)
        tb = np.ascontiguousarray(token_bytes, dtype=np.uint8)
        to = np.ascontiguousarray(token_off, dtype=np.int64)
        mem = np.ascontiguousarray(member_ids, dtype=np.int64)
        rgo = np.ascontiguousarray(rg_offsets, dtype=np.int64)
        par = np.ascontiguousarray(rg_parent, dtype=np.int32)
        rxo = np.ascontiguousarray(rx_offsets, dtype=np.int64)
        sb = np.frombuffer(salt, dtype=np.uint8).copy()
        n_syn, n_pairs, n_rg, n_rx = len(to) - 1, len(mem), len(rgo) - 1, len(rxo) - 1
        d_s, d_r, d_t = shapes[0][-1], shapes[2][-1], shapes[4][-1]
        out = {"u": np.empty((n_pairs, d)) if "u" in want else None,
               "h_s": np.empty((n_syn, d_s)) if "h_s" in want else None,
               "h_r": np.empty((n_rg, d_r)) if "h_r" in want else None,
               "h_t": np.empty((n_rx, d_t)) if "h_t" in want else None,
               "features": np.empty((n_syn, p)) if "features" in want else None}
        ptr = lambda a: _ptr(a) if a is not None else None  # noqa: E731
        self._u_pairs = n_pairs
        _check(self.lib.apex_encode_hierarchy(self._ctx, nets, _ptr(params), len(params), _ptr(tb), _ptr(to), n_syn,
                                              _ptr(sb), len(sb), int(p), float(scale), _ptr(mem), n_pairs, _ptr(rgo),
                                              n_rg, _ptr(par), _ptr(rxo), n_rx, int(d), int(d_u), ptr(out["u"]),
                                              ptr(out["h_s"]), ptr(out["h_r"]), ptr(out["h_t"]), ptr(out["features"])))
        return {k: v for k, v in out.items() if v is not None}

    def precompute_resident(self, head_w: np.ndarray, head_b: np.ndarray, want_values: bool = True):
        """K1 from the resident K8 pair matrix (apex_precompute_resident); the
        table becomes resident.  Returns the host copy of the table if asked."""
        w = np.ascontiguousarray(head_w, dtype=np.float64)
        b = np.ascontiguousarray(head_b, dtype=np.float64)
        out = np.empty((w.shape[0], self._u_pairs), dtype=np.float32) if want_values else None
        _check(self.lib.apex_precompute_resident(self._ctx, _ptr(w), _ptr(b), w.shape[0],
                                                 _ptr(out) if out is not None else None))
        return out

    def debug_thresholds(self, p: np.ndarray, b: np.ndarray, beta: np.ndarray):
        p = np.ascontiguousarray(p, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        beta = np.ascontiguousarray(beta, dtype=np.float64)
        up = np.empty(len(p), dtype=np.float32)
        lo = np.empty(len(p), dtype=np.float32)
        _check(self.lib.apex_debug_thresholds(self._ctx, _ptr(p), _ptr(b), _ptr(beta), len(p), _ptr(up), _ptr(lo)))
        return up, lo

    def debug_trace(self, cap: int) -> np.ndarray:
        """Per-item records of the last admission scan (needs set_option("trace", cap))."""
        out = np.zeros((cap, 8), dtype=np.uint64)
        n = C.c_int64(0)
        _check(self.lib.apex_debug_trace(self._ctx, _ptr(out), cap, C.byref(n)))
        return out[:n.value]


class MultiDeviceContext:
    """Owns one apex_multi: one process and host thread driving several GPUs
    (index range sharded per device, exact local top-k per device, merge on the
    first device with the gather fused into its load kernel over NVLink peer
    pointers).  Same query results as DeviceContext; device ids may repeat."""

    def __init__(self, devices: list[int]):
        self.lib = load_library()
        self._m = C.c_void_p()
        ids = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        _check(self.lib.apex_multi_create(len(devices), ids, C.byref(self._m)))
        self.devices = list(devices)

    def close(self) -> None:
        if self._m:
            self.lib.apex_multi_destroy(self._m)
            self._m = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> tuple[int, bool]:
        n, peer = C.c_int32(), C.c_int32()
        _check(self.lib.apex_multi_info(self._m, C.byref(n), C.byref(peer)))
        return n.value, bool(peer.value)

    def set_option(self, name: str, value: int) -> None:
        _check(self.lib.apex_multi_set_option(self._m, name.encode(), int(value)))

    def load_library(self, sizes, pair_offsets, g_offsets, n_pairs) -> None:
        n = len(sizes)
        arr = (Reaction * max(n, 1))()
        for t in range(n):
            c = len(sizes[t])
            if c > MAX_RGROUPS:
                raise NativeError(APEX_ELIMIT, f"reaction {t} has {c} R-groups (max {MAX_RGROUPS})")
            arr[t].n_rgroups = c
            for j in range(c):
                arr[t].sizes[j] = int(sizes[t][j])
                arr[t].pair_offset[j] = int(pair_offsets[t][j])
            arr[t].g_offset = int(g_offsets[t])
        _check(self.lib.apex_multi_load_library(self._m, arr, n, int(n_pairs)))

    def load_table(self, values: np.ndarray, biases: np.ndarray) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32)
        b = np.ascontiguousarray(biases, dtype=np.float64)
        _check(self.lib.apex_multi_load_table(self._m, _ptr(v), _ptr(b), v.shape[0], v.shape[1]))

    def load_cache(self, u: np.ndarray, head_w: np.ndarray, head_b: np.ndarray) -> np.ndarray:
        u = np.ascontiguousarray(u, dtype=np.float64)
        w = np.ascontiguousarray(head_w, dtype=np.float64)
        b = np.ascontiguousarray(head_b, dtype=np.float64)
        out = np.empty((w.shape[0], u.shape[0]), dtype=np.float32)
        _check(self.lib.apex_multi_load_cache(self._m, _ptr(u), u.shape[0], u.shape[1], _ptr(w), _ptr(b), w.shape[0],
                                              _ptr(out)))
        return out

    def query(self, queries: list[dict]) -> tuple[list[dict], dict]:
        specs, keep = DeviceContext._specs(queries)
        results, bufs = DeviceContext._result_buffers(queries)
        st = Stats()
        _check(self.lib.apex_multi_query(self._m, specs, len(queries), results, C.byref(st)))
        del keep
        return DeviceContext._unpack(results, bufs), st.as_dict()
