"""Ground-truth evaluation on the B200.

Mirror of the reference's exhaustive oracle top-j, ``evalkit.oracle_topk``
(reference ``pkg/src/apexcsl/evalkit.py:49-90``), computed on the device by
``apex_gt_topk`` (csrc/gt.cuh): every product of the range is evaluated with
the synthetic ground-truth oracle (``props.oracle_block_values``,
props.py:218-264: additive latents, the tanh term, the splitmix pairwise
terms), oracle-infeasible products are excluded (``violation == 0``), and the
best j by (objective in the query's direction desc, global index asc) are
returned best-first — without the reference's 1e8-product enumeration guard
(evalkit.py:23, 60-64), which exists because the CPU scan is too slow past it.

Same name, arguments and result shape (``OracleTopK`` of ``OracleEntry``
rows, built with the caller's classes when the oracle is a reference object).
Values agree with the reference bit for bit except through ``tanh``, whose
CUDA and numpy implementations may differ in the last ulp (docking tasks).
"""

from __future__ import annotations

import sys
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .csl import MultiIndex, product_count
from .engine import _error, default_device


@dataclass
class OracleEntry:
    global_index: int
    chi: MultiIndex
    objective: float


@dataclass
class OracleTopK:
    entries: list
    query: object
    j: int

    def global_indices(self) -> set:
        return {e.global_index for e in self.entries}


class _GtBound:
    """A device context holding one library's index space and one oracle."""

    def __init__(self, library, oracle, device):
        dev = device[0] if isinstance(device, (list, tuple)) else device
        self.ctx = _native.DeviceContext(int(dev))
        sizes, pair_off, g_off, members = [], [], [], []
        p, g = 0, 0
        for rx in library.reactions:
            s, o = [], []
            for rg in rx.rgroups:
                s.append(len(rg.synthon_ids))
                o.append(p)
                members.extend(rg.synthon_ids)
                p += len(rg.synthon_ids)
            sizes.append(s)
            pair_off.append(o)
            g_off.append(g)
            n = 1
            for x in s:
                n *= x
            g += n
        self.ctx.load_library(sizes, pair_off, g_off, p)
        # a one-task zero table: the merge's decode machinery needs a resident table
        self.ctx.load_table(np.zeros((1, max(p, 1)), dtype=np.float32)[:, :p], np.zeros(1))
        tasks, lat = [], []
        for i, t in enumerate(oracle.tasks):
            parts = set(t.mode.split("+"))
            flags = (1 if "nonlinear" in parts else 0) | (2 if "pairwise" in parts else 0)
            tasks.append({"flags": flags, "salt": (int(oracle.seed) * 1000003 + i * 8191) & 0xFFFFFFFF,
                          "nonlinear_scale": float(t.nonlinear_scale), "nonlinear_alpha": float(t.nonlinear_alpha),
                          "pair_scale": float(t.pair_scale), "pair_density": float(t.pair_density)})
            lat.append(np.asarray(t.latent, dtype=np.float64))
        width = max(len(x) for x in lat)
        latents = np.zeros((len(lat), width))
        for i, x in enumerate(lat):
            latents[i, : len(x)] = x
        self.ctx.gt_load(np.asarray(members, dtype=np.int64), latents, tasks)
        self.task_names = [t.name for t in oracle.tasks]


_GT: dict = {}


def _bind(library, oracle, device) -> _GtBound:
    key = (id(library), id(oracle), device if not isinstance(device, list) else tuple(device))
    hit = _GT.get(key)
    if hit is not None and hit[0]() is library and hit[1]() is oracle:
        return hit[2]
    b = _GtBound(library, oracle, device)
    if len(_GT) >= 2:
        _GT.pop(next(iter(_GT)))
    _GT[key] = (weakref.ref(library), weakref.ref(oracle), b)
    return b


def _oracle_task(names, name):
    try:
        return names.index(name)
    except ValueError:
        raise _error(f"unknown task {name!r}") from None


def oracle_topk(library, oracle, query, j: int, index_range=None, device=None):
    """True top-j oracle-feasible products, best first (evalkit.py:49-90), on
    the device."""
    total = product_count(library)
    start, end = index_range if index_range is not None else (0, total)
    if not 0 <= start <= end <= total:
        raise _error(f"index range [{start}, {end}) invalid")
    mod = sys.modules.get(type(oracle).__module__.replace("props", "evalkit"))
    entry_cls = getattr(mod, "OracleEntry", OracleEntry) if mod else OracleEntry
    topk_cls = getattr(mod, "OracleTopK", OracleTopK) if mod else OracleTopK
    if j <= 0 or end == start:
        return topk_cls(entries=[], query=query, j=j)
    b = _bind(library, oracle, default_device() if device is None else device)
    names = b.task_names
    nq = {"obj": _oracle_task(names, query.objective), "maximize": query.direction == "maximize",
          "cons": [(_oracle_task(names, c.task), float(c.lower), float(c.upper)) for c in query.constraints],
          "k": int(j), "start": int(start), "end": int(end)}
    try:
        res, _ = b.ctx.gt_topk(nq)
    except _native.NativeError as exc:
        raise _error(str(exc)) from None
    mi_cls = getattr(sys.modules.get(type(library).__module__), "MultiIndex", MultiIndex)
    entries = []
    for g, o, t, d in zip(res["g"].tolist(), res["objective"].tolist(), res["reaction"].tolist(),
                          res["digits"].tolist()):
        rx = library.reactions[t]
        chi = mi_cls(rx.reaction_id, tuple((rg.rgroup_id, rg.synthon_ids[x]) for rg, x in zip(rx.rgroups, d)))
        entries.append(entry_cls(int(g), chi, float(o)))
    return topk_cls(entries=entries, query=query, j=j)


# ---------------------------------------------------------------------------
# mirror oracle types (props.py:109-160), for callers without the reference
# package: the fields the device path reads
# ---------------------------------------------------------------------------

@dataclass
class TaskDef:
    name: str
    mode: str
    latent: np.ndarray
    nonlinear_scale: float = 0.0
    nonlinear_alpha: float = 0.05
    pair_scale: float = 0.0
    pair_density: float = 0.05


@dataclass
class GroundTruthOracle:
    tasks: list
    seed: int

    @property
    def task_names(self) -> list:
        return [t.name for t in self.tasks]
