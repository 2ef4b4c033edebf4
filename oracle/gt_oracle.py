"""CPU ORACLE for the ground-truth evaluation path — TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module, as the checker of the device's
evalkit.oracle_topk (paper_2510_24380_b200/evalkit.py, csrc/gt.cuh).  A numpy
restatement of the reference's synthetic ground-truth oracle and its
exhaustive top-j:

  * _splitmix / _pair_uniform / pair_coefficient   props.py:162-195
    (exact uint64 arithmetic)
  * oracle_block_values                            props.py:218-264
    base = ((lat[s0] + lat[s1]) + lat[s2]), + scale * tanh(alpha * base) for
    +nonlinear tasks, + the pair coefficients in lexicographic R-group pair
    order for +pairwise tasks
  * oracle_topk                                    evalkit.py:49-90
    oracle-feasible products (every constraint lo <= v <= hi) ranked by
    (signed objective desc, global index asc), best j

Pinned by tests/golden/gt_golden.json (recorded from the reference itself by
tests/golden/make_gt_golden.py): tests/test_oracle_golden.py.
"""

from __future__ import annotations

import numpy as np

M1 = np.uint64(0x9E3779B97F4A7C15)
M2 = np.uint64(0xBF58476D1CE4E5B9)
M3 = np.uint64(0x94D049BB133111EB)


def splitmix(x):
    with np.errstate(over="ignore"):
        x = (x + M1).astype(np.uint64)
        x ^= x >> np.uint64(30)
        x = (x * M2).astype(np.uint64)
        x ^= x >> np.uint64(27)
        x = (x * M3).astype(np.uint64)
        x ^= x >> np.uint64(31)
    return x


def pair_uniform(sa, sb, salt: int):
    a = np.asarray(sa, dtype=np.uint64)
    b = np.asarray(sb, dtype=np.uint64)
    lo, hi = np.minimum(a, b), np.maximum(a, b)
    with np.errstate(over="ignore"):
        h = splitmix(splitmix(lo * M1 + np.uint64(salt)) ^ (hi * M3))
    return (h >> np.uint64(11)).astype(np.float64) / float(1 << 53)


def pair_coefficient(task, salt: int, sa, sb):
    gate = pair_uniform(sa, sb, salt)
    value = pair_uniform(sa, sb, salt + 0x51ED)
    return np.where(gate < task.pair_density, task.pair_scale * (2.0 * value - 1.0), 0.0)


def task_salt(seed: int, index: int) -> int:
    return (seed * 1000003 + index * 8191) & 0xFFFFFFFF


def values(oracle, task_index: int, sids: np.ndarray) -> np.ndarray:
    """Oracle values of products given their synthon ids [n, c] (R-group order)."""
    task = oracle.tasks[task_index]
    lat = np.asarray(task.latent, dtype=np.float64)
    parts = set(task.mode.split("+"))
    base = lat[sids[:, 0]]
    for j in range(1, sids.shape[1]):
        base = base + lat[sids[:, j]]
    v = base.copy()
    if "nonlinear" in parts:
        v = v + task.nonlinear_scale * np.tanh(task.nonlinear_alpha * base)
    if "pairwise" in parts:
        salt = task_salt(int(oracle.seed), task_index)
        for a in range(sids.shape[1]):
            for b in range(a + 1, sids.shape[1]):
                v = v + pair_coefficient(task, salt, sids[:, a], sids[:, b])
    return v


def topk(library, oracle, obj: int, maximize: bool, cons, j: int, start: int = 0, end: int | None = None):
    """Exhaustive oracle top-j: (g, objective) arrays best-first.  cons:
    [(task index, lower, upper)].  Vectorized per reaction."""
    offs = [0]
    for rx in library.reactions:
        n = 1
        for rg in rx.rgroups:
            n *= len(rg.synthon_ids)
        offs.append(offs[-1] + n)
    end = offs[-1] if end is None else end
    gs, ss, os = [], [], []
    for t, rx in enumerate(library.reactions):
        lo, hi = max(start, offs[t]), min(end, offs[t + 1])
        if lo >= hi:
            continue
        loc = np.arange(lo - offs[t], hi - offs[t], dtype=np.int64)
        sizes = [len(rg.synthon_ids) for rg in rx.rgroups]
        sids = np.zeros((len(loc), len(sizes)), dtype=np.int64)
        rem = loc.copy()
        for jj in range(len(sizes) - 1, -1, -1):
            d = rem % sizes[jj]
            rem //= sizes[jj]
            sids[:, jj] = np.asarray(rx.rgroups[jj].synthon_ids, dtype=np.int64)[d]
        feas = np.ones(len(loc), dtype=bool)
        for task, lower, upper in cons:
            v = values(oracle, task, sids)
            feas &= (v >= lower) & (v <= upper)
        o = values(oracle, obj, sids)
        s = o if maximize else -o
        idx = np.nonzero(feas)[0]
        gs.append(offs[t] + loc[idx])
        ss.append(s[idx])
        os.append(o[idx])
    if not gs:
        return np.empty(0, dtype=np.int64), np.empty(0)
    g = np.concatenate(gs)
    s = np.concatenate(ss)
    o = np.concatenate(os)
    order = np.lexsort((g, -s))[:j]
    return g[order], o[order]
