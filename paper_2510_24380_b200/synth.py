"""Seeded synthetic CSL shapes, random-init heads and queries.

Shapes: per reaction c in {2, 3} (fraction ``frac3`` three-component), R-group
sizes round(exp(N(mu_c, sigma))) clipped to [2, 2e5], then rescaled by
f^(1/c) until the product count is within 0.2% of the target.  No synthon
sharing; reaction ids are positions; R-group ids and synthon ids are global
and dense, so the table's pair rows are R-group-major in declaration order
(factorizer.py:87-106 ``build_context``).

Model: a synthetic associative-embedding cache u (n_pairs x 64, iid N(0,1),
standing in for the factorizer output shape) and random-init linear heads
(0.01 * N(0,1), surrogate.py:178) for the 11 tasks dock_a..e, mw, logp, hbd,
hba, rotb, tpsa (props.py:307-308).  Property heads are affinely calibrated
(w <- a*w, b <- b') so a seeded uniform product sample has the target mean/std
(mw 400+-80, logp 3+-1.5, hbd 2+-1.2, hba 6+-2, rotb 6+-2.5, tpsa 90+-30), which
makes the RDKit-style preset bounds bite.  The table itself is produced on the
GPU by K1 (fp64 head_w @ u^T, fp32 rounding) or, for CPU-only use, by numpy.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DOCKING_TASKS = ["dock_a", "dock_b", "dock_c", "dock_d", "dock_e"]
PROPERTY_TASKS = ["mw", "logp", "hbd", "hba", "rotb", "tpsa"]
TASKS = DOCKING_TASKS + PROPERTY_TASKS
CALIBRATION = {"mw": (400.0, 80.0), "logp": (3.0, 1.5), "hbd": (2.0, 1.2), "hba": (6.0, 2.0),
               "rotb": (6.0, 2.5), "tpsa": (90.0, 30.0)}

# presets.py:11-34 (name -> [(task, lower, upper)])
INF = float("inf")
PRESETS = {
    "lipinski": [("mw", -INF, 500.0), ("logp", -INF, 5.0), ("hbd", -INF, 5.0), ("hba", -INF, 10.0)],
    "veber": [("rotb", -INF, 10.0), ("tpsa", -INF, 140.0)],
    "pfizer_3_75": [("logp", -INF, 3.0), ("tpsa", 75.0, INF)],
    "astex_ro3": [("mw", -INF, 300.0), ("logp", -INF, 3.0), ("hbd", -INF, 3.0), ("hba", -INF, 3.0),
                  ("rotb", -INF, 3.0), ("tpsa", -INF, 60.0)],
}


@dataclass(frozen=True)
class ShapeConfig:
    target: int
    n_reactions: int
    frac3: float
    mu2: float
    mu3: float
    sigma: float
    seed: int


SHAPES = {
    "c1": ShapeConfig(10_000_000, 40, 0.5, 5.5, 3.5, 0.6, 1),
    "c3": ShapeConfig(1_000_000_000, 60, 0.5, 7.0, 4.5, 1.0, 3),
    "c4": ShapeConfig(5_000_000_000, 120, 0.25, 8.0, 5.0, 1.0, 4),
}


@dataclass
class Shape:
    sizes: list          # per reaction, list of R-group sizes
    pair_off: list       # per reaction, table row of digit 0 of each R-group

    @property
    def n_pairs(self) -> int:
        return sum(sum(s) for s in self.sizes)

    @property
    def total(self) -> int:
        return sum(math.prod(s) for s in self.sizes)

    def g_offsets(self) -> list:
        out, g = [], 0
        for s in self.sizes:
            out.append(g)
            g += math.prod(s)
        return out


def make_shape(cfg: ShapeConfig) -> Shape:
    rng = np.random.default_rng(cfg.seed)
    comps = [3 if rng.random() < cfg.frac3 else 2 for _ in range(cfg.n_reactions)]
    raw = [np.exp(rng.normal(cfg.mu3 if c == 3 else cfg.mu2, cfg.sigma, size=c)) for c in comps]

    def sized(f):
        return [np.clip(np.round(r * f ** (1.0 / len(r))), 2, 200_000).astype(np.int64) for r in raw]

    def count(ss):
        return sum(int(np.prod(s.astype(object))) for s in ss)

    lo, hi = 1e-6, 1e6
    sizes = sized(1.0)
    for _ in range(200):
        f = math.sqrt(lo * hi)
        sizes = sized(f)
        n = count(sizes)
        if abs(n / cfg.target - 1) < 0.002:
            break
        if n < cfg.target:
            lo = f
        else:
            hi = f
    # deterministic fine adjustment on the largest reaction's first R-group
    n = count(sizes)
    if abs(n / cfg.target - 1) >= 0.002:
        big = max(range(len(sizes)), key=lambda t: count([sizes[t]]))
        rest = n - count([sizes[big]])
        inner = count([sizes[big][1:]])
        sizes[big][0] = max(2, round((cfg.target - rest) / inner))
    out_sizes = [[int(x) for x in s] for s in sizes]
    pair_off, p = [], 0
    for s in out_sizes:
        po = []
        for n_ in s:
            po.append(p)
            p += n_
        pair_off.append(po)
    return Shape(out_sizes, pair_off)


def scaled_shape(name: str, scale: int) -> Shape:
    """Shape of config `name` with the product target multiplied by `scale`
    (weak scaling: one config-sized shard per GPU)."""
    cfg = SHAPES[name]
    return make_shape(ShapeConfig(cfg.target * scale, cfg.n_reactions, cfg.frac3, cfg.mu2, cfg.mu3, cfg.sigma,
                                  cfg.seed))


def random_cache(n_pairs: int, d: int = 64, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((n_pairs, d))


def random_heads(n_tasks: int = len(TASKS), d: int = 64, seed: int = 0):
    rng = np.random.default_rng(seed + 1)
    return rng.standard_normal((n_tasks, d)) * 0.01, np.zeros(n_tasks)


def sample_products(shape: Shape, n: int, seed: int = 0):
    """Uniform product sample: returns (reaction index, digits) arrays."""
    rng = np.random.default_rng(seed + 2)
    g = np.sort(rng.integers(0, shape.total, size=n, dtype=np.uint64))
    offs = np.asarray(shape.g_offsets() + [shape.total], dtype=np.uint64)
    t = np.searchsorted(offs, g, side="right") - 1
    return g, t


def calibrate_heads(shape: Shape, u: np.ndarray, head_w: np.ndarray, head_b: np.ndarray, n_sample: int = 100_000,
                    seed: int = 0):
    """Affine calibration of the property heads on a uniform product sample."""
    g, t = sample_products(shape, n_sample, seed)
    offs = shape.g_offsets()
    rows = []  # per sample, the pair rows of its R-groups
    for gi, ti in zip(g.tolist(), t.tolist()):
        rem = gi - offs[ti]
        s = shape.sizes[ti]
        digs = [0] * len(s)
        for j in range(len(s) - 1, -1, -1):
            rem, digs[j] = divmod(rem, s[j])
        rows.append([shape.pair_off[ti][j] + digs[j] for j in range(len(s))])
    w = head_w.copy()
    b = head_b.copy()
    for i, name in enumerate(TASKS):
        if name not in CALIBRATION:
            continue
        contrib = u @ w[i] if u.shape[0] <= 2_000_000 else None
        vals = np.array([sum(float(contrib[r]) for r in rr) if contrib is not None
                         else sum(float(u[r] @ w[i]) for r in rr) for rr in rows])
        mean, std = CALIBRATION[name]
        a = std / max(vals.std(), 1e-12)
        w[i] *= a
        b[i] = mean - a * vals.mean()
    return w, b


def host_table(u: np.ndarray, head_w: np.ndarray) -> np.ndarray:
    """engine.py:82 on the host (numpy BLAS): fl32(head_w @ u^T)."""
    return (head_w @ u.T).astype(np.float32)


def c2_queries():
    """Config 2: 5 objectives (dock_a..e, minimize) x 4 presets, k = 1000.
    (Interpretation of "5 objectives x RDKit-property constraint sets".)"""
    out = []
    for obj in DOCKING_TASKS:
        for preset in ("lipinski", "veber", "pfizer_3_75", "astex_ro3"):
            out.append({"objective": obj, "direction": "minimize", "constraints": PRESETS[preset], "k": 1000,
                        "name": f"{obj}/{preset}"})
    return out


def c1_query():
    return {"objective": "dock_a", "direction": "minimize",
            "constraints": [("mw", -INF, 500.0), ("logp", -INF, 5.0)], "k": 100}


def c3_query():
    return {"objective": "dock_a", "direction": "minimize", "constraints": PRESETS["lipinski"], "k": 1000}


def c4_query():
    return {"objective": "dock_a", "direction": "minimize",
            "constraints": [("mw", 300.0, 500.0), ("logp", -1.0, 5.0), ("tpsa", 20.0, 140.0), ("hbd", -INF, 5.0),
                            ("hba", -INF, 10.0)], "k": 10_000}


def c5_queries(n: int = 1000, seed: int = 5):
    """Config 5: random objective (dock_a..e, minimize), 0-6 property windows
    from pairs of calibrated quantiles, k in {100, 1000, 10000}."""
    rng = np.random.default_rng(seed)
    from statistics import NormalDist
    out = []
    for _ in range(n):
        obj = DOCKING_TASKS[int(rng.integers(0, 5))]
        m = int(rng.integers(0, 7))
        props = list(rng.choice(PROPERTY_TASKS, size=m, replace=False)) if m else []
        cons = []
        for p in props:
            mean, std = CALIBRATION[p]
            qa, qb = sorted(rng.uniform(0.0, 1.0, size=2))
            lo = mean + std * NormalDist().inv_cdf(max(qa, 1e-6)) if qa > 0.05 else -INF
            hi = mean + std * NormalDist().inv_cdf(min(qb, 1 - 1e-6)) if qb < 0.95 else INF
            if not lo < hi:
                lo, hi = -INF, INF
            cons.append((str(p), float(lo), float(hi)))
        k = [100, 1000, 10_000][int(rng.integers(0, 3))]
        out.append({"objective": obj, "direction": "minimize", "constraints": cons, "k": k})
    return out


def to_native(q: dict, start: int, end: int) -> dict:
    """Query dict (task names) -> native spec dict (task indices)."""
    return {"obj": TASKS.index(q["objective"]), "maximize": q["direction"] == "maximize",
            "cons": [(TASKS.index(t), lo, hi) for t, lo, hi in q["constraints"]], "k": q["k"],
            "start": start, "end": end}


def build_model(shape: Shape, seed: int = 1, n_sample: int = 20000):
    """The benchmark model of a shape: synthetic pair-embedding cache, random
    heads, property heads calibrated on a uniform product sample."""
    u = random_cache(shape.n_pairs, seed=seed)
    w, b = random_heads(seed=seed)
    w, b = calibrate_heads(shape, u, w, b, n_sample=n_sample, seed=seed)
    return u, w, b


def mirror_objects(shape: Shape, values: np.ndarray, biases: np.ndarray):
    """CslLibrary / ContributionTable mirror objects of a synthetic shape, for
    driving the public operator API (engine.search_topk_stream): R-group r of
    reaction t has id 1000*t + r, synthon ids are distinct and dense, table
    rows follow shape.pair_off (R-group-major, factorizer.py:87-106)."""
    from . import csl, engine

    reactions, rg_ids, rg_off = [], [], []
    members = np.zeros(shape.n_pairs, dtype=np.int64)
    sid = 0
    for t, (sizes, offs) in enumerate(zip(shape.sizes, shape.pair_off)):
        rgs = []
        for r, (n, o) in enumerate(zip(sizes, offs)):
            ids = tuple(range(sid, sid + int(n)))
            sid += int(n)
            rgs.append(csl.RgroupSpec(1000 * t + r, ids))
            rg_ids.append(1000 * t + r)
            rg_off.append(int(o))
            members[int(o):int(o) + int(n)] = ids
        reactions.append(csl.ReactionSpec(t, tuple(rgs)))
    lib = csl.CslLibrary(tuple(reactions), tuple(csl.SynthonRecord(i, f"s{i}") for i in range(sid)))
    order = np.argsort(rg_off)
    table = engine.ContributionTable(values=values, biases=np.asarray(biases, dtype=np.float64),
                                     task_names=list(TASKS), member_ids=members,
                                     rg_offsets=np.append(np.asarray(rg_off)[order], shape.n_pairs),
                                     rg_ids=np.asarray(rg_ids)[order], fingerprint=csl.library_fingerprint(lib))
    return lib, table


def query_spec(q: dict):
    """engine.QuerySpec mirror of a query dict (task names)."""
    from . import engine

    return engine.QuerySpec(q["objective"], q["direction"],
                            tuple(engine.Constraint(t, lo, hi) for t, lo, hi in q["constraints"]), q["k"])
