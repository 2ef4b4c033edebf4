#!/usr/bin/env python3
"""Generate the golden parity fixtures FROM THE REFERENCE ITSELF.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``apexcsl`` (reference ``pkg/src/apexcsl``) and records, for every
case, the inputs (library as canonical cslv1 text, contribution table arrays,
queries) and the reference's own outputs of ``engine.search_topk_stream``
(engine.py:265-313): every entry's global index, objective, violation,
constraint values, reaction id and synthon ids (floats as float.hex, exact),
``retained``, ``discarded_for_violation``, ``scanned`` and the result TSV
written by ``engine.save_result`` (engine.py:466-489).

Cases (reference test that each one restates):
  * exact_*   test_engine.py:9-13 (small_library seed 11, additive oracle seed 9,
              f32-rounded latents, perfect additive table) with QUERIES :116-126,
              ties :147-169, index_range :171-182, k=0 / k>N / infeasible :191-216,
              constraint values :224-231
  * accept_*  test_acceptance.py:74-118 criterion-1 libraries (seeds 200+li,
              random tables from default_rng(100), same draw order)
  * model_*   random-init APEX surrogate + factorizer -> encode_hierarchy ->
              precompute_contributions (factorizer.py:218-233, engine.py:80-92):
              u / heads / table for the precompute parity check, plus queries
  * preset_*  presets.py:11-34 bundles on a property-scaled table
The outputs are written to tests/golden/golden.json + golden.npz.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REF.parent / "tests"))

from apexcsl import csl, engine, props  # noqa: E402
from apexcsl import factorizer as fz  # noqa: E402
from apexcsl import surrogate as sg  # noqa: E402
from apexcsl.nn import MLP  # noqa: E402
from apexcsl.presets import PRESET_CONSTRAINTS  # noqa: E402

OUT = Path(__file__).resolve().parent

cases = []
arrays = {}


def table_arrays(name, table):
    arrays[f"{name}/values"] = np.asarray(table.values, dtype=np.float32)
    arrays[f"{name}/biases"] = np.asarray(table.biases, dtype=np.float64)
    arrays[f"{name}/rg_offsets"] = np.asarray(table.rg_offsets, dtype=np.int64)
    arrays[f"{name}/rg_ids"] = np.asarray(table.rg_ids, dtype=np.int64)
    arrays[f"{name}/member_ids"] = np.asarray(table.member_ids, dtype=np.int64)


def query_json(q, index_range=None):
    return {
        "objective": q.objective,
        "direction": q.direction,
        "constraints": [[c.task, float(c.lower).hex(), float(c.upper).hex()] for c in q.constraints],
        "k": q.k,
        "index_range": list(index_range) if index_range is not None else None,
    }


def run_case(name, library, table, queries, tmpdir, table_name=None):
    table_name = table_name or name
    if f"{table_name}/values" not in arrays:
        table_arrays(table_name, table)
    qs = []
    for qi, (q, rng_) in enumerate(queries):
        res = engine.search_topk_stream(library, table, q, index_range=rng_)
        path = tmpdir / f"{name}_{qi}.tsv"
        engine.save_result(res, q, path)
        qs.append({
            "query": query_json(q, rng_),
            "entries": [
                [e.global_index, float(e.objective).hex(), float(e.violation).hex(),
                 [float(v).hex() for v in e.constraint_values], e.chi.reaction_id, list(e.chi.synthon_ids())]
                for e in res.entries
            ],
            "retained": res.retained,
            "discarded": res.discarded_for_violation,
            "scanned": res.scanned,
            "tsv": path.read_text(),
        })
    cases.append({
        "name": name,
        "library": csl.serialize_library(library),
        "table": table_name,
        "task_names": list(table.task_names),
        "fingerprint": table.fingerprint,
        "queries": qs,
    })


def zero_table(library, n_tasks=1):
    member_ids, rg_offsets, rg_ids = [], [0], []
    for rg in library.iter_rgroups():
        rg_ids.append(rg.rgroup_id)
        member_ids.extend(rg.synthon_ids)
        rg_offsets.append(len(member_ids))
    return engine.ContributionTable(
        values=np.zeros((n_tasks, len(member_ids)), dtype=np.float32), biases=np.zeros(n_tasks),
        task_names=["obj"][:n_tasks], member_ids=np.asarray(member_ids), rg_offsets=np.asarray(rg_offsets),
        rg_ids=np.asarray(rg_ids), fingerprint=csl.library_fingerprint(library))


def random_table(library, task_names, rng, scale=None, shift=None):
    member_ids, rg_offsets, rg_ids = [], [0], []
    for rg in library.iter_rgroups():
        rg_ids.append(rg.rgroup_id)
        member_ids.extend(rg.synthon_ids)
        rg_offsets.append(len(member_ids))
    vals = rng.standard_normal((len(task_names), len(member_ids)))
    biases = rng.standard_normal(len(task_names))
    if scale is not None:
        vals = vals * np.asarray(scale)[:, None] + np.asarray(shift)[:, None]
    return engine.ContributionTable(
        values=vals.astype(np.float32), biases=biases, task_names=list(task_names),
        member_ids=np.asarray(member_ids), rg_offsets=np.asarray(rg_offsets), rg_ids=np.asarray(rg_ids),
        fingerprint=csl.library_fingerprint(library))


def main():
    import tempfile
    from conftest import f32_round_latents, perfect_additive_table

    tmp = Path(tempfile.mkdtemp())
    C, Q = engine.Constraint, engine.QuerySpec

    # --- exact_setup (test_engine.py) ---------------------------------------
    small = csl.generate_synthetic(csl.SyntheticConfig(n_reactions=2, components=(2, 3), synthons_per_rgroup=5),
                                   seed=11)
    oracle = f32_round_latents(props.make_additive_oracle(small, seed=9, task_names=["obj", "c1", "c2"]))
    exact = perfect_additive_table(oracle, small, ["obj", "c1", "c2"])
    total = csl.product_count(small)
    queries = [
        (Q("obj", "maximize", (), k=10), None),
        (Q("obj", "minimize", (), k=7), None),
        (Q("obj", "maximize", (C("c1", upper=0.5),), k=10), None),
        (Q("obj", "minimize", (C("c1", -0.5, 0.5), C("c2", lower=-1.0)), k=25), None),
        (Q("obj", "maximize", (), k=5), (40, 120)),
        (Q("obj", "maximize", (), k=0), None),
        (Q("obj", "maximize", (), k=total + 50), None),
        (Q("obj", "maximize", (C("c1", 1e6, 1e6 + 1),), k=8), None),
        (Q("obj", "maximize", (C("c1", upper=10.0),), k=3), None),
        (Q("obj", "maximize", (C("c1", upper=10.0),), k=4), None),
        (Q("c2", "minimize", (C("obj", lower=0.0), C("c1", -1.0, 1.0)), k=17), (3, 149)),
        (Q("obj", "maximize", (C("obj", upper=0.8),), k=12), (0, 75)),
    ]
    run_case("exact", small, exact, queries, tmp)
    zt = zero_table(small)
    run_case("ties", small, zt, [(Q("obj", "maximize", (), k=5), None), (Q("obj", "minimize", (), k=9), (17, 121))],
             tmp)

    # --- acceptance criterion 1 libraries (test_acceptance.py:74-118) --------
    rng = np.random.default_rng(100)
    configs = []
    for i in range(9):
        configs.append(csl.SyntheticConfig(n_reactions=2, components=(2, 3), synthons_per_rgroup=10 + i))
    for i in range(8):
        configs.append(csl.SyntheticConfig(n_reactions=4, components=(2, 3), synthons_per_rgroup=8 + i))
    configs.append(csl.SyntheticConfig(n_reactions=1, components=(3,), synthons_per_rgroup=22))
    configs.append(csl.SyntheticConfig(n_reactions=1, components=(3,), synthons_per_rgroup=50))
    configs.append(csl.SyntheticConfig(n_reactions=1, components=(3,), synthons_per_rgroup=100))
    for li, config in enumerate(configs):
        library = csl.generate_synthetic(config, seed=200 + li)
        total = csl.product_count(library)
        table = random_table(library, ["obj", "c1", "c2"], rng)
        direction = "maximize" if li % 2 == 0 else "minimize"
        constraints = ()
        if li % 3 != 0:
            constraints = (
                C("c1", upper=float(rng.normal(0, 1))),
                C("c2", float(rng.normal(-2, 0.5)), float(rng.normal(2, 0.5) + 5)),
            )
        k = [1, 10, 100, 500][li % 4]
        _ = int(rng.integers(1, max(2, total // 3)))  # keep the test's draw order (batched chunk size)
        qs = [(Q("obj", direction, constraints, k=k), None)]
        if total < 200_000:
            a, b = total // 7, total - total // 5
            qs.append((Q("obj", direction, constraints, k=k), (a, b)))
        run_case(f"accept_{li}", library, table, qs, tmp)

    # --- random-init APEX model pipeline ------------------------------------
    lib_m = csl.generate_synthetic(csl.SyntheticConfig(n_reactions=4, components=(2, 3), synthons_per_rgroup=14),
                                   seed=21)
    fcfg = props.FeatureConfig()
    mrng = np.random.default_rng(5)
    feat_dim = fcfg.p + fcfg.q
    tasks = props.DOCKING_TASKS + props.PROPERTY_TASKS
    enc = MLP([feat_dim, 128, 128, 64], mrng, bias=True)
    model = sg.SurrogateModel(encoder=enc, head_w=mrng.standard_normal((len(tasks), 64)) * 0.01,
                              head_b=np.zeros(len(tasks)), task_names=list(tasks), feature_config=fcfg)
    factor = fz.Factorizer(fcfg.p, fz.FactorizerDims(), mrng, mode="mlp", feature_config=fcfg)
    cache = fz.encode_hierarchy(factor, lib_m)
    table_m = engine.precompute_contributions(cache, model)
    arrays["model/u"] = np.asarray(cache.u, dtype=np.float64)
    arrays["model/head_w"] = np.asarray(model.head_w, dtype=np.float64)
    arrays["model/head_b"] = np.asarray(model.head_b, dtype=np.float64)
    arrays["model/cache_rg_offsets"] = np.asarray(cache.rg_offsets, dtype=np.int64)
    mv = table_m.values.astype(np.float64)
    q50 = {t: float(np.quantile(mv[i], 0.5)) * 2 for i, t in enumerate(tasks)}
    qs = [
        (Q("dock_a", "minimize", (C("mw", upper=q50["mw"]), C("logp", upper=q50["logp"])), k=100), None),
        (Q("dock_b", "maximize", (), k=50), None),
        (Q("dock_c", "minimize", (C("tpsa", q50["tpsa"] - 0.01, q50["tpsa"] + 0.01), C("hbd", upper=0.0)), k=30),
         None),
    ]
    run_case("model", lib_m, table_m, qs, tmp)

    # --- preset bundles on a property-scaled table (presets.py) --------------
    lib_p = csl.generate_synthetic(csl.SyntheticConfig(n_reactions=3, components=(2, 3), synthons_per_rgroup=20),
                                   seed=33)
    prng = np.random.default_rng(7)
    # per-R-group contributions such that 2-3 component sums land near RDKit ranges
    scale = [1.0] * 5 + [40.0, 0.8, 0.6, 1.1, 1.3, 15.0]
    shift = [-1.0] * 5 + [140.0, 1.0, 0.7, 2.0, 2.0, 30.0]
    table_p = random_table(lib_p, tasks, prng, scale=scale, shift=shift)
    qs = []
    for obj_i, preset in enumerate(["lipinski", "veber", "pfizer_3_75", "astex_ro3"]):
        qs.append((Q(tasks[obj_i], "minimize", PRESET_CONSTRAINTS[preset], k=1000), None))
    qs.append((Q("dock_e", "minimize", (C("mw", 300.0, 500.0), C("logp", -1.0, 5.0), C("tpsa", 20.0, 140.0),
                                         C("hbd", upper=5.0), C("hba", upper=10.0)), k=100), (1000, 8000)))
    run_case("preset", lib_p, table_p, qs, tmp)

    (OUT / "golden.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                                                 "reference": "apexcsl (pkg/src) read-only", "cases": cases}))
    np.savez_compressed(OUT / "golden.npz", **arrays)
    n_q = sum(len(c["queries"]) for c in cases)
    print(f"wrote {len(cases)} cases / {n_q} queries")


if __name__ == "__main__":
    main()
