#!/usr/bin/env python3
"""Golden fixtures for the GPU ground-truth evaluation (evalkit.oracle_topk),
generated FROM THE REFERENCE ITSELF in the build container:

    python tests/golden/make_gt_golden.py

For seeded synthetic libraries (csl.generate_synthetic, csl.py:268-309) and
the reference's default oracle (props.make_default_oracle, props.py:311-346:
five docking tasks additive+nonlinear+pairwise, six additive property tasks)
it records the library (cslv1 text), the oracle (latents, parameters, seed)
and the reference's own evalkit.oracle_topk output (evalkit.py:49-90) for
queries with and without oracle constraints, both directions, index ranges
and j past the feasible count: global indices and objectives (float.hex).
Written to tests/golden/gt_golden.json + gt_golden.npz.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from apexcsl import csl, engine, evalkit, props  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    cases, arrays = [], {}
    specs = [("gt_small", csl.SyntheticConfig(n_reactions=2, components=(2, 3), synthons_per_rgroup=5), 11, 3),
             ("gt_medium", csl.SyntheticConfig(n_reactions=4, components=(2, 3), synthons_per_rgroup=12), 7, 5),
             ("gt_wide", csl.SyntheticConfig(n_reactions=5, components=(3, 2, 2), synthons_per_rgroup=20), 23, 9)]
    for name, cfg, lseed, oseed in specs:
        lib = csl.generate_synthetic(cfg, seed=lseed)
        oracle = props.make_default_oracle(lib, seed=oseed)
        total = csl.product_count(lib)
        for i, t in enumerate(oracle.tasks):
            arrays[f"{name}/latent/{i}"] = np.asarray(t.latent, dtype=np.float64)
        qs = [
            (engine.QuerySpec("dock_a", "minimize", (), 10), None),
            (engine.QuerySpec("dock_b", "maximize", (), 25), None),
            (engine.QuerySpec("dock_c", "minimize", (engine.Constraint("mw", upper=0.0),), 15), None),
            (engine.QuerySpec("dock_d", "maximize", (engine.Constraint("logp", -0.5, 0.5),
                                                     engine.Constraint("tpsa", lower=-0.2)), 20), None),
            (engine.QuerySpec("mw", "maximize", (engine.Constraint("hbd", upper=0.3),), 12), None),
            (engine.QuerySpec("dock_e", "minimize", (), 7), (total // 5, total - total // 7)),
            (engine.QuerySpec("dock_a", "maximize", (engine.Constraint("hba", -0.01, 0.01),), 5000), None),
        ]
        qrecs = []
        for q, rng in qs:
            top = evalkit.oracle_topk(lib, oracle, q, q.k, index_range=rng)
            qrecs.append({
                "objective": q.objective, "direction": q.direction,
                "constraints": [(c.task, float(c.lower).hex(), float(c.upper).hex()) for c in q.constraints],
                "j": q.k, "index_range": list(rng) if rng else None,
                "g": [e.global_index for e in top.entries],
                "objective_values": [float(e.objective).hex() for e in top.entries],
                "chi": [[e.chi.reaction_id, list(e.chi.synthon_ids())] for e in top.entries],
            })
        cases.append({
            "name": name, "library": csl.serialize_library(lib), "seed": oracle.seed,
            "tasks": [{"name": t.name, "mode": t.mode, "nonlinear_scale": float(t.nonlinear_scale).hex(),
                       "nonlinear_alpha": float(t.nonlinear_alpha).hex(), "pair_scale": float(t.pair_scale).hex(),
                       "pair_density": float(t.pair_density).hex()} for t in oracle.tasks],
            "queries": qrecs,
        })
    (OUT / "gt_golden.json").write_text(json.dumps({"cases": cases}, indent=1))
    np.savez_compressed(OUT / "gt_golden.npz", **arrays)
    print(f"{len(cases)} cases, {sum(len(c['queries']) for c in cases)} queries")


if __name__ == "__main__":
    main()
