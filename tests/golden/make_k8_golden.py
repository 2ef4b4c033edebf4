#!/usr/bin/env python3
"""Golden fixtures for the device encode_hierarchy (K8), generated FROM THE
REFERENCE ITSELF in the build container:

    python tests/golden/make_k8_golden.py

For seeded synthetic libraries (csl.generate_synthetic) and random-init
factorizers (factorizer.Factorizer, both modes "mlp" and "linear",
factorizer.py:109-132) it records the library (cslv1 text), every network's
parameters in param_groups order (factorizer.py:134-142), and the reference's
own encode_hierarchy output (factorizer.py:218-233): the hashed synthon
features (props.library_synthon_features, props.py:43-67), h_s, h_r, h_t and
the pair-row matrix u.  Written to tests/golden/k8_golden.npz (+ .json).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from apexcsl import csl, props  # noqa: E402
from apexcsl import factorizer as fz  # noqa: E402

OUT = Path(__file__).resolve().parent


def nets(f):
    """(name, MLP) in param_groups order."""
    return [("synthon", f.synthon_encoder), ("rg_phi", f.rgroup_encoder.phi), ("rg_rho", f.rgroup_encoder.rho),
            ("rx_phi", f.reaction_encoder.phi), ("rx_rho", f.reaction_encoder.rho), ("value", f.value_encoder),
            ("key", f.key_encoder)]


def main():
    arrays, cases = {}, []
    specs = [("k8_mlp", "mlp", csl.SyntheticConfig(n_reactions=4, components=(2, 3), synthons_per_rgroup=12), 7, 21),
             ("k8_linear", "linear", csl.SyntheticConfig(n_reactions=3, components=(3, 2), synthons_per_rgroup=9), 5, 8),
             ("k8_shared", "mlp", csl.SyntheticConfig(n_reactions=5, components=(2, 3, 2), synthons_per_rgroup=10,
                                                      share_rate=0.3), 13, 4)]
    for name, mode, cfg, lseed, fseed in specs:
        lib = csl.generate_synthetic(cfg, seed=lseed)
        f = fz.Factorizer(props.DEFAULT_FEATURE_DIM, fz.FactorizerDims(), np.random.default_rng(fseed), mode=mode)
        cache = fz.encode_hierarchy(f, lib)
        ctx = fz.build_context(lib, f.feature_config)
        shapes = []
        for nname, mlp in nets(f):
            shapes.append({"name": nname, "dims": list(mlp.dims)})
            for li, p in enumerate(mlp.params):
                arrays[f"{name}/{nname}/{li}"] = np.asarray(p, dtype=np.float64)
        for key, val in (("features", ctx.features), ("h_s", cache.h_s), ("h_r", cache.h_r), ("h_t", cache.h_t),
                         ("u", cache.u), ("member_ids", cache.member_ids), ("rg_offsets", cache.rg_offsets)):
            arrays[f"{name}/{key}"] = np.asarray(val)
        cases.append({"name": name, "mode": mode, "library": csl.serialize_library(lib), "nets": shapes,
                      "feature": {"p": f.feature_config.p, "seed": f.feature_config.seed},
                      "dims": {"d": f.dims.d, "d_u": f.dims.d_u}})
    (OUT / "k8_golden.json").write_text(json.dumps({"cases": cases}, indent=1))
    np.savez_compressed(OUT / "k8_golden.npz", **arrays)
    print(f"{len(cases)} cases")


if __name__ == "__main__":
    main()
