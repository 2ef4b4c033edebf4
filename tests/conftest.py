import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
REFERENCE_SRC = Path("/root/reference/pkg/src")
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def have_reference() -> bool:
    return (REFERENCE_SRC / "apexcsl" / "engine.py").exists()


def import_reference():
    """The read-only reference package (only present in the build container)."""
    if not have_reference():
        pytest.skip("reference package not present on this machine")
    if str(REFERENCE_SRC) not in sys.path:
        sys.path.insert(0, str(REFERENCE_SRC))
    import apexcsl.csl as rcsl
    import apexcsl.engine as rengine

    return rcsl, rengine


def unhex(x):
    return float.fromhex(x)


class GoldenCase:
    """One golden case: library text, table arrays, per-query expected output
    recorded from the reference (tests/golden/make_golden.py)."""

    def __init__(self, d, arrays):
        self.name = d["name"]
        self.library_text = d["library"]
        self.task_names = d["task_names"]
        self.fingerprint = d["fingerprint"]
        t = d["table"]
        self.values = arrays[f"{t}/values"]
        self.biases = arrays[f"{t}/biases"]
        self.rg_offsets = arrays[f"{t}/rg_offsets"]
        self.rg_ids = arrays[f"{t}/rg_ids"]
        self.member_ids = arrays[f"{t}/member_ids"]
        self.queries = d["queries"]

    def library(self):
        from paper_2510_24380_b200 import csl

        return csl.deserialize_library(self.library_text)

    def table(self):
        from paper_2510_24380_b200 import engine

        return engine.ContributionTable(values=self.values, biases=self.biases, task_names=list(self.task_names),
                                        member_ids=self.member_ids, rg_offsets=self.rg_offsets, rg_ids=self.rg_ids,
                                        fingerprint=self.fingerprint)

    def lib_arrays(self):
        from oracle import scan_oracle as orc

        return orc.lib_from_reference(self.library(), self.table())

    def task(self, name):
        return self.task_names.index(name)

    def oracle_query(self, qd):
        from oracle import scan_oracle as orc

        q = qd["query"]
        cons = [(self.task(t), unhex(lo), unhex(hi)) for t, lo, hi in q["constraints"]]
        return orc.Query(obj=self.task(q["objective"]), maximize=q["direction"] == "maximize", cons=cons, k=q["k"])

    def mirror_query(self, qd):
        from paper_2510_24380_b200 import engine

        q = qd["query"]
        cons = tuple(engine.Constraint(t, unhex(lo), unhex(hi)) for t, lo, hi in q["constraints"])
        return engine.QuerySpec(q["objective"], q["direction"], cons, q["k"])


_GOLDEN_CACHE = {}


def golden_cases():
    if "cases" not in _GOLDEN_CACHE:
        doc = json.loads((GOLDEN / "golden.json").read_text())
        arrays = dict(np.load(GOLDEN / "golden.npz"))
        _GOLDEN_CACHE["cases"] = [GoldenCase(d, arrays) for d in doc["cases"]]
        _GOLDEN_CACHE["arrays"] = arrays
    return _GOLDEN_CACHE["cases"]


def golden_arrays():
    golden_cases()
    return _GOLDEN_CACHE["arrays"]


def golden_query_ids():
    return [(ci, qi) for ci, c in enumerate(golden_cases()) for qi in range(len(c.queries))]
