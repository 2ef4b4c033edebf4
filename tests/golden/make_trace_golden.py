#!/usr/bin/env python3
"""Golden BatchTrace fixtures FROM THE REFERENCE ITSELF (build container):

    python tests/golden/make_trace_golden.py

For the golden cases of tests/golden/golden.json (libraries + tables recorded
by make_golden.py) it runs the reference's search_topk_batched
(engine.py:345-398) with a BatchTrace (engine.py:338-342) for several chunk
sizes, k and constraint sets — including infeasible-heavy queries, where the
chain's selections hold violating products — and records the trace lists.
Written to tests/golden/trace_golden.json.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from apexcsl import csl, engine  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    doc = json.loads((OUT / "golden.json").read_text())
    arrays = dict(np.load(OUT / "golden.npz"))
    recs = []
    for case in doc["cases"][:6]:
        lib = csl.deserialize_library(case["library"])
        t = case["table"]
        table = engine.ContributionTable(values=arrays[f"{t}/values"], biases=arrays[f"{t}/biases"],
                                         task_names=list(case["task_names"]), member_ids=arrays[f"{t}/member_ids"],
                                         rg_offsets=arrays[f"{t}/rg_offsets"], rg_ids=arrays[f"{t}/rg_ids"],
                                         fingerprint=case["fingerprint"])
        names = list(case["task_names"])
        total = csl.product_count(lib)
        v = np.asarray(table.values, dtype=np.float64)
        qs = [engine.QuerySpec(names[0], "maximize", (), 6),
              engine.QuerySpec(names[0], "minimize", (), 50)]
        if len(names) > 1:
            mid = float(np.median(v[1]))
            qs.append(engine.QuerySpec(names[0], "maximize", (engine.Constraint(names[1], upper=mid),), 25))
            # nearly infeasible: the chain's selections hold violating products
            qs.append(engine.QuerySpec(names[-1], "minimize",
                                       (engine.Constraint(names[1], mid, mid + 1e-9),), 40))
        for qi, q in enumerate(qs):
            for chunk in (1, 7, 20, 64, 10**6):
                for rng in (None, (total // 5, total - total // 9)):
                    trace = engine.BatchTrace([], [], [])
                    engine.search_topk_batched(lib, table, q, chunk, index_range=rng, trace=trace)
                    recs.append({"case": case["name"], "query": qi, "objective": q.objective,
                                 "direction": q.direction,
                                 "constraints": [[c.task, float(c.lower).hex(), float(c.upper).hex()]
                                                 for c in q.constraints],
                                 "k": q.k, "chunk": chunk, "index_range": list(rng) if rng else None,
                                 "batch_sizes": trace.batch_sizes, "new": trace.new_elements,
                                 "carried": trace.carried_elements})
    (OUT / "trace_golden.json").write_text(json.dumps({"traces": recs}))
    print(len(recs), "traces")


if __name__ == "__main__":
    main()
