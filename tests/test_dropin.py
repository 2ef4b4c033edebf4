"""CPU: dropin.install() rebinds the reference operator API and maps errors to
the reference's EngineError (validation happens before any device call)."""

import pytest

from conftest import golden_cases, import_reference


def test_install_rebinds_reference_api():
    rcsl, rengine = import_reference()
    import apexcsl.evalkit as revalkit

    from paper_2510_24380_b200 import dropin, engine

    dropin.install()
    try:
        assert rengine.search_topk_stream is engine.search_topk_stream
        assert rengine.search_topk_batched is engine.search_topk_batched
        assert rengine.precompute_contributions is engine.precompute_contributions
        assert revalkit.search_topk_stream is engine.search_topk_stream
        case = golden_cases()[0]
        lib = rcsl.deserialize_library(case.library_text)
        table = rengine.ContributionTable(values=case.values, biases=case.biases, task_names=list(case.task_names),
                                          member_ids=case.member_ids, rg_offsets=case.rg_offsets,
                                          rg_ids=case.rg_ids, fingerprint=case.fingerprint)
        with pytest.raises(rengine.EngineError, match="unknown task"):
            rengine.search_topk_stream(lib, table, rengine.QuerySpec("nope", "maximize", k=3))
        with pytest.raises(rengine.EngineError, match="index range"):
            rengine.search_topk_stream(lib, table, rengine.QuerySpec("obj", "maximize", k=3), index_range=(9, 2))
        with pytest.raises(rengine.EngineError, match="chunk size"):
            rengine.search_topk_batched(lib, table, rengine.QuerySpec("obj", "maximize", k=3), 0)
    finally:
        dropin.uninstall()
    assert rengine.search_topk_stream is not engine.search_topk_stream
