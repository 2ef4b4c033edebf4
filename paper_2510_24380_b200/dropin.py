"""Select the B200 path inside the unmodified reference package.

    from paper_2510_24380_b200 import dropin
    dropin.install()          # apexcsl.engine / apexcsl.evalkit now call the B200 path
    # or run the reference CLI on the B200 path:
    python -m paper_2510_24380_b200.dropin search --library ... --table ... --query ... --out ...

install() rebinds the reference's operator API for this path (the three
search / precompute functions, load_table (memory-mapped) and
evalkit.oracle_topk (ground truth on the device)) — the names its
callers resolve at call time (cli.py:166, 180-183, 199-202 via
`engine.<name>`; evalkit.py:12-20 imports `search_topk_stream` by name, so
that module attribute is rebound too) — and makes the drop-in raise the
reference's own `EngineError` class, so `pytest.raises(engine.EngineError)`
and the CLI's error mapping (cli.py:357-366) behave unchanged.
"""

from __future__ import annotations

import sys

from . import engine as _b200

_SAVED: dict = {}


def install() -> None:
    import apexcsl.engine as ref_engine

    _b200._ERROR_CLASS[0] = ref_engine.EngineError
    def load_table(path):  # memory-mapped arrays, the reference's table class
        return _b200.load_table(path, mmap=True, cls=ref_engine.ContributionTable)

    targets = [(ref_engine, "search_topk_stream", _b200.search_topk_stream),
               (ref_engine, "search_topk_batched", _b200.search_topk_batched),
               (ref_engine, "precompute_contributions", _b200.precompute_contributions),
               (ref_engine, "load_table", load_table)]
    try:
        import apexcsl.evalkit as ref_evalkit

        from . import evalkit as _b200_eval
        targets.append((ref_evalkit, "search_topk_stream", _b200.search_topk_stream))
        # ground truth on the device, past the 1e8 enumeration guard (evalkit.py:23)
        targets.append((ref_evalkit, "oracle_topk", _b200_eval.oracle_topk))
    except ImportError:
        pass
    for mod, name, fn in targets:
        _SAVED.setdefault((mod.__name__, name), getattr(mod, name))
        setattr(mod, name, fn)


def uninstall() -> None:
    import importlib

    for (mod_name, name), fn in _SAVED.items():
        setattr(importlib.import_module(mod_name), name, fn)
    _SAVED.clear()
    _b200._ERROR_CLASS[0] = _b200.EngineError


def main(argv=None) -> int:
    install()
    from apexcsl import cli

    return cli.main(argv)


if __name__ == "__main__":
    sys.exit(main())
