"""CPU: the C-ABI library is built for sm_100a, loads, and exports every
symbol include/apex_b200.h declares.  No compute calls without a GPU."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "apex_b200.h"
LIB = ROOT / "paper_2510_24380_b200" / "libapexb200.so"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(apex_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("apex_ctx_create", "apex_load_library", "apex_load_table", "apex_load_cache", "apex_query",
                 "apex_query_local", "apex_merge_finalize", "apex_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not LIB.exists():
        import __graft_entry__ as g
        g.build()
    from paper_2510_24380_b200 import _native
    lib = _native.load_library()
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(apex_\w+)", out))
    for name in declared():
        assert name in exported, name
        assert hasattr(lib, name)
    assert set(_native.EXPORTED) <= exported
    assert b"sm_100a" in lib.apex_version()


def test_kernels_are_sm100a_cubins():
    out = subprocess.run(["cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_24380_b200 import _native
    with pytest.raises(_native.NativeError) as exc:
        _native.DeviceContext(0)
    assert exc.value.code == _native.APEX_ECUDA
    assert "no CPU fallback" in str(exc.value)
