"""CPU-side checks of the drop-in boundary: the C-ABI library exists, loads,
and exports every symbol ``include/spmd_b200.h`` declares (no compute calls
without a GPU), and the ctypes binding covers exactly that set."""

import os
import re

import pytest

from paper_2105_04663_b200 import _capi as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            text = open(os.path.join(ROOT, "include", fn)).read()
            names |= set(re.findall(r"\b(spmd_[a-z0-9_]+)\s*\(", text))
    return names


def test_header_declares_entry_points():
    names = _declared()
    for n in ("spmd_dot", "spmd_all_gather", "spmd_local_all_to_all", "spmd_dynamic_slice",
              "spmd_collective_permute", "spmd_convolution", "spmd_reduce"):
        assert n in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(C.library_path()):
        from paper_2105_04663_b200.csrc import build as B  # noqa: F401
        pytest.skip("library not built")
    import ctypes
    lib = ctypes.CDLL(C.library_path())
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_matches_header():
    declared = _declared()
    bound = set(C.exported_symbols())
    # every declared function is bound; extra bound symbols are library extras
    assert declared <= bound, declared - bound


def test_library_loads_and_reports_version():
    if not os.path.exists(C.library_path()):
        pytest.skip("library not built")
    assert b"sm_100a" in C.lib().spmd_version()
    assert C.lib().spmd_status_string(4) == b"integer division by zero"
