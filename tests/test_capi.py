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


def test_host_bf16_rounding_matches_the_oracle():
    """upload_stacked ships bf16 bit patterns rounded on the host; they must
    equal the oracle's round-to-nearest-even (and the device conversion)."""
    import numpy as np
    from oracle import evaluator as O
    from paper_2105_04663_b200.executor import bf16_bits
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10.0 ** rng.integers(-30, 30, 10000),
                        np.array([0.0, -0.0, np.inf, -np.inf, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8,
                                  3.3895314e38], np.float32)]).astype(np.float32)
    got = (bf16_bits(x).astype(np.uint32) << 16).view(np.float32)
    np.testing.assert_array_equal(got, O.to_bf16(x))
    nan = (bf16_bits(np.array([np.nan], np.float32)).astype(np.uint32) << 16).view(np.float32)
    assert np.isnan(nan).all()
