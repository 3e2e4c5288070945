"""The C-ABI library loads (without a GPU) and exports every entry point include/dsinf.h declares."""
import ctypes as C
import os
import re

from paper_2207_00032_b200 import _capi as capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "dsinf.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dsinf_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 40
    lib = C.CDLL(capi.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_the_header():
    assert set(declared_functions()) == set(capi.SIGNATURES)


def test_errors_map_to_reference_exceptions():
    from paper_2207_00032_b200 import infersim as I

    try:
        I.derive_schedule(I.GemmShape(0, 4, 1, 2), I.b200_device())
    except I.ConfigError as e:
        assert "gemm shape dims must be positive" in str(e)  # gemm.hpp:36-37 message
    else:
        raise AssertionError("ConfigError expected")
    assert capi.lib.dsinf_version().decode().startswith("dsinf-b200")
