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


def test_python_constants_match_header():
    """Every integer #define of include/dsinf.h that _capi mirrors (DSINF_<NAME> -> <NAME>) has the
    header's value, so the Python host API and a C caller agree on modes, dtypes and error codes."""
    import re

    from paper_2207_00032_b200 import _capi

    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "dsinf.h")).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"^#define DSINF_([A-Z0-9_]+) (\d+)", src, re.M)}
    checked = 0
    for name, value in defs.items():
        if hasattr(_capi, name):
            assert getattr(_capi, name) == value, name
            checked += 1
    assert checked >= 20 and "TP_SLICE" in defs
