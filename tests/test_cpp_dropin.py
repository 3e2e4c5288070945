"""Builds and runs tests/cpp/test_infersim_hpp.cpp: a C++ caller of the drop-in header
include/dsinf_infersim.hpp (reference names over the C ABI), linked against libdsinf.so.
Host-only calls, so it runs without a GPU."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2207_00032_b200")


@pytest.mark.skipif(shutil.which("g++") is None and not os.path.exists("/usr/bin/g++"), reason="no C++ compiler")
def test_cpp_dropin_header(tmp_path):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    exe = tmp_path / "test_infersim_hpp"
    src = os.path.join(ROOT, "tests", "cpp", "test_infersim_hpp.cpp")
    r = subprocess.run([cxx, "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), src,
                        "-L", LIB, "-ldsinf", f"-Wl,-rpath,{LIB}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert run.stdout.strip() == "ok"
