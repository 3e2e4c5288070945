"""Builds and runs tests/cpp/test_infersim_hpp.cpp: a C++ caller of the drop-in header
include/dsinf_infersim.hpp (reference names over the C ABI), linked against libdsinf.so.
The host-only calls run without a GPU; the `gpu` variant adds exec_reference on the device."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2207_00032_b200")
HAVE_CXX = shutil.which("g++") is not None or os.path.exists("/usr/bin/g++")


def _build(tmp_path):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    exe = tmp_path / "test_infersim_hpp"
    src = os.path.join(ROOT, "tests", "cpp", "test_infersim_hpp.cpp")
    r = subprocess.run([cxx, "-std=c++17", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"), src,
                        "-L", LIB, "-ldsinf", f"-Wl,-rpath,{LIB}", "-o", str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.mark.skipif(not HAVE_CXX, reason="no C++ compiler")
def test_cpp_dropin_header(tmp_path):
    exe = _build(tmp_path)
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr
    assert run.stdout.strip() == "ok"


@pytest.mark.gpu
@pytest.mark.skipif(not HAVE_CXX, reason="no C++ compiler")
def test_cpp_dropin_exec_reference_on_gpu(tmp_path):
    exe = _build(tmp_path)
    run = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, run.stdout + run.stderr
    assert run.stdout.strip() == "ok"
