"""The C++ drop-in header (include/trimatch_gpu.hpp): compiles against the
C-ABI on CPU; runs the SPEC.md examples + an RMAT graph on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

LIBDIR = os.path.join(ROOT, "paper_1909_02127_b200")
BIN = os.path.join(ROOT, "build", "test_dropin")


def _compile():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    cmd = [cxx, "-std=c++20", "-O1", "-Wall", "-Wextra", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-L", LIBDIR, "-ltcb200",
           f"-Wl,-rpath,{LIBDIR}", "-o", BIN]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return BIN


def test_dropin_header_compiles():
    assert os.path.exists(_compile())


@pytest.mark.gpu
def test_dropin_runs(oracle, cuda_ok):
    exe = _compile()
    scale = 12
    off, nb, E, _, _ = oracle.build_graph(oracle.gen_rmat(scale, 16), 1 << scale)
    T = oracle.count(off, nb)
    r = subprocess.run([exe, str(scale), str(T), str(E)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr
