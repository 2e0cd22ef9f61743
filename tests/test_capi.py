"""CPU: the C-ABI library loads, exports every symbol include/tcb200.h declares,
and its host-only entry points (MatrixMarket / TRIMCSR1 parsing, argument
validation) behave like the reference's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tcb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols(tc):
    lib = C.CDLL(tc.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(tc.EXPORTED_SYMBOLS)
    assert tc.abi_version() == 3


def test_sm100a_only_binary(tc):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tc.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_no_link_time_nccl(tc):
    """NCCL is bound at the first multi-GPU call (multi.cu dlopen), not at
    link time: loading libtcb200.so before torch must not pin the system
    libnccl.so.2 under the soname torch's own NCCL uses (that made
    `import torch` fail with an undefined ncclDevCommCreate)."""
    import subprocess
    import sys
    out = subprocess.run(["readelf", "-d", tc.LIB_PATH], capture_output=True, text=True)
    if out.returncode == 0:
        assert "libnccl" not in out.stdout
    code = ("import ctypes, sys; ctypes.CDLL(sys.argv[1]); import torch, torch.distributed; "
            "print('torch ok', torch.__version__)")
    r = subprocess.run([sys.executable, "-c", code, tc.LIB_PATH], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "torch ok" in r.stdout, r.stderr[-2000:]


MM_CASES = [
    b"%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 2\n1 3\n2 3\n",
    b"%%MatrixMarket matrix coordinate real general\n% comment\n\n2 2 1\n1 1 0.5\n",
    b"%%matrixmarket MATRIX Coordinate\n4 3 2\n4 1\n2 3 7 8\n% trailing\n\n",
    b"%%MatrixMarket matrix coordinate\n3 3 2\n1 2\r\n2 3\r\n",
    b"",
    b"%%MatrixMarket matrix array real\n3 3 1\n1 1\n",
    b"%%MatrixMarket matrix coordinate\n",
    b"%%MatrixMarket matrix coordinate\n3 3\n",
    b"%%MatrixMarket matrix coordinate\n3 3 x\n",
    b"%%MatrixMarket matrix coordinate\n3 3 2\n1 2\n",
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1 4\n",
    b"%%MatrixMarket matrix coordinate\n3 3 1\n0 1\n",
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1\n",
    b"%%MatrixMarket matrix coordinate\n3 3 1\n1 2\n3 1\n",
    b"%%MatrixMarket matrix coordinate\n3 3 1\n-1 2\n",
    b"%%MatrixMarket matrix coordinate\n4294967296 1 0\n",
    b"%%MatrixMarket matrix coordinate\n4294967295 1 1\n4294967295 1\n",
]


@pytest.mark.parametrize("i", range(len(MM_CASES)))
def test_matrix_market_parity(tc, ref, i):
    text = MM_CASES[i]
    try:
        exp_pairs, exp_n = ref.parse_matrix_market(text)
        exp_err = None
    except Exception as e:  # RefError
        exp_err = e.msg
    if exp_err is None:
        el = tc.parse_matrix_market(text)
        assert el.num_vertices_declared == exp_n
        assert np.array_equal(el.pairs().reshape(-1), exp_pairs)
    else:
        with pytest.raises(tc.ParseError) as ei:
            tc.parse_matrix_market(text)
        assert str(ei.value) == exp_err


def test_matrix_market_error_line(tc):
    with pytest.raises(tc.ParseError) as ei:
        tc.parse_matrix_market(b"%%MatrixMarket matrix coordinate\n% c\n3 3 1\n\n1 9\n")
    assert ei.value.line == 5


def test_csr_cache_rejects_corruption(tc):
    with pytest.raises(tc.ParseError):
        tc._check(tc._lib.tc_csr_cache_to_graph(b"NOTMAGIC" + b"\0" * 40, 48, 0, C.byref(C.c_void_p())))
    # header checks run on the host (the offsets/adjacency invariants on the
    # device: test_gpu_parity::test_csr_cache_corruption)
    hdr = b"TRIMCSR1" + np.array([1, 2, 1], "<u8").tobytes()
    with pytest.raises(tc.ParseError) as ei:
        tc._check(tc._lib.tc_csr_cache_to_graph(hdr + b"\0" * 8, len(hdr) + 8, 0, C.byref(C.c_void_p())))
    assert "truncated CSR cache" in str(ei.value)
    bad_ver = b"TRIMCSR1" + np.array([2, 2, 1], "<u8").tobytes() + b"\0" * 32
    with pytest.raises(tc.ParseError) as ei:
        tc._check(tc._lib.tc_csr_cache_to_graph(bad_ver, len(bad_ver), 0, C.byref(C.c_void_p())))
    assert "unsupported CSR cache version" in str(ei.value)
    with pytest.raises(tc.ParseError) as ei:
        tc._check(tc._lib.tc_csr_cache_to_graph(hdr[:20], 20, 0, C.byref(C.c_void_p())))


def test_count_rejects_bad_options_before_device_work(tc):
    o = tc.TcCountOpts(3, 0, 0, 1, 1)
    total = np.zeros(1, np.uint64)
    rc = tc._lib.tc_count(C.c_void_p(1), C.byref(o), C.c_void_p(total.ctypes.data), None, None)
    assert rc == tc.TC_EINVAL and b"lookahead" in tc._lib.tc_last_error()
    o = tc.TcCountOpts(2, 1, 0, 1, 1)
    rc = tc._lib.tc_count(C.c_void_p(1), C.byref(o), C.c_void_p(total.ctypes.data), None, None)
    assert rc == tc.TC_EUNSUPPORTED
    rc = tc._lib.tc_count(None, None, None, None, None)
    assert rc == tc.TC_EINVAL


def test_generator_counts(tc, oracle):
    assert tc.gen_num_edges(tc.GEN_RMAT, 24, 16) == 1 << 28
    assert tc.gen_num_edges(tc.GEN_ER, 20, 32) == 1 << 24
    assert tc.gen_num_edges(tc.GEN_KRON, 26, 32) == 1 << 31
