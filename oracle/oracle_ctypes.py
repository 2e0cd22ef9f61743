"""ctypes bindings for the test-only checkers built by oracle/Makefile.

TEST INFRASTRUCTURE ONLY.  Importable from tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs; the product package
(paper_1909_02127_b200) never imports this module.

  Oracle  -- oracle/liboracle.so: the C restatement (oracle.c)
  Ref     -- oracle/_ref/libtrimatch_ref.so: the reference's own sources +
             ref_shim.cpp (every call goes through trimatch's public API)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtrimatch_ref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """Compile oracle/ (and oracle/_ref when /root/reference is present)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class Oracle:
    """The C restatement of the reference path (oracle/oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.oracle_rmat_num_edges.restype = C.c_uint64
        L.oracle_rmat_num_edges.argtypes = [C.c_int, C.c_int]
        L.oracle_er_num_edges.restype = C.c_uint64
        L.oracle_er_num_edges.argtypes = [C.c_int, C.c_int]
        L.oracle_gen_rmat.argtypes = [C.c_int, C.c_int, C.c_int, u32p]
        L.oracle_gen_er.argtypes = [C.c_int, C.c_int, u32p]
        L.oracle_build_graph.restype = C.c_int
        L.oracle_build_graph.argtypes = [u32p, C.c_uint64, C.c_uint32, C.POINTER(u64p),
                                         C.POINTER(u32p), u64p, u64p, u64p]
        L.oracle_free.argtypes = [C.c_void_p]
        L.oracle_count.restype = C.c_uint64
        L.oracle_count.argtypes = [u64p, u32p, C.c_uint32, u64p, C.c_int]
        L.oracle_count_dag.restype = C.c_uint64
        L.oracle_count_dag.argtypes = [u64p, u32p, C.c_uint32, u64p, C.c_int]
        L.oracle_brute_force.restype = C.c_uint64
        L.oracle_brute_force.argtypes = [u64p, u32p, C.c_uint32]
        L.oracle_fnv1a64.restype = C.c_uint64
        L.oracle_fnv1a64.argtypes = [C.c_void_p, C.c_uint64]
        L.oracle_dag_stats.argtypes = [u64p, u32p, C.c_uint32, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double), u32p]
        L.oracle_seed_costs.argtypes = [u64p, u32p, C.c_uint32, C.POINTER(C.c_double)]

    def seed_costs(self, offsets: np.ndarray, nbrs: np.ndarray) -> np.ndarray:
        n = offsets.size - 1
        out = np.zeros(max(n, 1), dtype=np.float64)
        nb = nbrs if nbrs.size else np.zeros(1, np.uint32)
        self.lib.oracle_seed_costs(_ptr(offsets, u64p), _ptr(nb, u32p), n, _ptr(out, C.POINTER(C.c_double)))
        return out[:n]

    # generators ---------------------------------------------------------
    def gen_rmat(self, scale: int, edgefactor: int = 16, permute: bool = False) -> np.ndarray:
        m = self.lib.oracle_rmat_num_edges(scale, edgefactor)
        pairs = np.empty(2 * m, dtype=np.uint32)
        self.lib.oracle_gen_rmat(scale, edgefactor, int(permute), _ptr(pairs, u32p))
        return pairs

    def gen_er(self, scale: int, avg_degree: int = 32) -> np.ndarray:
        m = self.lib.oracle_er_num_edges(scale, avg_degree)
        pairs = np.empty(2 * m, dtype=np.uint32)
        self.lib.oracle_gen_er(scale, avg_degree, _ptr(pairs, u32p))
        return pairs

    # build_graph ----------------------------------------------------------
    def build_graph(self, pairs: np.ndarray, n: int):
        """Returns (offsets u64[n+1], nbrs u32[2E], E, loops, dups); raises
        ValueError like the reference's std::invalid_argument."""
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        off = u64p()
        nb = u32p()
        E = C.c_uint64()
        lo = C.c_uint64()
        du = C.c_uint64()
        rc = self.lib.oracle_build_graph(_ptr(pairs, u32p), pairs.size // 2, n, C.byref(off),
                                         C.byref(nb), C.byref(E), C.byref(lo), C.byref(du))
        if rc != 0:
            raise ValueError("build_graph: vertex id out of declared range")
        offsets = np.ctypeslib.as_array(off, shape=(n + 1,)).copy()
        nbrs = np.ctypeslib.as_array(nb, shape=(max(2 * E.value, 1),))[: 2 * E.value].copy()
        self.lib.oracle_free(off)
        self.lib.oracle_free(nb)
        return offsets, nbrs, E.value, lo.value, du.value

    # counting ----------------------------------------------------------------
    def count(self, offsets: np.ndarray, nbrs: np.ndarray, per_vertex: bool = False, threads: int = 0):
        n = offsets.size - 1
        pv = np.zeros(n, dtype=np.uint64) if per_vertex else None
        nb = nbrs if nbrs.size else np.zeros(1, np.uint32)
        t = self.lib.oracle_count(_ptr(offsets, u64p), _ptr(nb, u32p), n,
                                  _ptr(pv, u64p) if per_vertex else None, threads)
        return (t, pv) if per_vertex else t

    def count_dag(self, offsets: np.ndarray, nbrs: np.ndarray, per_vertex: bool = False, threads: int = 0):
        """The degree-ordered pivot-join checker (oracle_count_dag)."""
        n = offsets.size - 1
        pv = np.zeros(n, dtype=np.uint64) if per_vertex else None
        nb = nbrs if nbrs.size else np.zeros(1, np.uint32)
        t = self.lib.oracle_count_dag(_ptr(offsets, u64p), _ptr(nb, u32p), n,
                                      _ptr(pv, u64p) if per_vertex else None, threads)
        return (t, pv) if per_vertex else t

    def brute_force(self, offsets: np.ndarray, nbrs: np.ndarray) -> int:
        nb = nbrs if nbrs.size else np.zeros(1, np.uint32)
        r = self.lib.oracle_brute_force(_ptr(offsets, u64p), _ptr(nb, u32p), offsets.size - 1)
        if r == 2**64 - 1:
            raise ValueError("brute force size guard (n <= 5000)")
        return r

    def fnv(self, a: np.ndarray) -> str:
        a = np.ascontiguousarray(a)
        return "%016x" % self.lib.oracle_fnv1a64(a.ctypes.data, a.nbytes)

    def dag_stats(self, offsets: np.ndarray, nbrs: np.ndarray):
        W, S2, J = C.c_double(), C.c_double(), C.c_double()
        mx = C.c_uint32()
        nb = nbrs if nbrs.size else np.zeros(1, np.uint32)
        self.lib.oracle_dag_stats(_ptr(offsets, u64p), _ptr(nb, u32p), offsets.size - 1,
                                  C.byref(W), C.byref(S2), C.byref(J), C.byref(mx))
        return dict(W=W.value, S2=S2.value, J=J.value, max_dplus=mx.value)


class RefError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class Ref:
    """The reference library itself (oracle/_ref/libtrimatch_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_build_graph.restype = C.c_int
        L.ref_build_graph.argtypes = [u32p, C.c_uint64, C.c_uint32, C.POINTER(u64p), C.POINTER(u32p),
                                      u64p, u64p, u64p]
        L.ref_graph_new.restype = C.c_void_p
        L.ref_graph_new.argtypes = [u64p, u32p, C.c_uint32, C.c_uint64]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_count_triangles.restype = C.c_int
        L.ref_count_triangles.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, u64p, u64p,
                                          C.POINTER(C.c_double)]
        L.ref_segmented_intersect.restype = C.c_int
        L.ref_segmented_intersect.argtypes = [C.c_void_p, C.c_int, u64p]
        L.ref_segmented_intersect_pv.restype = C.c_int
        L.ref_segmented_intersect_pv.argtypes = [C.c_void_p, C.c_int, u64p, u64p]
        L.ref_count_sample.restype = C.c_int
        L.ref_count_sample.argtypes = [C.c_void_p, u32p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                       C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       u64p, u64p, u64p]
        L.ref_parse_matrix_market.restype = C.c_int
        L.ref_parse_matrix_market.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(u32p), u64p, u32p]
        L.ref_load_graph.restype = C.c_int
        L.ref_load_graph.argtypes = [C.c_char_p, C.POINTER(u64p), C.POINTER(u32p), u32p, u64p, u64p, u64p]
        L.ref_write_csr_cache.restype = C.c_int
        L.ref_write_csr_cache.argtypes = [C.c_char_p, C.c_void_p]

    def _check(self, rc: int):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def build_graph(self, pairs: np.ndarray, n: int):
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
        off, nb = u64p(), u32p()
        E, lo, du = C.c_uint64(), C.c_uint64(), C.c_uint64()
        p = pairs if pairs.size else np.zeros(2, np.uint32)
        self._check(self.lib.ref_build_graph(_ptr(p, u32p), pairs.size // 2, n, C.byref(off),
                                             C.byref(nb), C.byref(E), C.byref(lo), C.byref(du)))
        offsets = np.ctypeslib.as_array(off, shape=(n + 1,)).copy()
        nbrs = np.ctypeslib.as_array(nb, shape=(max(2 * E.value, 1),))[: 2 * E.value].copy()
        self.lib.ref_free(off)
        self.lib.ref_free(nb)
        return offsets, nbrs, E.value, lo.value, du.value

    def graph(self, offsets: np.ndarray, nbrs: np.ndarray) -> "RefGraph":
        return RefGraph(self, offsets, nbrs)

    def parse_matrix_market(self, text: bytes):
        pairs, m, n = u32p(), C.c_uint64(), C.c_uint32()
        self._check(self.lib.ref_parse_matrix_market(text, len(text), C.byref(pairs), C.byref(m), C.byref(n)))
        arr = np.ctypeslib.as_array(pairs, shape=(2 * m.value + 2,))[: 2 * m.value].copy()
        self.lib.ref_free(pairs)
        return arr, n.value

    def load_graph(self, path: str):
        off, nb = u64p(), u32p()
        n, E, lo, du = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self.lib.ref_load_graph(path.encode(), C.byref(off), C.byref(nb), C.byref(n),
                                            C.byref(E), C.byref(lo), C.byref(du)))
        offsets = np.ctypeslib.as_array(off, shape=(n.value + 1,)).copy()
        nbrs = np.ctypeslib.as_array(nb, shape=(max(2 * E.value, 1),))[: 2 * E.value].copy()
        self.lib.ref_free(off)
        self.lib.ref_free(nb)
        return offsets, nbrs, E.value, lo.value, du.value


class RefGraph:
    def __init__(self, ref: Ref, offsets: np.ndarray, nbrs: np.ndarray):
        self.ref = ref
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.nbrs = np.ascontiguousarray(nbrs, dtype=np.uint32)
        self.n = self.offsets.size - 1
        self.E = int(self.offsets[-1]) // 2
        nb = self.nbrs if self.nbrs.size else np.zeros(1, np.uint32)
        self.h = ref.lib.ref_graph_new(_ptr(self.offsets, u64p), _ptr(nb, u32p), self.n, self.E)
        if not self.h:
            raise RefError(1, ref.lib.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_graph_free(self.h)
            self.h = None

    def count_triangles(self, lookahead: int = 2, workers: int = 0, per_vertex: bool = False):
        c = C.c_uint64()
        ms = C.c_double()
        pv = np.zeros(self.n, dtype=np.uint64) if per_vertex else None
        self.ref._check(self.ref.lib.ref_count_triangles(self.h, lookahead, workers, 0, C.byref(c),
                                                         _ptr(pv, u64p) if per_vertex else None,
                                                         C.byref(ms)))
        return (c.value, pv) if per_vertex else c.value

    def segmented_intersect(self, workers: int = 0, per_vertex: bool = False):
        c = C.c_uint64()
        if per_vertex:
            pv = np.zeros(self.n, dtype=np.uint64)
            self.ref._check(self.ref.lib.ref_segmented_intersect_pv(self.h, workers, C.byref(c),
                                                                    _ptr(pv, u64p)))
            return c.value, pv
        self.ref._check(self.ref.lib.ref_segmented_intersect(self.h, workers, C.byref(c)))
        return c.value

    def count_sample(self, seeds: np.ndarray, row_stride: int = 1, max_chunk_visits: int = 1 << 27,
                     lookahead: int = 2, workers: int = 0):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint32)
        fm, l1, l2 = C.c_double(), C.c_double(), C.c_double()
        cnt, vis, rows = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.ref._check(self.ref.lib.ref_count_sample(self.h, _ptr(seeds, u32p), seeds.size, row_stride,
                                                      max_chunk_visits, lookahead, workers, C.byref(fm),
                                                      C.byref(l1), C.byref(l2), C.byref(cnt), C.byref(vis),
                                                      C.byref(rows)))
        return dict(filter_ms=fm.value, l1_ms=l1.value, l2_ms=l2.value, count=cnt.value, visits=vis.value,
                    l1_rows=rows.value)

    def write_csr_cache(self, path: str):
        self.ref._check(self.ref.lib.ref_write_csr_cache(path.encode(), self.h))
