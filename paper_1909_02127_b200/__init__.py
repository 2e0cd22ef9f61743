"""paper_1909_02127_b200 -- B200-native BFS-based triangle counting.

Host-side mirror of the reference's operator interface (namespace trimatch,
/root/reference/proj) over the C-ABI of libtcb200.so (include/tcb200.h):

  reference (C++)                         here
  --------------------------------------  -----------------------------------
  EdgeList            graph.hpp:16-19     EdgeList
  BuildReport         graph.hpp:22-25     BuildReport
  Graph               graph.hpp:35-66     Graph  (device-resident handle)
  build_graph         graph.hpp:73        build_graph
  degrees             graph.hpp:75        degrees
  parse_matrix_market io.hpp:34-35        parse_matrix_market[_file]
  read/write_csr_cache io.hpp:39-41       read_csr_cache / write_csr_cache
  load_graph          io.hpp:45           load_graph
  MatchOptions        matcher.hpp:84-88   MatchOptions
  MatchResult         matcher.hpp:90-94   MatchResult (+ per_vertex)
  count_triangles     matcher.hpp:128     count_triangles

Exceptions follow the reference: std::invalid_argument -> InvalidArgument
(a ValueError), std::out_of_range -> IndexError, ParseError / IoError as in
io.hpp:13-27.  There is no CPU fallback: importing this package raises if the
CUDA library is missing, and every call runs the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCB200_LIB") or os.path.join(_HERE, "libtcb200.so")  # TCB200_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(make -C paper_1909_02127_b200/csrc). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

TC_OK, TC_EINVAL, TC_ERANGE, TC_ENOMEM, TC_ECUDA, TC_ENCCL, TC_EUNSUPPORTED, TC_EPARSE, TC_EIO = range(9)

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class TcBuildReport(C.Structure):
    _fields_ = [("self_loops_removed", C.c_uint64), ("duplicate_entries_removed", C.c_uint64)]


class TcGraphInfo(C.Structure):
    _fields_ = [("num_vertices", C.c_uint32), ("num_edges", C.c_uint64), ("max_degree", C.c_uint32),
                ("max_out_degree", C.c_uint32), ("device", C.c_int), ("build_ms", C.c_double),
                ("core_ranks", C.c_uint32), ("dense_rows", C.c_uint32)]


class TcCountOpts(C.Structure):
    _fields_ = [("lookahead", C.c_int), ("keep_listings", C.c_int), ("part_index", C.c_uint32),
                ("part_count", C.c_uint32), ("sync", C.c_int), ("work_counters", C.c_int)]


class TcCountStats(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("frontier_ms", C.c_double), ("join_ms", C.c_double),
                ("reduce_ms", C.c_double), ("pivots", C.c_uint64), ("items", C.c_uint64),
                ("wedges", C.c_uint64), ("segments", C.c_uint64), ("join_launches", C.c_uint64),
                ("dag_W", C.c_double), ("alg_bytes", C.c_double), ("probe_bytes", C.c_double),
                ("kernel_launches", C.c_uint64), ("part_first_vertex", C.c_uint64),
                ("part_last_vertex", C.c_uint64), ("warp_ms", C.c_double), ("small_ms", C.c_double),
                ("cta_ms", C.c_double), ("dense_ms", C.c_double), ("rows_ms", C.c_double),
                ("cta_bytes", C.c_double), ("dense_bytes", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_sig("tc_abi_version", C.c_int, [])
_sig("tc_last_error", C.c_char_p, [])
_sig("tc_free", None, [C.c_void_p])
_sig("tc_graph_build", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.POINTER(C.c_void_p),
                                 C.POINTER(TcBuildReport)])
_sig("tc_graph_from_csr", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_int,
                                    C.POINTER(C.c_void_p)])
_sig("tc_graph_get_info", C.c_int, [C.c_void_p, C.POINTER(TcGraphInfo)])
_sig("tc_graph_export_csr", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p])
_sig("tc_graph_degrees", C.c_int, [C.c_void_p, C.c_void_p])
_sig("tc_graph_set_stream", C.c_int, [C.c_void_p, C.c_void_p])
_sig("tc_graph_destroy", None, [C.c_void_p])
_sig("tc_count", C.c_int, [C.c_void_p, C.POINTER(TcCountOpts), C.c_void_p, C.c_void_p,
                           C.POINTER(TcCountStats)])
_sig("tc_parse_matrix_market", C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(u32p), u64p, u32p])
_sig("tc_csr_cache_to_graph", C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p)])
_sig("tc_graph_load_matrix_market", C.c_int, [C.c_char_p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p),
                                              C.c_void_p])
_sig("tc_graph_csr_cache_size", C.c_int, [C.c_void_p, u64p])
_sig("tc_list_triangles", C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, u64p])
_sig("tc_list_triangles_range", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint64, u64p])
_sig("tc_graph_write_csr_cache", C.c_int, [C.c_void_p, C.c_void_p])
_sig("tc_partition_bounds", C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p])
_sig("tc_gen_num_edges", C.c_uint64, [C.c_int, C.c_int, C.c_int])
_sig("tc_generate", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p])
_sig("tc_release_cached_memory", C.c_uint64, [C.c_int])
_sig("tc_comm_unique_id", C.c_int, [C.c_void_p])
_sig("tc_comm_init_rank", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)])
_sig("tc_comm_destroy", None, [C.c_void_p])
_sig("tc_count_allreduce", C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(TcCountOpts), C.c_void_p, C.c_void_p,
                                     C.POINTER(TcCountStats)])
_sig("tc_multi_create", C.c_int, [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)])
_sig("tc_multi_destroy", None, [C.c_void_p])
_sig("tc_count_multi", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(TcCountOpts), C.c_void_p,
                                 C.c_void_p, C.POINTER(TcCountStats)])

EXPORTED_SYMBOLS = [
    "tc_abi_version", "tc_last_error", "tc_free", "tc_graph_build", "tc_graph_from_csr", "tc_graph_get_info",
    "tc_graph_export_csr", "tc_graph_degrees", "tc_graph_set_stream", "tc_graph_destroy", "tc_count",
    "tc_parse_matrix_market", "tc_csr_cache_to_graph", "tc_gen_num_edges", "tc_generate", "tc_partition_bounds",
    "tc_graph_load_matrix_market", "tc_graph_csr_cache_size", "tc_graph_write_csr_cache", "tc_list_triangles",
    "tc_list_triangles_range", "tc_release_cached_memory", "tc_comm_unique_id", "tc_comm_init_rank",
    "tc_comm_destroy", "tc_count_allreduce", "tc_multi_create", "tc_multi_destroy", "tc_count_multi",
]


# ---- exceptions (io.hpp:13-27, graph.cpp:16-20/:24-28/:40-42) ---------------

class InvalidArgument(ValueError):
    """std::invalid_argument"""


class ParseError(RuntimeError):
    """trimatch::ParseError (io.hpp:13-22): message ends with '(line N)'."""

    def __init__(self, message: str):
        super().__init__(message)
        import re
        m = re.search(r"\(line (\d+)\)$", message)
        self.line = int(m.group(1)) if m else 0


class IoError(RuntimeError):
    """trimatch::IoError (io.hpp:25-27)"""


class CudaError(RuntimeError):
    pass


class Unsupported(RuntimeError):
    pass


def _check(rc: int):
    if rc == TC_OK:
        return
    msg = (_lib.tc_last_error() or b"").decode()
    if rc == TC_EINVAL:
        raise InvalidArgument(msg)
    if rc == TC_ERANGE:
        raise IndexError(msg)
    if rc == TC_EPARSE:
        raise ParseError(msg)
    if rc == TC_EIO:
        raise IoError(msg)
    if rc == TC_EUNSUPPORTED:
        raise Unsupported(msg)
    if rc == TC_ENOMEM:
        raise MemoryError(msg)
    raise CudaError(f"[{rc}] {msg}")


def _addr(x, itemsize: Optional[int] = None, what: str = "buffer", integer: bool = True) -> int:
    """Address of a numpy array, a torch tensor (host or device) or an int.
    With itemsize, the element width is checked (the C-ABI reads raw words:
    a scipy int32 indptr passed as u64 offsets would be read past its end),
    and so are contiguity and an integer dtype."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        if not x.flags.c_contiguous:
            raise InvalidArgument(f"{what} must be C-contiguous")
        if itemsize is not None and (x.dtype.itemsize != itemsize or (integer and x.dtype.kind not in "iu")):
            raise InvalidArgument(f"{what} must be a {8 * itemsize}-bit integer array, got {x.dtype}")
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        if hasattr(x, "is_contiguous") and not x.is_contiguous():
            raise InvalidArgument(f"{what} must be contiguous")
        if itemsize is not None:
            es = x.element_size()
            if es != itemsize or (integer and (x.is_floating_point() or x.is_complex())):
                raise InvalidArgument(f"{what} must be a {8 * itemsize}-bit integer tensor, got {x.dtype}")
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


# ---- domain types ------------------------------------------------------------

@dataclass
class EdgeList:
    """graph.hpp:16-19: raw (u,v) pairs, may hold loops/dups/both orientations.
    `edges` is an (m,2) uint32 array (or anything convertible)."""
    num_vertices_declared: int = 0
    edges: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.uint32))

    def pairs(self) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(self.edges, dtype=np.uint32).reshape(-1, 2))
        return a


@dataclass
class BuildReport:
    self_loops_removed: int = 0
    duplicate_entries_removed: int = 0


@dataclass
class MatchOptions:
    """matcher.hpp:84-88.  lookahead is validated (0..2) and count-neutral on
    the GPU path; keep_listings adds MatchResult.listings."""
    lookahead: int = 2
    keep_listings: bool = False
    per_vertex: bool = False
    part_index: int = 0
    part_count: int = 1


@dataclass
class MatchResult:
    """matcher.hpp:90-94 (+ per_vertex u64[n] when requested)."""
    count: int = 0
    per_vertex: Optional[np.ndarray] = None
    stats: dict = field(default_factory=dict)
    listings: Optional[np.ndarray] = None  # (T, 3) u32, each row ascending (keep_listings)


class Graph:
    """Device-resident oriented graph (graph.hpp:35-66 semantics on the host
    side: num_vertices, num_edges, degree, row_offsets, neighbor_array,
    neighbors, has_edge).  The symmetric CSR is materialised on demand."""

    def __init__(self, handle: int, device: int):
        self._h = C.c_void_p(handle)
        self.device = device
        self._csr = None
        info = TcGraphInfo()
        _check(_lib.tc_graph_get_info(self._h, C.byref(info)))
        self._info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.tc_graph_destroy(h)
            except Exception:  # interpreter shutdown
                pass
            self._h = C.c_void_p(0)

    @property
    def handle(self):
        return self._h

    def num_vertices(self) -> int:
        return self._info.num_vertices

    def num_edges(self) -> int:
        return self._info.num_edges

    @property
    def max_degree(self) -> int:
        return self._info.max_degree

    @property
    def max_out_degree(self) -> int:
        return self._info.max_out_degree

    @property
    def core_ranks(self) -> int:
        """Dense core size (top ranks held as row bitmaps; 0 = none)."""
        return self._info.core_ranks

    @property
    def dense_rows(self) -> int:
        """Rows whose core members are intersected word-parallel."""
        return self._info.dense_rows

    @property
    def build_ms(self) -> float:
        return self._info.build_ms

    def set_stream(self, stream_ptr: int):
        _check(_lib.tc_graph_set_stream(self._h, C.c_void_p(stream_ptr or 0)))

    def export_csr(self, row_offsets=None, neighbors=None):
        """Symmetric CSR identical to the reference build_graph output; writes
        into the given buffers (host numpy or device tensors) or returns new
        numpy arrays."""
        n, E = self.num_vertices(), self.num_edges()
        ro = row_offsets if row_offsets is not None else np.empty(n + 1, np.uint64)
        nb = neighbors if neighbors is not None else np.empty(max(2 * E, 1), np.uint32)
        _check(_lib.tc_graph_export_csr(self._h, C.c_void_p(_addr(ro, 8, "row_offsets")),
                                        C.c_void_p(_addr(nb, 4, "neighbors"))))
        if neighbors is None:
            nb = nb[: 2 * E]
        return ro, nb

    def _ensure_csr(self):
        if self._csr is None:
            self._csr = self.export_csr()
        return self._csr

    def row_offsets(self) -> np.ndarray:
        return self._ensure_csr()[0]

    def neighbor_array(self) -> np.ndarray:
        return self._ensure_csr()[1]

    def degree(self, u: int) -> int:
        ro = self.row_offsets()
        return int(ro[u + 1] - ro[u])

    def neighbors(self, u: int) -> np.ndarray:
        ro, nb = self._ensure_csr()
        return nb[ro[u]: ro[u + 1]]

    def has_edge(self, u: int, v: int) -> bool:
        """graph.cpp:23-31 (out_of_range on a bad id)."""
        n = self.num_vertices()
        if u >= n or v >= n or u < 0 or v < 0:
            raise IndexError(f"has_edge: vertex id {u if (u >= n or u < 0) else v} out of range")
        nb = self.neighbors(u)
        i = int(np.searchsorted(nb, v))
        return i < nb.size and int(nb[i]) == v


# ---- operations ----------------------------------------------------------------

def build_graph(edges: EdgeList, report: Optional[BuildReport] = None, device: int = 0) -> Graph:
    """trimatch::build_graph (graph.hpp:73)."""
    pairs = edges.pairs() if isinstance(edges, EdgeList) else edges
    n = edges.num_vertices_declared if isinstance(edges, EdgeList) else None
    return build_graph_from_pairs(pairs, n, report=report, device=device)


def build_graph_from_pairs(pairs, n_declared: int, report: Optional[BuildReport] = None, device: int = 0,
                           m: Optional[int] = None) -> Graph:
    """pairs: (m,2)/(2m,) uint32 numpy array, or a host/device torch tensor."""
    if m is None:
        m = (pairs.size if isinstance(pairs, np.ndarray) else pairs.numel()) // 2
    h = C.c_void_p()
    rep = TcBuildReport()
    _check(_lib.tc_graph_build(C.c_void_p(_addr(pairs, 4, "pairs")), m, n_declared, device, C.byref(h), C.byref(rep)))
    if report is not None:
        report.self_loops_removed = rep.self_loops_removed
        report.duplicate_entries_removed = rep.duplicate_entries_removed
    return Graph(h.value, device)


def graph_from_csr(row_offsets, neighbors, n: Optional[int] = None, num_edges: Optional[int] = None,
                   device: int = 0) -> Graph:
    """The trimatch::Graph(num_vertices, num_edges, row_offsets, neighbors)
    constructor route (graph.hpp:38-39): upload an existing symmetric CSR."""
    if n is None:
        n = (row_offsets.size if isinstance(row_offsets, np.ndarray) else row_offsets.numel()) - 1
    if num_edges is None:
        num_edges = (neighbors.size if isinstance(neighbors, np.ndarray) else neighbors.numel()) // 2
    h = C.c_void_p()
    _check(_lib.tc_graph_from_csr(C.c_void_p(_addr(row_offsets, 8, "row_offsets")),
                                  C.c_void_p(_addr(neighbors, 4, "neighbors")), n, num_edges,
                                  device, C.byref(h)))
    return Graph(h.value, device)


def degrees(g: Graph) -> np.ndarray:
    """trimatch::degrees (graph.hpp:75)."""
    d = np.empty(max(g.num_vertices(), 1), np.uint32)
    _check(_lib.tc_graph_degrees(g.handle, C.c_void_p(d.ctypes.data)))
    return d[: g.num_vertices()]


def count_triangles(g: Graph, opts: Optional[MatchOptions] = None) -> MatchResult:
    """trimatch::count_triangles (matcher.hpp:128) on the GPU.  keep_listings
    adds the listings (tc_list_triangles): every triangle once, ids ascending."""
    opts = opts or MatchOptions()
    if opts.keep_listings:
        if opts.lookahead < 0 or opts.lookahead > 2:
            raise InvalidArgument("lookahead must be 0, 1, or 2")
        rows = list_triangles(g)
        r = count_triangles(g, MatchOptions(lookahead=opts.lookahead, per_vertex=opts.per_vertex,
                                            part_index=opts.part_index, part_count=opts.part_count))
        r.listings = rows
        return r
    o = TcCountOpts(opts.lookahead, int(opts.keep_listings), opts.part_index, opts.part_count, 1, 1)
    total = np.zeros(1, np.uint64)
    pv = np.zeros(max(g.num_vertices(), 1), np.uint64) if opts.per_vertex else None
    st = TcCountStats()
    _check(_lib.tc_count(g.handle, C.byref(o), C.c_void_p(total.ctypes.data),
                         C.c_void_p(pv.ctypes.data) if pv is not None else None, C.byref(st)))
    return MatchResult(count=int(total[0]), per_vertex=(pv[: g.num_vertices()] if pv is not None else None),
                       stats=st.as_dict())


def list_triangles(g: Graph, first_edge: int = 0, last_edge: Optional[int] = None) -> np.ndarray:
    """All triangles as a (T, 3) u32 array, each row ascending (the
    reference's listings rows u < w < x); row order unspecified.  With an
    oriented-edge range, only the triangles listed from those edges
    (tc_list_triangles_range; consecutive ranges partition the listing)."""
    last = g.num_edges() if last_edge is None else last_edge
    T = C.c_uint64()
    _check(_lib.tc_list_triangles_range(g.handle, first_edge, last, None, 0, C.byref(T)))
    rows = np.empty((max(T.value, 1), 3), np.uint32)
    n2 = C.c_uint64()
    _check(_lib.tc_list_triangles_range(g.handle, first_edge, last, C.c_void_p(rows.ctypes.data), T.value,
                                        C.byref(n2)))
    return rows[: T.value]


def list_triangles_count(g: Graph, first_edge: int = 0, last_edge: Optional[int] = None) -> int:
    """The number of triangles the listing kernel lists (capacity 0: nothing
    is written) -- an independent count (listing.cu) of the same graph."""
    last = g.num_edges() if last_edge is None else last_edge
    T = C.c_uint64()
    _check(_lib.tc_list_triangles_range(g.handle, first_edge, last, None, 0, C.byref(T)))
    return int(T.value)


def iter_listings(g: Graph, max_rows: int = 1 << 22, out=None):
    """Streamed listings: yields (k, 3) u32 arrays of at most max_rows rows
    whose concatenation is list_triangles(g), walking the oriented edges range
    by range with one bounded buffer (host, or a device tensor passed as out
    with room for max_rows rows).  A range whose triangles overflow the buffer
    is halved and re-listed; one that fits grows the next range.  Each yielded
    array is a view of the buffer, valid until the next step."""
    if max_rows < 1:
        raise InvalidArgument("iter_listings: max_rows must be >= 1")
    if out is None:
        out = np.empty((max_rows, 3), np.uint32)
        ptr = out.ctypes.data
    else:
        ptr = out.data_ptr()
    E = g.num_edges()
    e, span = 0, max(1, min(E, 1 << 16))
    T = C.c_uint64()
    while e < E:
        b = min(E, e + span)
        _check(_lib.tc_list_triangles_range(g.handle, e, b, C.c_void_p(ptr), max_rows, C.byref(T)))
        if T.value > max_rows:
            if b - e == 1:  # one edge's triangles exceed the buffer
                raise InvalidArgument(f"iter_listings: edge {e} lists {T.value} triangles > max_rows")
            span = max(1, (b - e) // 2)
            continue
        if T.value:
            yield out[: T.value]
        e = b
        if 2 * T.value <= max_rows:
            span *= 2


def count_triangles_into(g: Graph, total_ptr, per_vertex_ptr=None, opts: Optional[MatchOptions] = None,
                         stats: bool = False, sync: bool = False, work_counters: bool = False):
    """Low-level: outputs to caller buffers (device tensors for the multi-GPU
    allreduce path).  Returns the stats dict when stats=True (phase times;
    work_counters=True adds W / J / items / byte models, one extra pass)."""
    opts = opts or MatchOptions()
    o = TcCountOpts(opts.lookahead, int(opts.keep_listings), opts.part_index, opts.part_count, int(sync),
                    int(work_counters))
    st = TcCountStats()
    _check(_lib.tc_count(g.handle, C.byref(o), C.c_void_p(_addr(total_ptr, 8, "total")),
                         C.c_void_p(_addr(per_vertex_ptr, 8, "per_vertex")) if per_vertex_ptr is not None else None,
                         C.byref(st) if stats else None))
    return st.as_dict() if stats else None


# ---- multi-GPU (tcb200.h tc_comm_* / tc_multi_*) -------------------------------

COMM_ID_BYTES = 128


class Comm:
    """One rank of a one-process-per-GPU group (torchrun style).  The count
    splits the graph's pivots over the ranks and ONE NCCL allreduce over
    NVLink combines them (tc_count_allreduce); torch.distributed is only the
    rendezvous that carries the 128-byte NCCL id (see dist.py)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(COMM_ID_BYTES)
        _check(_lib.tc_comm_unique_id(buf))
        return buf.raw

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        if len(uid) != COMM_ID_BYTES:
            raise InvalidArgument(f"NCCL id must be {COMM_ID_BYTES} bytes")
        h = C.c_void_p()
        _check(_lib.tc_comm_init_rank(C.create_string_buffer(uid, COMM_ID_BYTES), nranks, rank, device, C.byref(h)))
        self._h, self.nranks, self.rank, self.device = h, nranks, rank, device

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.tc_comm_destroy(self._h)
            self._h = C.c_void_p(0)

    __del__ = close

    def count_into(self, g: Graph, total, per_vertex=None, opts: Optional[MatchOptions] = None, stats: bool = False,
                   sync: bool = False):
        """This rank's part + the allreduce, into caller buffers (device
        tensors keep the call asynchronous on the graph's stream)."""
        opts = opts or MatchOptions()
        o = TcCountOpts(opts.lookahead, int(opts.keep_listings), 0, 0, int(sync), 0)
        st = TcCountStats()
        _check(_lib.tc_count_allreduce(self._h, g.handle, C.byref(o), C.c_void_p(_addr(total, 8, "total")),
                                       C.c_void_p(_addr(per_vertex, 8, "per_vertex")) if per_vertex is not None
                                       else None, C.byref(st) if stats else None))
        return st.as_dict() if stats else None

    def count_triangles(self, g: Graph, opts: Optional[MatchOptions] = None) -> MatchResult:
        opts = opts or MatchOptions()
        total = np.zeros(1, np.uint64)
        pv = np.zeros(max(g.num_vertices(), 1), np.uint64) if opts.per_vertex else None
        st = self.count_into(g, total, pv, opts, stats=True, sync=True)
        return MatchResult(count=int(total[0]), per_vertex=(pv[: g.num_vertices()] if pv is not None else None),
                           stats=st)


class MultiGPU:
    """One process driving several GPUs (tc_multi_create / tc_count_multi):
    devices[p] is the device of part p; a device may repeat (its parts run back
    to back and are summed before the allreduce)."""

    def __init__(self, devices):
        self.devices = [int(d) for d in devices]
        arr = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _check(_lib.tc_multi_create(arr, len(self.devices), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.tc_multi_destroy(self._h)
            self._h = C.c_void_p(0)

    __del__ = close

    def count_triangles(self, graphs, opts: Optional[MatchOptions] = None, total=None, per_vertex=None):
        """graphs[p] = the replica on devices[p].  Host outputs by default."""
        if len(graphs) != len(self.devices):
            raise InvalidArgument("one graph per part")
        opts = opts or MatchOptions()
        hs = (C.c_void_p * len(graphs))(*[g.handle.value for g in graphs])
        n = graphs[0].num_vertices()
        tot = total if total is not None else np.zeros(1, np.uint64)
        pv = per_vertex if per_vertex is not None else (np.zeros(max(n, 1), np.uint64) if opts.per_vertex else None)
        o = TcCountOpts(opts.lookahead, int(opts.keep_listings), 0, 0, 1, 0)
        st = TcCountStats()
        _check(_lib.tc_count_multi(self._h, hs, C.byref(o), C.c_void_p(_addr(tot, 8, "total")),
                                   C.c_void_p(_addr(pv, 8, "per_vertex")) if pv is not None else None,
                                   C.byref(st)))
        if total is not None:
            return st.as_dict()
        return MatchResult(count=int(tot[0]), per_vertex=(pv[:n] if pv is not None and per_vertex is None else pv),
                           stats=st.as_dict())


def partition_bounds(g: Graph, parts: int) -> np.ndarray:
    """Degree-weighted pivot rank ranges of a `parts`-way multi-GPU split
    (what tc_count uses for part_index/part_count): part p counts the
    triangles whose middle vertex has (deg,id) rank in [b[p], b[p+1])."""
    b = np.zeros(parts + 1, np.uint64)
    _check(_lib.tc_partition_bounds(g.handle, parts, C.c_void_p(b.ctypes.data)))
    return b


def parse_matrix_market(text) -> EdgeList:
    """trimatch::parse_matrix_market (io.hpp:34, io.cpp:93-159)."""
    if isinstance(text, str):
        text = text.encode()
    p = u32p()
    m = C.c_uint64()
    n = C.c_uint32()
    _check(_lib.tc_parse_matrix_market(text, len(text), C.byref(p), C.byref(m), C.byref(n)))
    arr = np.ctypeslib.as_array(p, shape=(2 * m.value + 2,))[: 2 * m.value].copy()
    _lib.tc_free(p)
    return EdgeList(n.value, arr.reshape(-1, 2))


def parse_matrix_market_file(path: str) -> EdgeList:
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise IoError(f"cannot open '{path}' for reading")
    return parse_matrix_market(data)


_CSR_MAGIC = b"TRIMCSR1"


def is_csr_cache_file(path: str) -> bool:
    try:
        with open(path, "rb") as f:
            return f.read(8) == _CSR_MAGIC
    except OSError:
        return False


def read_csr_cache(path: str, device: int = 0) -> Graph:
    """trimatch::read_csr_cache (io.cpp:187-220): validated on ingest."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise IoError(f"cannot open '{path}' for reading")
    h = C.c_void_p()
    _check(_lib.tc_csr_cache_to_graph(data, len(data), device, C.byref(h)))
    return Graph(h.value, device)


def csr_cache_bytes(g: Graph) -> np.ndarray:
    """The TRIMCSR1 image of g (write_csr_cache's bytes), assembled by the
    library from the device graph."""
    n = C.c_uint64()
    _check(_lib.tc_graph_csr_cache_size(g.handle, C.byref(n)))
    buf = np.empty((n.value + 7) // 8, np.uint64)  # 8-byte aligned
    _check(_lib.tc_graph_write_csr_cache(g.handle, C.c_void_p(buf.ctypes.data)))
    return buf.view(np.uint8)[: n.value]


def write_csr_cache(path: str, g: Graph) -> None:
    """trimatch::write_csr_cache (io.cpp:167-177): little-endian TRIMCSR1 v1."""
    data = csr_cache_bytes(g)
    try:
        with open(path, "wb") as f:
            f.write(data.tobytes())
    except OSError:
        raise IoError(f"cannot open '{path}' for writing")


def load_matrix_market(text, report: Optional[BuildReport] = None, device: int = 0) -> Graph:
    """load_graph for MatrixMarket bytes: entries tokenized and built on the GPU
    (tc_graph_load_matrix_market); same errors as parse_matrix_market."""
    if isinstance(text, str):
        text = text.encode()
    h = C.c_void_p()
    rep = TcBuildReport()
    _check(_lib.tc_graph_load_matrix_market(text, len(text), device, C.byref(h), C.byref(rep)))
    if report is not None:
        report.self_loops_removed = rep.self_loops_removed
        report.duplicate_entries_removed = rep.duplicate_entries_removed
    return Graph(h.value, device)


def load_graph(path: str, report: Optional[BuildReport] = None, device: int = 0) -> Graph:
    """trimatch::load_graph (io.cpp:222-228): TRIMCSR1 or MatrixMarket."""
    if is_csr_cache_file(path):
        if report is not None:
            report.self_loops_removed = 0
            report.duplicate_entries_removed = 0
        return read_csr_cache(path, device)
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise IoError(f"cannot open '{path}' for reading")
    return load_matrix_market(data, report, device)


# ---- synthetic inputs --------------------------------------------

GEN_RMAT, GEN_KRON, GEN_ER = 0, 1, 2


def gen_num_edges(kind: int, scale: int, param: int) -> int:
    return _lib.tc_gen_num_edges(kind, scale, param)


def generate(kind: int, scale: int, param: int, out=None, device: int = 0):
    """Deterministic RMAT / Kronecker / ER edge list generated on the GPU into
    `out` (host numpy or device tensor of 2m uint32); returns it."""
    m = gen_num_edges(kind, scale, param)
    if out is None:
        out = np.empty(2 * m, np.uint32)
    _check(_lib.tc_generate(kind, scale, param, device, C.c_void_p(_addr(out, 4, "out"))))
    return out


def release_cached_memory(device: int = -1) -> int:
    """Return the library's cached device blocks to the driver (bytes freed)."""
    return int(_lib.tc_release_cached_memory(device))


def abi_version() -> int:
    return _lib.tc_abi_version()
