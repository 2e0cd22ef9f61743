/*
 * tcb200.h -- C-ABI of libtcb200.so, the B200-native drop-in for the reference
 * triangle-counting hot path (trimatch, /root/reference/proj).
 *
 * Plain pointers and sizes only; no CUDA or torch types cross this boundary
 * (streams are passed as void*).  Every input/output buffer may live in host
 * memory or in device memory of the handle's device: the library inspects each
 * pointer (cudaPointerGetAttributes) and copies as needed.
 *
 * Entry point                 replaces (reference, relative to proj/)
 * ---------------------------------------------------------------------------
 * tc_graph_build              trimatch::build_graph      include/trimatch/graph.hpp:73
 *                             (graph.cpp:33-85; BuildReport graph.hpp:22-25)
 * tc_graph_from_csr           trimatch::Graph ctor       graph.hpp:38-39 (graph.cpp:9-21)
 *                             -- the route count_triangles(const Graph&) takes
 * tc_graph_export_csr         Graph::row_offsets()/neighbor_array() graph.hpp:58-59
 * tc_graph_degrees            trimatch::degrees          graph.hpp:75 (graph.cpp:87-91)
 * tc_count                    trimatch::count_triangles  matcher.hpp:128
 *                             (matcher.cpp:301-303 -> match :249-299 ->
 *                              count_final_level :204-245)
 * tc_parse_matrix_market      trimatch::parse_matrix_market io.hpp:34 (io.cpp:93-159)
 * tc_graph_load_matrix_market trimatch::load_graph (MatrixMarket) io.hpp:45
 * tc_list_triangles           count_triangles(keep_listings).listings matcher.hpp:92
 * tc_list_triangles_range     the same listing streamed by oriented-edge range  matcher.cpp:169-181
 * tc_graph_write_csr_cache    trimatch::write_csr_cache  io.hpp:39 (io.cpp:167-177)
 * tc_csr_cache_parse          trimatch::read_csr_cache   io.hpp:40 (io.cpp:187-220)
 * tc_graph_destroy            ~Graph
 * tc_comm_init_rank / tc_count_allreduce   multi-GPU count, one process per GPU
 * tc_multi_create / tc_count_multi         multi-GPU count, one process (SURVEY 8b
 *                             tc_count_multi; the reference is single-node CPU,
 *                             this is the north-star's 8-GPU split)
 * tc_last_error               the what() of the exception the reference throws
 *
 * Errors: the reference throws C++ exceptions; here each maps to a status code
 * (graph.cpp:40-42 invalid_argument -> TC_EINVAL; graph.cpp:24-28 out_of_range
 * -> TC_ERANGE; io.hpp:13-22 ParseError -> TC_EPARSE; io.hpp:25-27 IoError ->
 * TC_EIO).  include/trimatch_gpu.hpp maps them back to the same exception types.
 * On error no handle is returned and outputs are left untouched.
 *
 * Threading: calls on one handle are serialised on the handle's stream; handles
 * on different devices are independent.  tc_last_error() is thread-local.
 */
#ifndef TCB200_H
#define TCB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCB200_ABI_VERSION 3

typedef enum tc_status {
  TC_OK = 0,
  TC_EINVAL = 1,       /* std::invalid_argument */
  TC_ERANGE = 2,       /* std::out_of_range, or a size past the 32-bit id / edge limits */
  TC_ENOMEM = 3,       /* device allocation failed */
  TC_ECUDA = 4,        /* CUDA runtime error (message in tc_last_error) */
  TC_ENCCL = 5,        /* NCCL error in the multi-GPU allreduce, or NCCL not loadable (bound at
                          first multi-GPU call: libnccl.so.2 or $TCB_NCCL_LIB) */
  TC_EUNSUPPORTED = 6, /* keep_listings etc. (out of scope on the GPU path) */
  TC_EPARSE = 7,       /* trimatch::ParseError */
  TC_EIO = 8           /* trimatch::IoError */
} tc_status;

typedef struct tc_graph tc_graph;

/* trimatch::BuildReport (graph.hpp:22-25). */
typedef struct tc_build_report {
  uint64_t self_loops_removed;
  uint64_t duplicate_entries_removed;
} tc_build_report;

typedef struct tc_graph_info {
  uint32_t num_vertices;   /* Graph::num_vertices()   graph.hpp:41 */
  uint64_t num_edges;      /* Graph::num_edges()      graph.hpp:43 (undirected, once) */
  uint32_t max_degree;
  uint32_t max_out_degree; /* max d+ in the (deg,id)-oriented DAG */
  int device;
  double build_ms;         /* device time of the last build/from_csr (CUDA events) */
  uint32_t core_ranks;     /* dense core: the top core_ranks ranks (0 = no dense rows) */
  uint32_t dense_rows;     /* rows whose core members are held as a core bitmap */
} tc_graph_info;

/* trimatch::MatchOptions (matcher.hpp:84-88) + GPU extensions. */
typedef struct tc_count_opts {
  int lookahead;        /* validated in {0,1,2} like matcher.cpp:250-252; count-neutral */
  int keep_listings;    /* must be 0 here: listings are tc_list_triangles */
  uint32_t part_index;  /* multi-GPU: this rank's share of the degree-weighted */
  uint32_t part_count;  /*   pivot rank ranges (0/1 = whole graph)            */
  int sync;             /* 1: block until outputs are final (default for 0-init = async
                           only when both outputs are device pointers) */
  int work_counters;    /* 1 (with stats): also count W, J, items (one extra pass) */
} tc_count_opts;

/* trimatch::MatchStats analogue (matcher.hpp:69-82) for the GPU path. */
typedef struct tc_count_stats {
  double total_ms;        /* device time of the whole tc_count (CUDA events) */
  double frontier_ms;     /* level-1 frontier plan: pivot classes + work segments */
  double join_ms;         /* advance + fused join kernels + per-vertex row pass */
  double reduce_ms;       /* per-vertex gather + total                         */
  uint64_t pivots;        /* vertices v with d+(v)>0 and >=1 in-edge (seeds)   (work_counters) */
  uint64_t items;         /* in-edges (u->v) whose wedge suffix is non-empty  (work_counters) */
  uint64_t wedges;        /* J = candidate wedges probed = sum of suffix lengths (work_counters) */
  uint64_t segments;      /* reserved */
  uint64_t join_launches; /* join kernel launches                              */
  double dag_W;           /* W = sum_{u->v} d+(v) (SURVEY 8d wedge-stream model; work_counters) */
  double alg_bytes;       /* B_alg = 4W + 12|E+| + 8(|V|+1) [+8|V| per-vertex]  (work_counters) */
  double probe_bytes;     /* bytes the implemented join streams (work_counters) */
  uint64_t kernel_launches; /* all libtcb200 kernels this call launched */
  uint64_t part_first_vertex; /* this part's pivot rank range [first, last) */
  uint64_t part_last_vertex;
  /* per-kernel device times of this call (CUDA events around each launch) */
  double warp_ms;         /* k_join_warp   (pivots with d+ <= 64)            */
  double small_ms;        /* k_join_small  (pivots with <= 32 in-edges)      */
  double cta_ms;          /* k_join_cta    (sparse join, the dominant kernel) */
  double dense_ms;        /* k_join_dense  (dense-core items)                */
  double rows_ms;         /* k_pv_rows + k_pv_rows_heavy (per-vertex masks)  */
  /* algorithmic bytes of one launch (work_counters): what the kernel's
   * algorithm must move -- k_join_cta: 2 B per sparse hot candidate + 4 B per
   * cold candidate + 32 B per item (its in-edge item record) + its
   * per-vertex mask bytes + 4 B per pivot member and 16 B per segment;
   * k_join_dense: 8 B per dense item (list entry, row rank) + 4 B per core
   * word of its row + 288 B per segment (pivot descriptor + core words) */
  double cta_bytes;
  double dense_bytes;
} tc_count_stats;

/* ---- graph construction ------------------------------------------------ */

/* build_graph: pairs = 2*m u32 interleaved (u,v) -- the memory layout of
 * trimatch::EdgeList::edges (vector<pair<u32,u32>>), host or device.  Drops
 * self-loops and duplicates, symmetrises; ids >= n_declared -> TC_EINVAL. */
tc_status tc_graph_build(const uint32_t* pairs, uint64_t m, uint32_t n_declared, int device,
                         tc_graph** out, tc_build_report* report);

/* Graph ctor route: an existing symmetric CSR (row_offsets n+1 u64, neighbors
 * 2E u32, rows strictly ascending, the Graph invariants graph.hpp:29-32). */
tc_status tc_graph_from_csr(const uint64_t* row_offsets, const uint32_t* neighbors, uint32_t n,
                            uint64_t num_edges, int device, tc_graph** out);

tc_status tc_graph_get_info(const tc_graph* g, tc_graph_info* info);

/* Symmetric CSR byte-identical to the reference build_graph output:
 * row_offsets (n+1 u64) and neighbors (2E u32), caller-owned, host or device. */
tc_status tc_graph_export_csr(tc_graph* g, uint64_t* row_offsets, uint32_t* neighbors);

/* degrees(g) (graph.cpp:87-91): n u32, caller-owned, host or device. */
tc_status tc_graph_degrees(tc_graph* g, uint32_t* degrees);

/* Launch subsequent work on this CUDA stream (cudaStream_t as void*; NULL =
 * the handle's own stream). */
tc_status tc_graph_set_stream(tc_graph* g, void* stream);

void tc_graph_destroy(tc_graph* g);

/* ---- the hot path ------------------------------------------------------ */

/* count_triangles: total (u64, host or device) and optional per-vertex
 * counts (n u64 in original vertex ids; host or device; NULL = total only).
 * With opts->part_count > 1 only this part's work ranges are counted; summing
 * total/per_vertex over all parts (one NCCL allreduce) gives the full result. */
tc_status tc_count(tc_graph* g, const tc_count_opts* opts, uint64_t* total, uint64_t* per_vertex,
                   tc_count_stats* stats);

/* Multi-GPU split: bounds[0..parts] (parts+1 u64, host) of the degree-weighted
 * pivot rank ranges tc_count uses for part_index/part_count: part p counts the
 * triangles whose middle vertex (in (deg,id) order) has rank in
 * [bounds[p], bounds[p+1]).  Computed once per graph and part count. */
tc_status tc_partition_bounds(tc_graph* g, uint32_t parts, uint64_t* bounds);

/* ---- multi-GPU ----------------------------------------------
 * Every GPU holds a replica of the graph (built from the same edge list or
 * CSR: no communication).  Part p of P counts the triangles whose middle
 * vertex lies in its degree-weighted pivot range (tc_partition_bounds); ONE
 * ncclAllReduce(ncclUint64, ncclSum) over NVLink of [per-vertex | total] on the
 * count stream combines the parts.  Outputs as tc_count (host or device of the
 * handle's device; with device outputs and opts->sync = 0 the call does not
 * block). */
typedef struct tc_comm tc_comm;
typedef struct tc_multi tc_multi;
#define TC_COMM_ID_BYTES 128

/* One process per GPU (torchrun style): rank 0 makes the 128-byte id, the
 * host framework hands it to every rank, each rank joins with its device. */
tc_status tc_comm_unique_id(void* id);
tc_status tc_comm_init_rank(const void* id, int nranks, int rank, int device, tc_comm** out);
void tc_comm_destroy(tc_comm* comm);
/* This rank's part (part_index = rank, part_count = nranks) + the allreduce:
 * every rank receives the whole graph's total / per-vertex counts. */
tc_status tc_count_allreduce(tc_comm* comm, tc_graph* g, const tc_count_opts* opts, uint64_t* total,
                             uint64_t* per_vertex, tc_count_stats* stats);

/* One process driving several GPUs (ncclCommInitAll, one stream per GPU):
 * devices[p] = the device of part p (a device may repeat: its parts run back
 * to back and are summed locally before the allreduce). */
tc_status tc_multi_create(const int* devices, int nparts, tc_multi** out);
void tc_multi_destroy(tc_multi* m);
/* graphs[p] = the replica on devices[p] (one handle may serve several parts of
 * its device).  Outputs on the host or on part 0's device; blocks until final.
 * stats (nullable): part 0's phases, total_ms = the slowest part. */
tc_status tc_count_multi(tc_multi* m, tc_graph* const* graphs, const tc_count_opts* opts, uint64_t* total,
                         uint64_t* per_vertex, tc_count_stats* stats);

/* ---- adjacent formats ------------------------------------- */

/* parse_matrix_market over an in-memory byte buffer (host).  On success
 * *pairs is a malloc'ed 2*m u32 buffer (free with tc_free). */
tc_status tc_parse_matrix_market(const char* text, uint64_t len, uint32_t** pairs, uint64_t* m,
                                 uint32_t* n_declared);

/* TRIMCSR1 binary cache (io.cpp:18-19, :167-220) held in memory: validates
 * and builds a handle straight from the CSR (no sort). */
tc_status tc_csr_cache_to_graph(const void* bytes, uint64_t len, int device, tc_graph** out);

/* count_triangles(keep_listings = true) listings (matcher.hpp:92,
 * matcher.cpp:169-181): every triangle once as 3 u32 vertex ids in ascending
 * order (the reference's u < w < x).  Writes min(T, capacity) rows to rows
 * (host or device, 3*capacity u32) and T to *count; capacity 0 sizes the
 * buffer.  Row order is unspecified. */
tc_status tc_list_triangles(tc_graph* g, uint32_t* rows, uint64_t capacity, uint64_t* count);

/* Streamed listings: the triangles listed from the oriented edges
 * [first_edge, last_edge) of the degree-ordered DAG (each triangle from
 * exactly one edge, so consecutive ranges partition the listing; 0 <= first
 * <= last <= num_edges).  Same output contract as tc_list_triangles, so a
 * caller with a bounded buffer walks the edges range by range. */
tc_status tc_list_triangles_range(tc_graph* g, uint64_t first_edge, uint64_t last_edge, uint32_t* rows,
                                  uint64_t capacity, uint64_t* count);

/* load_graph for MatrixMarket text (io.cpp:222-228 -> parse_matrix_market
 * io.cpp:93-159 -> build_graph graph.cpp:33-85) held in memory: the banner and
 * size line on the host, the entry lines tokenized on the device, then the
 * device build.  Malformed text fails with TC_EPARSE and the reference's
 * message and line number. */
tc_status tc_graph_load_matrix_market(const char* text, uint64_t len, int device, tc_graph** out,
                                      tc_build_report* report);

/* write_csr_cache (io.cpp:167-177) into caller memory: *len bytes (8-byte
 * aligned buffer), little-endian TRIMCSR1 image of the graph. */
tc_status tc_graph_csr_cache_size(const tc_graph* g, uint64_t* len);
tc_status tc_graph_write_csr_cache(tc_graph* g, void* bytes);

/* ---- synthetic inputs (SURVEY 8d generators, bit-exact on device) ------- */

/* kind: 0 = RMAT (Graph500 a,b,c = .57,.19,.19), 1 = Kronecker (RMAT +
 * seeded Fisher-Yates label permutation), 2 = Erdos-Renyi G(n,m).
 * param = edgefactor (RMAT/Kron) or average degree (ER).  pairs: 2*m u32,
 * host or device.  tc_gen_num_edges gives m. */
uint64_t tc_gen_num_edges(int kind, int scale, int param);
tc_status tc_generate(int kind, int scale, int param, int device, uint32_t* pairs);

void tc_free(void* p);

/* Device memory: graph handles and count scratch come from a caching
 * allocator (freed blocks are reused by the next handle / count without
 * remapping).  The cache is bounded (TCB_CACHE_MB, default 40% of the
 * device); this returns every cached block of `device` (-1 = all) to the
 * driver and reports the bytes released, e.g. before a host framework in the
 * same process allocates. */
uint64_t tc_release_cached_memory(int device);
const char* tc_last_error(void);
int tc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TCB200_H */
