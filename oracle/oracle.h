/*
 * oracle.h -- CPU restatement of the reference triangle-counting path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1909_02127_b200/,
 * include/) links or calls this.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it, and there only
 * as the checker, never as the thing measured for the GPU arm.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  The restatement is pinned against the reference
 * itself (oracle/_ref, compiled from the reference sources by oracle/Makefile)
 * and against the golden vectors in tests/golden/ (see tests/test_oracle.py).
 */
#ifndef TC_ORACLE_H
#define TC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Deterministic counter-based generators (bit-exact).
 * pairs: 2*m u32, interleaved (u,v) like trimatch::EdgeList::edges. */
uint64_t oracle_rmat_num_edges(int scale, int edgefactor);
void oracle_gen_rmat(int scale, int edgefactor, int permute, uint32_t* pairs);
uint64_t oracle_er_num_edges(int scale, int avg_degree);
void oracle_gen_er(int scale, int avg_degree, uint32_t* pairs);
/* Edges [i0, i1) only (kind 0 = RMAT/Kronecker with perm = nullable
 * relabelling from oracle_kron_perm, 1 = ER): the big-config driver
 * (oracle/big_golden.c) streams a 2^31-edge graph through it. */
void oracle_gen_range(int kind, int scale, int param, uint64_t i0, uint64_t i1, const uint32_t* perm,
                      uint32_t* pairs);
void oracle_kron_perm(int scale, uint32_t* perm);

/* build_graph restatement (graph.cpp:33-85).  Returns 0 on success, -1 when an
 * id is out of range (the reference throws std::invalid_argument,
 * graph.cpp:40-42).  *offsets (n+1 u64) and *nbrs (2|E| u32) are malloc'ed and
 * owned by the caller (free with oracle_free). */
int oracle_build_graph(const uint32_t* pairs, uint64_t m, uint32_t n,
                       uint64_t** offsets, uint32_t** nbrs, uint64_t* num_edges,
                       uint64_t* self_loops, uint64_t* dups);
void oracle_free(void* p);

/* Triangle count by the reference's segmented intersection with
 * above_dst_only over the pairs {(u,v): u<v} (frontier.cpp:14-81,
 * SPEC.md:376 equality with count_triangles).  per_vertex (nullable, n u64):
 * t[x] = number of triangles containing x (the histogram of the listings
 * count_triangles(keep_listings=true) returns, matcher.hpp:92). */
uint64_t oracle_count(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n,
                      uint64_t* per_vertex, int threads);

/* Degree-ordered DAG count (pivot join over the (deg,id) orientation, the
 * SURVEY.md 8c host-validated algorithm): same total and per-vertex array as
 * oracle_count, orders of magnitude faster on skewed graphs.  The independent
 * checker for configs where oracle_count does not finish (C5); pinned against
 * the reference goldens by tests/test_oracle.py. */
uint64_t oracle_count_dag(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n,
                          uint64_t* per_vertex, int threads);

/* Brute force a<b<c over has_edge, n <= 5000 guard.
 * Returns UINT64_MAX when the guard trips. */
uint64_t oracle_brute_force(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n);

/* FNV-1a-64 over a byte buffer; the golden per-vertex fingerprints use it over
 * the little-endian u64 array. */
uint64_t oracle_fnv1a64(const void* data, uint64_t nbytes);

/* Per-seed visit cost deg(u)*|N(u) > u| of the reference's final level
 * (bench.py's bounded CPU sample). */
void oracle_seed_costs(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n, double* cost);

/* Sum over the oriented DAG (deg,id) of the work model used by bench.py's
 * roofline: fills W = sum_{u->v} d+(v), S2 = sum_u d+(u)^2,
 * and J = sum_u C(d+(u),2) restricted to pivots with d+>0 (the pivot join's
 * probe count). */
void oracle_dag_stats(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n,
                      double* W, double* S2, double* J, uint32_t* max_dplus);

#ifdef __cplusplus
}
#endif
#endif
