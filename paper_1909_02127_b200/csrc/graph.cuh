// graph.cuh -- the device-resident graph handle behind the opaque tc_graph.
//
// HBM layout (all arrays in degree-rank space, rank = position of (deg, id) in
// ascending order, so the north-star orientation u->v iff (deg u,u) < (deg v,v)
// is simply rank(u) < rank(v)):
//   off[n+1]  u32  oriented CSR row offsets (|E+| = |E| < 2^32)
//   col[|E|]  u32  N+(r) as ranks, strictly ascending per row, +16 B tail pad
//   src[|E|]  u32  source rank of each oriented edge (COO companion of col)
//   deg[n]    u32  undirected degree by rank
//   id_of[n]  u32  rank -> original vertex id
//   rank_of[n]u32  original vertex id -> rank
// 16 B per oriented edge + 16 B per vertex: C4 (RMAT s24) = 4.4 GB,
// C5 (RMAT s26 ef32) = 34 GB of 180 GB.
#pragma once

#include <vector>

#include "common.cuh"

struct tc_graph {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  uint32_t n = 0;
  uint64_t E = 0;
  uint32_t max_deg = 0;
  uint32_t max_dplus = 0;
  int id_bits = 1;  // bits_for(n-1)
  double build_ms = 0;
  tcb::DBuf<uint32_t> off, col, src, deg, id_of, rank_of;
  // multi-GPU work partition (count.cu): oriented-edge ranges [b[p], b[p+1])
  // with ~equal wedge work, cached for the last part count requested
  uint32_t cached_parts = 0;
  std::vector<uint64_t> part_bounds;
};

namespace tcb {

// Build pipeline entry points (build.cu).
void build_from_pairs(tc_graph& g, const uint32_t* d_pairs, uint64_t m, uint32_t n,
                      tc_build_report* rep);
void build_from_csr(tc_graph& g, const uint64_t* d_off, const uint32_t* d_nbrs, uint32_t n,
                    uint64_t num_edges);
void export_csr(tc_graph& g, uint64_t* d_off, uint32_t* d_nbrs);
void export_degrees(tc_graph& g, uint32_t* d_deg);

// Count pipeline (count.cu).
void count_triangles(tc_graph& g, const tc_count_opts& opts, uint64_t* d_total,
                     uint64_t* d_per_vertex, tc_count_stats* stats);

// Generators (gen.cu).
uint64_t gen_num_edges(int kind, int scale, int param);
void generate(int kind, int scale, int param, uint32_t* d_pairs, cudaStream_t s);

}  // namespace tcb
