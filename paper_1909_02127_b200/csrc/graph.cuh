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
  // Hot window: the top kHotBits ranks [h0, n), where ~97% of wedge endpoints
  // of a power-law DAG fall (n-x < 2^16 for 97% of probes).  Each
  // row's members >= h0 form its sorted suffix; they are mirrored as 16-bit
  // offsets x - h0 in colH (row r at [offH[r], offH[r+1])), halving the bytes
  // the join streams and letting a probe index the pivot bitmap directly.
  uint32_t h0 = 0;
  tcb::DBuf<uint16_t> colH;
  tcb::DBuf<uint32_t> offH;
  // Level-1 frontier index (frontier.cu): the useful in-edges u->v of every
  // pivot v (d+(v) > 0, non-empty suffix), grouped by v and sorted by edge id
  // e -- the transpose of the oriented CSR restricted to wedge-producing
  // edges, i.e. the reference's level-1 PartialTable rows (u,v)
  // (matcher.cpp:136-198).  Graph-static, built once with the CSR.
  //   fr_items[i] = {hb,he,cb,ce} (CTA-bin pivots: hot range in colH, cold
  //                 range in col) or {b,e,0,0} (warp-bin pivots: col range)
  //   fr_e[i]     = the edge id (source u = src[e]; multi-GPU ranges)
  //   fr_in[v]    = first item of pivot v (n+1)
  //   fr_wsegs / fr_csegs = {v, i0, i1, 0} work segments per bin (whole graph)
  tcb::DBuf<uint4> fr_items;
  tcb::DBuf<uint32_t> fr_e, fr_in;
  //   fr_moff[e] = byte offset of edge e's per-vertex hit masks (1 byte per
  //   hot chunk of its CTA-bin item), exclusive scan in edge order (E+1), so
  //   a row's masks are contiguous and an item's length gives its first chunk
  tcb::DBuf<uint64_t> fr_moff;
  uint64_t fr_mask_bytes = 0;
  tcb::DBuf<uint4> fr_wsegs, fr_csegs;
  uint64_t fr_nitems = 0, fr_nwsegs = 0, fr_ncsegs = 0, fr_pivots = 0;
  uint64_t fr_W = 0, fr_J = 0, fr_hot = 0, fr_nitems_c = 0;
  double frontier_ms = 0;
  // multi-GPU work partition (count.cu): oriented-edge ranges [b[p], b[p+1])
  // with ~equal wedge work, cached for the last part count requested
  uint32_t cached_parts = 0;
  std::vector<uint64_t> part_bounds;
};

namespace tcb {

constexpr uint32_t kHotBits = 1u << 16;
constexpr uint32_t kWarpMaxDeg = 48;    // warp bin: d+(v) <= 48 (128-slot warp table)
constexpr uint32_t kWarpSegItems = 64;  // items per warp-bin segment
constexpr uint32_t kCtaSegItems = 512;  // items per CTA-bin segment

// Level-1 frontier index (frontier.cu), called at the end of every build.
void build_frontier(tc_graph& g);
// Segments of one multi-GPU part (edge range [e0,e1)) -> wsegs/csegs.
void part_segments(tc_graph& g, uint64_t e0, uint64_t e1, DBuf<uint4>& wsegs, uint64_t& nw, DBuf<uint4>& csegs,
                   uint64_t& nc);

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
// Degree-weighted oriented-edge ranges of a P-way split (cached per handle).
const std::vector<uint64_t>& partition_bounds(tc_graph& g, uint32_t parts);

// Generators (gen.cu).
uint64_t gen_num_edges(int kind, int scale, int param);
void generate(int kind, int scale, int param, uint32_t* d_pairs, cudaStream_t s);

}  // namespace tcb
