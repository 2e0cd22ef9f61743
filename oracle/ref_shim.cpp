// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference library
// (namespace trimatch, /root/reference/proj), compiled by oracle/Makefile into
// oracle/_ref/libtrimatch_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used by tests/ (to pin the C restatement in
// oracle.c and to generate tests/golden/), and by bench.py's --impl reference /
// cpu_baseline legs.  Every call goes through the reference's own public API:
//   build_graph          graph.hpp:73        (graph.cpp:33-85)
//   Graph ctor           graph.hpp:38-39     (graph.cpp:9-21)
//   count_triangles      matcher.hpp:128     (matcher.cpp:301-303)
//   filter_candidates    matcher.hpp:69-70   (matcher.cpp:46-87)
//   expand_level         matcher.hpp:86-89   (matcher.cpp:136-198)
//   segmented_intersect  frontier.hpp:229-231 (frontier.cpp:51-81)
//   parse_matrix_market  io.hpp:34          (io.cpp:93-159)
//   read/write_csr_cache io.hpp:39-41       (io.cpp:167-220)
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "trimatch/frontier.hpp"
#include "trimatch/graph.hpp"
#include "trimatch/io.hpp"
#include "trimatch/matcher.hpp"
#include "trimatch/query_plan.hpp"

using namespace trimatch;

namespace {
thread_local std::string g_err;

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Error codes mirror include/tcb200.h's tc_status so tests can compare them.
int map_exception() {
  try {
    throw;
  } catch (const ParseError& e) {
    g_err = e.what();
    return 7;
  } catch (const IoError& e) {
    g_err = e.what();
    return 8;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 99;
  }
}

void* dup_bytes(const void* p, size_t n) {
  void* q = std::malloc(n ? n : 1);
  if (n) std::memcpy(q, p, n);
  return q;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// trimatch::build_graph over interleaved (u,v) pairs.
int ref_build_graph(const uint32_t* pairs, uint64_t m, uint32_t n, uint64_t** offsets,
                    uint32_t** nbrs, uint64_t* num_edges, uint64_t* loops, uint64_t* dups) {
  try {
    EdgeList el;
    el.num_vertices_declared = n;
    el.edges.resize(m);
    for (uint64_t i = 0; i < m; ++i) el.edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    BuildReport rep;
    Graph g = build_graph(el, &rep);
    *offsets = (uint64_t*)dup_bytes(g.row_offsets().data(), g.row_offsets().size() * 8);
    *nbrs = (uint32_t*)dup_bytes(g.neighbor_array().data(), g.neighbor_array().size() * 4);
    *num_edges = g.num_edges();
    *loops = rep.self_loops_removed;
    *dups = rep.duplicate_entries_removed;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Opaque Graph built from CSR arrays through the public constructor.
void* ref_graph_new(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n, uint64_t num_edges) {
  try {
    std::vector<uint64_t> off(offsets, offsets + (size_t)n + 1);
    std::vector<VertexId> nb(nbrs, nbrs + 2 * num_edges);
    return new Graph(n, num_edges, std::move(off), std::move(nb));
  } catch (...) {
    map_exception();
    return nullptr;
  }
}
void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

// trimatch::count_triangles -- THE reference hot path.  per_vertex
// (nullable) is the histogram of the keep_listings rows (matcher.hpp:92).
int ref_count_triangles(void* gp, int lookahead, int workers, int keep_listings,
                        uint64_t* count, uint64_t* per_vertex, double* total_ms) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    MatchOptions opts;
    opts.lookahead = lookahead;
    opts.keep_listings = keep_listings != 0 || per_vertex != nullptr;
    opts.exec.workers = workers > 0 ? (unsigned)workers : 0u;
    MatchResult r = count_triangles(g, opts);
    *count = r.count;
    if (total_ms) *total_ms = r.stats.total_millis();
    if (per_vertex) {
      std::memset(per_vertex, 0, (size_t)g.num_vertices() * 8);
      const PartialTable& t = *r.listings;
      for (uint64_t i = 0; i < t.num_rows(); ++i)
        for (VertexId x : t.row(i)) per_vertex[x] += 1;
    }
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// trimatch::segmented_intersect over {(u,v): u<v} with above_dst_only; the
// oracle path SPEC.md:376 equates with count_triangles.  Count only; pairs are
// fed in chunks of rows so the frontier stays bounded.
int ref_segmented_intersect(void* gp, int workers, uint64_t* count) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    ExecPolicy exec;
    exec.workers = workers > 0 ? (unsigned)workers : 0u;
    IntersectOptions io;
    io.above_dst_only = true;
    uint64_t total = 0;
    const VertexId nv = g.num_vertices();
    VertexId u = 0;
    while (u < nv) {
      std::vector<EdgeItem> items;
      while (u < nv && items.size() < (1u << 22)) {
        for (VertexId v : g.neighbors(u))
          if (v > u) items.push_back(EdgeItem{u, v, 0});
        ++u;
      }
      total += segmented_intersect(g, Frontier::of_edges(std::move(items)), io, exec).total();
    }
    *count = total;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Same as above with per-vertex histogram of listings (t[u],t[v],t[w] += 1
// per listed triangle (u,v,w)).
int ref_segmented_intersect_pv(void* gp, int workers, uint64_t* count, uint64_t* per_vertex) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    ExecPolicy exec;
    exec.workers = workers > 0 ? (unsigned)workers : 0u;
    IntersectOptions io;
    io.above_dst_only = true;
    io.keep_listings = true;
    std::memset(per_vertex, 0, (size_t)g.num_vertices() * 8);
    uint64_t total = 0;
    const VertexId nv = g.num_vertices();
    VertexId u = 0;
    while (u < nv) {
      std::vector<EdgeItem> items;
      while (u < nv && items.size() < (1u << 22)) {
        for (VertexId v : g.neighbors(u))
          if (v > u) items.push_back(EdgeItem{u, v, 0});
        ++u;
      }
      std::vector<EdgeItem> keep = items;
      IntersectResult r = segmented_intersect(g, Frontier::of_edges(std::move(items)), io, exec);
      total += r.total();
      for (size_t i = 0; i < keep.size(); ++i) {
        const uint64_t c = r.counts[i];
        if (!c) continue;
        per_vertex[keep[i].src] += c;
        per_vertex[keep[i].dst] += c;
        for (uint64_t k = r.listing_offsets[i]; k < r.listing_offsets[i + 1]; ++k)
          per_vertex[r.listing_values[k]] += 1;
      }
    }
    *count = total;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// Bounded sample of count_triangles for the CPU baseline: the reference's own
// filter_candidates over the whole graph, then its expand_level for level 1
// and level 2 seeded with the given seed vertices only (the same per-row
// accept + look-ahead logic count_final_level applies, matcher.cpp:204-245,
// through the public expand_level).  Reports filter/verify ms and the level-2
// visits the reference's own LevelStats count.
// Level 2 (final) is run on every row_stride-th level-1 row, fed to
// expand_level in chunks of at most max_chunk_visits scratch entries (the
// reference's advance allocates one slot per visited edge, frontier.hpp:123,
// so a hub seed's rows cannot go through in one call).
int ref_count_sample(void* gp, const uint32_t* seeds, uint64_t nseeds, uint64_t row_stride,
                     uint64_t max_chunk_visits, int lookahead, int workers, double* filter_ms, double* l1_ms,
                     double* l2_ms, uint64_t* count, uint64_t* visits, uint64_t* l1_rows) {
  try {
    const Graph& g = *static_cast<Graph*>(gp);
    MatchOptions opts;
    opts.lookahead = lookahead;
    opts.exec.workers = workers > 0 ? (unsigned)workers : 0u;
    const QueryPlan plan = compile_plan(QueryGraph::triangle());
    auto t0 = std::chrono::steady_clock::now();
    CandidateSet c = filter_candidates(g, plan, opts.exec);
    *filter_ms = ms_since(t0);
    auto t1 = std::chrono::steady_clock::now();
    PartialTable table(3);
    table.set_level(1);
    for (uint64_t i = 0; i < nseeds; ++i) {
      if (!c.contains(seeds[i])) continue;
      table.cells().push_back(seeds[i]);
      table.cells().push_back(kInvalidVertex);
      table.cells().push_back(kInvalidVertex);
    }
    LevelStats s1;
    PartialTable l2 = expand_level(g, plan, c, table, 1, opts, &s1);
    *l1_ms = ms_since(t1);
    *l1_rows = l2.num_rows();
    if (row_stride == 0) row_stride = 1;
    uint64_t found = 0, vis = 0;
    double ms2 = 0;
    PartialTable chunk(3);
    chunk.set_level(2);
    uint64_t chunk_vis = 0;
    auto flush = [&]() {
      if (chunk.num_rows() == 0) return;
      auto t2 = std::chrono::steady_clock::now();
      LevelStats s2;
      PartialTable l3 = expand_level(g, plan, c, chunk, 2, opts, &s2);
      ms2 += ms_since(t2);
      found += l3.num_rows();
      vis += s2.edges_visited;
      chunk.cells().clear();
      chunk_vis = 0;
    };
    for (uint64_t r = 0; r < l2.num_rows(); r += row_stride) {
      auto row = l2.row(r);
      const uint64_t d = g.degree(row[0]);
      if (chunk_vis + d > max_chunk_visits) flush();
      chunk.cells().insert(chunk.cells().end(), row.begin(), row.end());
      chunk_vis += d;
    }
    flush();
    *l2_ms = ms2;
    *count = found;
    *visits = vis;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// MatrixMarket parser (io.cpp:93-159) over an in-memory buffer.
int ref_parse_matrix_market(const char* text, uint64_t len, uint32_t** pairs, uint64_t* m,
                            uint32_t* n_declared) {
  try {
    std::istringstream in(std::string(text, len));
    EdgeList el = parse_matrix_market(in);
    *m = el.edges.size();
    *n_declared = el.num_vertices_declared;
    uint32_t* p = (uint32_t*)std::malloc(el.edges.size() * 8 + 8);
    for (size_t i = 0; i < el.edges.size(); ++i) {
      p[2 * i] = el.edges[i].first;
      p[2 * i + 1] = el.edges[i].second;
    }
    *pairs = p;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

// load_graph (io.cpp:222-228): sniffs TRIMCSR1, else MatrixMarket + build.
int ref_load_graph(const char* path, uint64_t** offsets, uint32_t** nbrs, uint32_t* n,
                   uint64_t* num_edges, uint64_t* loops, uint64_t* dups) {
  try {
    BuildReport rep;
    Graph g = load_graph(path, &rep);
    *offsets = (uint64_t*)dup_bytes(g.row_offsets().data(), g.row_offsets().size() * 8);
    *nbrs = (uint32_t*)dup_bytes(g.neighbor_array().data(), g.neighbor_array().size() * 4);
    *n = g.num_vertices();
    *num_edges = g.num_edges();
    *loops = rep.self_loops_removed;
    *dups = rep.duplicate_entries_removed;
    return 0;
  } catch (...) {
    return map_exception();
  }
}

int ref_write_csr_cache(const char* path, void* gp) {
  try {
    write_csr_cache(path, *static_cast<Graph*>(gp));
    return 0;
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
