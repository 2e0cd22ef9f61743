// trimatch_gpu.hpp -- C++ drop-in for the reference's triangle-counting entry
// points (namespace trimatch, /root/reference/proj/include/trimatch/*.hpp),
// header-only over the C-ABI of libtcb200.so (tcb200.h).
//
//   reference                                   here (namespace trimatch_gpu)
//   EdgeList            graph.hpp:16-19         EdgeList (same fields)
//   BuildReport         graph.hpp:22-25         BuildReport (same fields)
//   Graph               graph.hpp:35-66         Graph (device-resident, same accessors)
//   build_graph         graph.hpp:73            build_graph
//   degrees             graph.hpp:75            degrees
//   ParseError/IoError  io.hpp:13-27            ParseError / IoError
//   parse_matrix_market io.hpp:34-35            parse_matrix_market[_file]
//   write/read_csr_cache, is_csr_cache_file     same names (io.hpp:39-41)
//   load_graph          io.hpp:45               load_graph
//   PartialTable        matcher.hpp:35-58       PartialTable (listings: width 3)
//   LevelStats/MatchStats matcher.hpp:60-82     LevelStats / MatchStats (same fields)
//   MatchOptions/Result matcher.hpp:84-94       MatchOptions / MatchResult (+ per_vertex)
//   count_triangles     matcher.hpp:128         count_triangles
//   (multi-GPU)         --                      MultiGpu (tc_count_multi), Communicator
//                                               (tc_count_allreduce)
//
// Errors map back to the exception types the reference throws:
// TC_EINVAL -> std::invalid_argument, TC_ERANGE -> std::out_of_range,
// TC_EPARSE -> ParseError, TC_EIO -> IoError, others -> std::runtime_error.
// A reference user switches by replacing `trimatch::` with `trimatch_gpu::`;
// an existing trimatch::Graph can be counted without conversion through
// count_triangles_csr(g) (any type with num_vertices/num_edges/row_offsets/
// neighbor_array).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <istream>
#include <iterator>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <array>
#include <vector>

#include "tcb200.h"

namespace trimatch_gpu {

using VertexId = std::uint32_t;
inline constexpr VertexId kInvalidVertex = static_cast<VertexId>(-1);

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& message, std::uint64_t line)
      : std::runtime_error(message + " (line " + std::to_string(line) + ")"), line_(line) {}
  // Built from the library's already-formatted "... (line N)" message.
  explicit ParseError(const std::string& formatted) : std::runtime_error(formatted), line_(0) {
    const auto p = formatted.rfind("(line ");
    if (p != std::string::npos) line_ = std::strtoull(formatted.c_str() + p + 6, nullptr, 10);
  }
  std::uint64_t line() const { return line_; }

 private:
  std::uint64_t line_;
};

class IoError : public std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(tc_status s) {
  if (s == TC_OK) return;
  const std::string msg = tc_last_error();
  switch (s) {
    case TC_EINVAL: throw std::invalid_argument(msg);
    case TC_ERANGE: throw std::out_of_range(msg);
    case TC_EPARSE: throw ParseError(msg);
    case TC_EIO: throw IoError(msg);
    default: throw std::runtime_error("tcb200: " + msg);
  }
}
struct GraphDeleter {
  void operator()(tc_graph* g) const { tc_graph_destroy(g); }
};
}  // namespace detail

struct EdgeList {
  VertexId num_vertices_declared = 0;
  std::vector<std::pair<VertexId, VertexId>> edges;
};

struct BuildReport {
  std::uint64_t self_loops_removed = 0;
  std::uint64_t duplicate_entries_removed = 0;
};

// Immutable undirected simple graph, resident on a B200 as the
// (deg,id)-oriented CSR + in-edge index.  Copies share the device handle; like
// the reference Graph (graph.hpp:33-34) it may be used from several threads:
// the library serialises calls on one handle (a per-handle lock around its
// count scratch).  The symmetric CSR the accessors expose is materialised on
// first use.
class Graph {
 public:
  Graph() = default;
  explicit Graph(tc_graph* h) : h_(h, detail::GraphDeleter{}) { detail::check(tc_graph_get_info(h, &info_)); }
  // The reference constructor signature (graph.hpp:38-39): upload a CSR.
  Graph(VertexId num_vertices, std::uint64_t num_edges, std::vector<std::uint64_t> row_offsets,
        std::vector<VertexId> neighbors, int device = 0) {
    if (row_offsets.size() != static_cast<std::size_t>(num_vertices) + 1 || row_offsets.back() != 2 * num_edges ||
        neighbors.size() != 2 * num_edges)
      throw std::invalid_argument("Graph: inconsistent CSR arrays");
    tc_graph* h = nullptr;
    detail::check(tc_graph_from_csr(row_offsets.data(), neighbors.data(), num_vertices, num_edges, device, &h));
    h_.reset(h, detail::GraphDeleter{});
    detail::check(tc_graph_get_info(h, &info_));
    std::call_once(lazy_->once, [&] {
      lazy_->csr.off = std::move(row_offsets);
      lazy_->csr.nbrs = std::move(neighbors);
    });
  }

  VertexId num_vertices() const { return info_.num_vertices; }
  std::uint64_t num_edges() const { return info_.num_edges; }
  std::uint32_t degree(VertexId u) const {
    const auto& o = csr().off;
    return static_cast<std::uint32_t>(o[u + 1] - o[u]);
  }
  std::span<const VertexId> neighbors(VertexId u) const {
    const auto& c = csr();
    return {c.nbrs.data() + c.off[u], c.nbrs.data() + c.off[u + 1]};
  }
  bool has_edge(VertexId u, VertexId v) const {
    if (u >= num_vertices() || v >= num_vertices())
      throw std::out_of_range("has_edge: vertex id " + std::to_string(u >= num_vertices() ? u : v) +
                              " out of range");
    auto nb = neighbors(u);
    auto it = std::lower_bound(nb.begin(), nb.end(), v);
    return it != nb.end() && *it == v;
  }
  const std::vector<std::uint64_t>& row_offsets() const { return csr().off; }
  const std::vector<VertexId>& neighbor_array() const { return csr().nbrs; }

  tc_graph* handle() const { return h_.get(); }
  const tc_graph_info& info() const { return info_; }

 private:
  struct Csr {
    std::vector<std::uint64_t> off;
    std::vector<VertexId> nbrs;
  };
  struct Lazy {
    std::once_flag once;
    Csr csr;
  };
  const Csr& csr() const {
    std::call_once(lazy_->once, [this] {
      Csr& c = lazy_->csr;
      c.off.resize(static_cast<std::size_t>(num_vertices()) + 1);
      c.nbrs.resize(2 * num_edges());
      detail::check(tc_graph_export_csr(h_.get(), c.off.data(), c.nbrs.data()));
    });
    return lazy_->csr;
  }
  std::shared_ptr<tc_graph> h_;
  tc_graph_info info_{};
  std::shared_ptr<Lazy> lazy_ = std::make_shared<Lazy>();
};

using DegreeArray = std::vector<std::uint32_t>;

inline Graph build_graph(const EdgeList& edges, BuildReport* report = nullptr, int device = 0) {
  static_assert(sizeof(std::pair<VertexId, VertexId>) == 8, "EdgeList pairs must be two packed u32");
  tc_graph* h = nullptr;
  tc_build_report rep{};
  detail::check(tc_graph_build(reinterpret_cast<const std::uint32_t*>(edges.edges.data()), edges.edges.size(),
                               edges.num_vertices_declared, device, &h, &rep));
  if (report) {
    report->self_loops_removed = rep.self_loops_removed;
    report->duplicate_entries_removed = rep.duplicate_entries_removed;
  }
  return Graph(h);
}

inline DegreeArray degrees(const Graph& g) {
  DegreeArray d(g.num_vertices());
  detail::check(tc_graph_degrees(g.handle(), d.data()));
  return d;
}

// ---- io ------------------------------------------------------------------------

inline EdgeList parse_matrix_market(std::istream& in) {
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::uint32_t* pairs = nullptr;
  std::uint64_t m = 0;
  std::uint32_t n = 0;
  detail::check(tc_parse_matrix_market(text.data(), text.size(), &pairs, &m, &n));
  EdgeList el;
  el.num_vertices_declared = n;
  el.edges.resize(m);
  for (std::uint64_t i = 0; i < m; ++i) el.edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
  tc_free(pairs);
  return el;
}

inline EdgeList parse_matrix_market_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open '" + path + "' for reading");
  return parse_matrix_market(in);
}

inline bool is_csr_cache_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  char magic[8] = {};
  in.read(magic, 8);
  return in.gcount() == 8 && std::string(magic, 8) == "TRIMCSR1";
}

inline Graph read_csr_cache(const std::string& path, int device = 0) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open '" + path + "' for reading");
  std::string bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  tc_graph* h = nullptr;
  detail::check(tc_csr_cache_to_graph(bytes.data(), bytes.size(), device, &h));
  return Graph(h);
}

inline void write_csr_cache(const std::string& path, const Graph& g) {
  // the TRIMCSR1 image (io.cpp:167-177 layout) assembled by the library
  std::uint64_t len = 0;
  detail::check(tc_graph_csr_cache_size(g.handle(), &len));
  std::vector<std::uint64_t> buf((len + 7) / 8);  // 8-byte aligned
  detail::check(tc_graph_write_csr_cache(g.handle(), buf.data()));
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot open '" + path + "' for writing");
  out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(len));
  if (!out) throw IoError("write failed for '" + path + "'");
}

inline Graph load_graph(const std::string& path, BuildReport* report = nullptr, int device = 0) {
  if (is_csr_cache_file(path)) {
    if (report) *report = BuildReport{};
    return read_csr_cache(path, device);
  }
  // MatrixMarket: entries tokenized and built on the device
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open '" + path + "' for reading");
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  tc_graph* h = nullptr;
  tc_build_report rep{};
  detail::check(tc_graph_load_matrix_market(text.data(), text.size(), device, &h, &rep));
  if (report) {
    report->self_loops_removed = rep.self_loops_removed;
    report->duplicate_entries_removed = rep.duplicate_entries_removed;
  }
  return Graph(h);
}

// ---- matcher -------------------------------------------------------------------

struct ExecPolicy {
  unsigned workers = 0;  // accepted for source compatibility; the GPU ignores it
};

// matcher.hpp:35-58: fixed-width table of (partial) embeddings.  Here it holds
// the keep_listings rows: width 3, level 3, one triangle per row, ids ascending.
class PartialTable {
 public:
  explicit PartialTable(std::uint32_t width) : width_(width) {}

  std::uint32_t width() const { return width_; }
  std::uint32_t level() const { return level_; }
  std::uint64_t num_rows() const { return width_ == 0 ? 0 : cells_.size() / width_; }

  std::span<const VertexId> row(std::uint64_t r) const { return {cells_.data() + r * width_, width_}; }
  std::span<const VertexId> row_prefix(std::uint64_t r) const { return {cells_.data() + r * width_, level_}; }

  std::vector<VertexId>& cells() { return cells_; }
  const std::vector<VertexId>& cells() const { return cells_; }
  void set_level(std::uint32_t level) { level_ = level; }

 private:
  std::uint32_t width_;
  std::uint32_t level_ = 0;
  std::vector<VertexId> cells_;
};

// matcher.hpp:60-67 / :69-82.  On the GPU path (MatchOptions::level_stats):
//   candidates = seed_rows = pivots (d+(v) > 0 with in-edges; the orientation
//                replaces the 2-core peel, so peel_rounds = 0)
//   levels[0]  = the level-1 rows (u, w): rows_in = seeds, edges_visited =
//                |E| oriented edges, rows_out = in-edges with a non-empty suffix
//   levels[1]  = the final level: rows_in = levels[0].rows_out,
//                edges_visited = candidate wedges probed, rows_out = count
//   filter_millis = the count plan, verify_millis = advance + join + reduce
struct LevelStats {
  std::uint64_t rows_in = 0;
  std::uint64_t edges_visited = 0;
  std::uint64_t rows_out = 0;
  std::uint64_t rows_masked = 0;
  std::uint64_t lookahead_pruned = 0;
  double millis = 0.0;
};

struct MatchStats {
  double filter_millis = 0.0;
  double verify_millis = 0.0;
  std::uint64_t candidates = 0;
  std::uint32_t peel_rounds = 0;
  std::uint64_t seed_rows = 0;
  std::vector<LevelStats> levels;

  double total_millis() const { return filter_millis + verify_millis; }
  std::uint64_t rows_at(std::uint32_t slots) const {
    return slots <= 1 ? seed_rows : levels[slots - 2].rows_out;
  }
};

struct MatchOptions {
  int lookahead = 2;           // validated (0..2); count-neutral on the GPU path
  bool keep_listings = false;  // listings from the GPU listing kernel (tc_list_triangles)
  ExecPolicy exec{};
  bool per_vertex = false;     // GPU extension: triangles per vertex
  bool level_stats = true;     // GPU extension: fill stats.levels (one extra pass)
};

struct MatchResult {
  std::uint64_t count = 0;
  std::optional<PartialTable> listings;  // keep_listings: rows u < w < x, order unspecified
  MatchStats stats;
  std::optional<std::vector<std::uint64_t>> per_vertex;  // GPU extension
};

namespace detail {
inline tc_count_opts count_opts(const MatchOptions& opts) {
  if (opts.lookahead < 0 || opts.lookahead > 2) throw std::invalid_argument("lookahead must be 0, 1, or 2");
  tc_count_opts o{};
  o.lookahead = opts.lookahead;
  o.sync = 1;
  o.work_counters = opts.level_stats ? 1 : 0;
  return o;
}
inline void fill_stats(MatchResult& r, const tc_count_stats& st, std::uint64_t num_edges, bool level_stats) {
  r.stats.filter_millis = st.frontier_ms;
  r.stats.verify_millis = st.join_ms + st.reduce_ms;
  if (!level_stats) return;
  r.stats.candidates = r.stats.seed_rows = st.pivots;
  r.stats.peel_rounds = 0;
  LevelStats l1, l2;
  l1.rows_in = st.pivots;
  l1.edges_visited = num_edges;
  l1.rows_out = st.items;
  l1.millis = st.frontier_ms;
  l2.rows_in = st.items;
  l2.edges_visited = st.wedges;
  l2.rows_out = r.count;
  l2.millis = st.join_ms;
  r.stats.levels = {l1, l2};
}
inline PartialTable listings(tc_graph* h) {
  std::uint64_t T = 0;
  check(tc_list_triangles(h, nullptr, 0, &T));
  PartialTable t(3);
  t.cells().resize(3 * T);
  std::uint64_t T2 = 0;
  if (T) check(tc_list_triangles(h, t.cells().data(), T, &T2));
  t.set_level(3);
  return t;
}
}  // namespace detail

inline MatchResult count_triangles(const Graph& g, const MatchOptions& opts = {}) {
  tc_count_opts o = detail::count_opts(opts);
  MatchResult r;
  tc_count_stats st{};
  std::vector<std::uint64_t> pv;
  if (opts.per_vertex) pv.resize(g.num_vertices());
  detail::check(tc_count(g.handle(), &o, &r.count, opts.per_vertex ? pv.data() : nullptr, &st));
  if (opts.per_vertex) r.per_vertex = std::move(pv);
  detail::fill_stats(r, st, g.num_edges(), opts.level_stats);
  if (opts.keep_listings) r.listings = detail::listings(g.handle());
  return r;
}

// ---- multi-GPU (tcb200.h tc_multi_* / tc_comm_*) --------------------------------

// One process driving several B200s: part p of the degree-weighted pivot
// split runs on devices[p] against its replica; ONE NCCL allreduce combines
// the parts.  A device may repeat (its parts run back to back).
class MultiGpu {
 public:
  explicit MultiGpu(std::vector<int> devices) : devices_(std::move(devices)) {
    tc_multi* m = nullptr;
    detail::check(tc_multi_create(devices_.data(), static_cast<int>(devices_.size()), &m));
    m_.reset(m, [](tc_multi* x) { tc_multi_destroy(x); });
  }
  const std::vector<int>& devices() const { return devices_; }

  // One replica per distinct device, built from the same edge list.
  std::vector<Graph> build_replicas(const EdgeList& edges, BuildReport* report = nullptr) const {
    std::vector<Graph> out;
    std::vector<int> seen;
    for (int d : devices_) {
      if (std::find(seen.begin(), seen.end(), d) != seen.end()) continue;
      seen.push_back(d);
      out.push_back(build_graph(edges, report, d));
    }
    return out;
  }

  // replicas: one Graph per distinct device (any order); parts are mapped to
  // the replica on their device.
  MatchResult count_triangles(const std::vector<Graph>& replicas, const MatchOptions& opts = {}) const {
    std::vector<tc_graph*> hs;
    for (int d : devices_) {
      tc_graph* h = nullptr;
      for (const Graph& g : replicas)
        if (g.info().device == d) h = g.handle();
      if (!h) throw std::invalid_argument("MultiGpu: no replica on device " + std::to_string(d));
      hs.push_back(h);
    }
    tc_count_opts o = detail::count_opts(opts);
    o.work_counters = 0;
    MatchResult r;
    tc_count_stats st{};
    std::vector<std::uint64_t> pv;
    if (opts.per_vertex) pv.resize(replicas.at(0).num_vertices());
    detail::check(tc_count_multi(m_.get(), hs.data(), &o, &r.count, opts.per_vertex ? pv.data() : nullptr, &st));
    if (opts.per_vertex) r.per_vertex = std::move(pv);
    detail::fill_stats(r, st, replicas.at(0).num_edges(), false);
    if (opts.keep_listings) r.listings = detail::listings(hs[0]);
    return r;
  }

 private:
  std::vector<int> devices_;
  std::shared_ptr<tc_multi> m_;
};

// One rank of a one-process-per-GPU group; the 128-byte id travels through
// the host framework (MPI, a TCP store, ...): rank 0 calls unique_id().
class Communicator {
 public:
  using Id = std::array<unsigned char, TC_COMM_ID_BYTES>;
  static Id unique_id() {
    Id id{};
    detail::check(tc_comm_unique_id(id.data()));
    return id;
  }
  Communicator(const Id& id, int nranks, int rank, int device) {
    tc_comm* c = nullptr;
    detail::check(tc_comm_init_rank(id.data(), nranks, rank, device, &c));
    c_.reset(c, [](tc_comm* x) { tc_comm_destroy(x); });
  }
  // This rank's share + the allreduce: every rank gets the whole result.
  MatchResult count_triangles(const Graph& g, const MatchOptions& opts = {}) const {
    tc_count_opts o = detail::count_opts(opts);
    o.work_counters = 0;
    MatchResult r;
    tc_count_stats st{};
    std::vector<std::uint64_t> pv;
    if (opts.per_vertex) pv.resize(g.num_vertices());
    detail::check(tc_count_allreduce(c_.get(), g.handle(), &o, &r.count, opts.per_vertex ? pv.data() : nullptr, &st));
    if (opts.per_vertex) r.per_vertex = std::move(pv);
    detail::fill_stats(r, st, g.num_edges(), false);
    if (opts.keep_listings) r.listings = detail::listings(g.handle());
    return r;
  }

 private:
  std::shared_ptr<tc_comm> c_;
};

// Streamed listings: calls sink(const std::array<VertexId, 3>* rows, size_t k)
// with chunks of at most max_rows triangles whose union is the full listing,
// walking the oriented edges range by range with one bounded host buffer
// (tc_list_triangles_range); a range that overflows is halved and re-listed.
template <typename Sink>
void for_each_triangle_chunk(Graph& g, Sink&& sink, std::size_t max_rows = std::size_t(1) << 22) {
  if (max_rows == 0) throw std::invalid_argument("for_each_triangle_chunk: max_rows must be >= 1");
  std::vector<std::array<VertexId, 3>> buf(max_rows);
  tc_graph_info info{};
  detail::check(tc_graph_get_info(g.handle(), &info));
  const std::uint64_t E = info.num_edges;
  std::uint64_t e = 0, span = E < (1u << 16) ? (E ? E : 1) : (1u << 16);
  while (e < E) {
    const std::uint64_t b = std::min<std::uint64_t>(E, e + span);
    std::uint64_t T = 0;
    detail::check(tc_list_triangles_range(g.handle(), e, b, reinterpret_cast<VertexId*>(buf.data()), max_rows, &T));
    if (T > max_rows) {
      if (b - e == 1) throw std::invalid_argument("for_each_triangle_chunk: one edge lists more than max_rows");
      span = std::max<std::uint64_t>(1, (b - e) / 2);
      continue;
    }
    if (T) sink(static_cast<const std::array<VertexId, 3>*>(buf.data()), static_cast<std::size_t>(T));
    e = b;
    if (2 * T <= max_rows) span *= 2;
  }
}

// Count an existing reference-style graph object (trimatch::Graph or anything
// exposing the same accessors) without converting it by hand.
template <typename G>
MatchResult count_triangles_csr(const G& g, const MatchOptions& opts = {}, int device = 0) {
  tc_graph* h = nullptr;
  detail::check(tc_graph_from_csr(g.row_offsets().data(), g.neighbor_array().data(), g.num_vertices(),
                                  g.num_edges(), device, &h));
  Graph dg(h);
  return count_triangles(dg, opts);
}

}  // namespace trimatch_gpu
