// test_dropin.cpp -- the C++ drop-in header (include/trimatch_gpu.hpp) used the
// way reference code uses trimatch:: (SPEC.md examples; reference behaviour
// pinned in tests/golden/known.json).  Built and run by tests/test_dropin.py.
//   test_dropin <rmat-scale> <expected-T> <expected-E>
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <stdexcept>
#include <string>

#include "trimatch_gpu.hpp"

namespace tg = trimatch_gpu;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <typename Ex, typename F>
static bool throws(F f) {
  try {
    f();
  } catch (const Ex&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// A stand-in for a reference trimatch::Graph: same accessor names.
struct RefLikeGraph {
  std::vector<std::uint64_t> off;
  std::vector<std::uint32_t> nb;
  std::uint32_t num_vertices() const { return (std::uint32_t)off.size() - 1; }
  std::uint64_t num_edges() const { return nb.size() / 2; }
  const std::vector<std::uint64_t>& row_offsets() const { return off; }
  const std::vector<std::uint32_t>& neighbor_array() const { return nb; }
};

int main(int argc, char** argv) {
  // K3
  tg::EdgeList k3{3, {{0, 1}, {0, 2}, {1, 2}}};
  tg::Graph g3 = tg::build_graph(k3);
  CHECK(g3.num_edges() == 3);
  CHECK((g3.row_offsets() == std::vector<std::uint64_t>{0, 2, 4, 6}));
  CHECK((g3.neighbor_array() == std::vector<std::uint32_t>{1, 2, 0, 2, 0, 1}));
  CHECK(tg::count_triangles(g3).count == 1);
  CHECK(g3.has_edge(0, 2) && !g3.has_edge(0, 0));
  CHECK(throws<std::out_of_range>([&] { (void)g3.has_edge(0, 3); }));

  // self-loop + mirror
  tg::BuildReport rep;
  tg::Graph g2 = tg::build_graph(tg::EdgeList{2, {{0, 0}, {0, 1}, {1, 0}}}, &rep);
  CHECK(g2.num_edges() == 1 && rep.self_loops_removed == 1 && rep.duplicate_entries_removed == 1);

  // K4 / K5 / star / path
  auto clique = [](std::uint32_t k) {
    tg::EdgeList el{k, {}};
    for (std::uint32_t a = 0; a < k; ++a)
      for (std::uint32_t b = a + 1; b < k; ++b) el.edges.push_back({a, b});
    return el;
  };
  CHECK(tg::count_triangles(tg::build_graph(clique(4))).count == 4);
  CHECK(tg::count_triangles(tg::build_graph(clique(5))).count == 10);
  auto d4 = tg::degrees(tg::build_graph(clique(4)));
  CHECK(d4.size() == 4 && d4[0] == 3 && d4[3] == 3);
  CHECK(tg::count_triangles(tg::build_graph(tg::EdgeList{5, {{0, 1}, {0, 2}, {0, 3}, {0, 4}}})).count == 0);
  CHECK(tg::count_triangles(tg::build_graph(tg::EdgeList{3, {{0, 1}, {1, 2}}})).count == 0);
  CHECK(tg::count_triangles(tg::build_graph(tg::EdgeList{0, {}})).count == 0);

  // per-vertex counts: K4 -> 3 each
  tg::MatchOptions pvo;
  pvo.per_vertex = true;
  auto r4 = tg::count_triangles(tg::build_graph(clique(4)), pvo);
  CHECK(r4.per_vertex && (*r4.per_vertex)[0] == 3 && (*r4.per_vertex)[3] == 3);

  // errors the reference throws
  CHECK(throws<std::invalid_argument>([] { tg::build_graph(tg::EdgeList{3, {{0, 5}}}); }));
  tg::MatchOptions bad;
  bad.lookahead = 3;
  CHECK(throws<std::invalid_argument>([&] { tg::count_triangles(g3, bad); }));
  std::istringstream mm("%%MatrixMarket matrix coordinate pattern general\n% c\n3 3 1\n\n1 9\n");
  bool pe = false;
  try {
    tg::parse_matrix_market(mm);
  } catch (const tg::ParseError& e) {
    pe = e.line() == 5;
  }
  CHECK(pe);
  std::istringstream ok("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 3\n1 2\n1 3\n2 3\n");
  CHECK(tg::count_triangles(tg::build_graph(tg::parse_matrix_market(ok))).count == 1);
  CHECK(throws<tg::IoError>([] { tg::parse_matrix_market_file("/nonexistent/x.mtx"); }));

  // TRIMCSR1 round trip + load_graph dispatch
  tg::write_csr_cache("/tmp/tcb200_k5.trimcsr", tg::build_graph(clique(5)));
  CHECK(tg::is_csr_cache_file("/tmp/tcb200_k5.trimcsr"));
  CHECK(tg::count_triangles(tg::load_graph("/tmp/tcb200_k5.trimcsr")).count == 10);

  // an existing reference-style Graph object, counted without conversion
  RefLikeGraph rg{{0, 2, 4, 6}, {1, 2, 0, 2, 0, 1}};
  CHECK(tg::count_triangles_csr(rg).count == 1);

  // a synthetic RMAT graph against the oracle's answer passed by the test
  if (argc >= 4) {
    const int scale = std::atoi(argv[1]);
    const std::uint64_t T = std::strtoull(argv[2], nullptr, 10), E = std::strtoull(argv[3], nullptr, 10);
    const std::uint64_t m = tc_gen_num_edges(0, scale, 16);
    std::vector<std::uint32_t> pairs(2 * m);
    tg::detail::check(tc_generate(0, scale, 16, 0, pairs.data()));
    tg::EdgeList el{1u << scale, {}};
    el.edges.resize(m);
    for (std::uint64_t i = 0; i < m; ++i) el.edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
    tg::Graph g = tg::build_graph(el);
    CHECK(g.num_edges() == E);
    CHECK(tg::count_triangles(g).count == T);
    // the Graph(n, E, offsets, nbrs) constructor route gives the same answer
    tg::Graph g_csr(g.num_vertices(), g.num_edges(), g.row_offsets(), g.neighbor_array());
    CHECK(tg::count_triangles(g_csr).count == T);
    // streamed listings through a 777-row buffer: T rows, each ascending
    std::uint64_t listed = 0, ascending = 0;
    tg::for_each_triangle_chunk(g, [&](const std::array<tg::VertexId, 3>* rows, std::size_t k) {
      CHECK(k <= 777);
      listed += k;
      for (std::size_t i = 0; i < k; ++i) ascending += rows[i][0] < rows[i][1] && rows[i][1] < rows[i][2];
    }, 777);
    CHECK(listed == T && ascending == T);

    // reference MatchStats / MatchResult shapes (matcher.hpp:35-94): levels,
    // rows_at, listings as an optional<PartialTable>
    tg::MatchOptions lo;
    lo.keep_listings = true;
    auto rl = tg::count_triangles(g, lo);
    CHECK(rl.count == T);
    CHECK(rl.listings.has_value() && rl.listings->width() == 3 && rl.listings->level() == 3);
    CHECK(rl.listings->num_rows() == T);
    std::uint64_t asc = 0;
    for (std::uint64_t i = 0; i < rl.listings->num_rows(); ++i) {
      auto row = rl.listings->row(i);
      asc += row[0] < row[1] && row[1] < row[2] && g.has_edge(row[0], row[2]);
    }
    CHECK(asc == T);
    CHECK(rl.stats.levels.size() == 2 && rl.stats.rows_at(3) == T);
    CHECK(rl.stats.levels[1].rows_in == rl.stats.levels[0].rows_out);
    CHECK(rl.stats.levels[1].edges_visited >= T && rl.stats.total_millis() > 0.0);
    CHECK(rl.stats.seed_rows > 0 && rl.stats.candidates == rl.stats.seed_rows);

    // multi-GPU through the C-ABI: 3 parts of the pivot split on device 0
    // (one NCCL allreduce over a 1-rank communicator)
    tg::MultiGpu mg({0, 0, 0});
    std::vector<tg::Graph> reps = mg.build_replicas(el);
    CHECK(reps.size() == 1);
    tg::MatchOptions mp;
    mp.per_vertex = true;
    auto rm = mg.count_triangles(reps, mp);
    auto r1 = tg::count_triangles(g, mp);
    CHECK(rm.count == T && rm.per_vertex && *rm.per_vertex == *r1.per_vertex);
    // one process per GPU, 1-rank group
    tg::Communicator comm(tg::Communicator::unique_id(), 1, 0, 0);
    CHECK(comm.count_triangles(g).count == T);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
