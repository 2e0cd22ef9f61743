// capi.cu -- the extern "C" boundary of libtcb200.so (include/tcb200.h).
// Every entry point catches library errors and maps them to tc_status; no
// C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>

#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "graph.cuh"
#include "io_host.h"

namespace {

thread_local std::string g_last_error;

tc_status set_error(tc_status c, const std::string& m) {
  g_last_error = m;
  return c;
}

#define TC_API_TRY try {
#define TC_API_CATCH                                                        \
  }                                                                         \
  catch (const tcb::Error& e) {                                             \
    return set_error(e.code, e.what());                                     \
  }                                                                         \
  catch (const tcb::IoFail& e) {                                            \
    return set_error(e.code, e.what());                                     \
  }                                                                         \
  catch (const std::bad_alloc&) {                                           \
    return set_error(TC_ENOMEM, "host allocation failed");                  \
  }                                                                         \
  catch (const std::exception& e) {                                         \
    return set_error(TC_ECUDA, e.what());                                   \
  }

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  const cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    if (getenv("TCB_ALLOC_DEBUG")) fprintf(stderr, "[tcb] cudaPointerGetAttributes: %s\n", cudaGetErrorString(e));
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Input view: a device pointer as-is, or a host buffer staged to the device.
template <typename T>
struct DevIn {
  const T* p = nullptr;
  tcb::DBuf<T> staged;
  bool host() const { return staged.get() != nullptr; }
  DevIn(const T* src, uint64_t count, cudaStream_t s) {
    if (count == 0 || is_device_ptr(src)) {
      p = src;
      return;
    }
    staged.alloc(count, s);
    tcb::copy_h2d(staged.get(), src, count * sizeof(T), s);
    p = staged.get();
  }
};

// Output view: a device pointer as-is, or a device temporary copied back to
// the host buffer by finish().
template <typename T>
struct DevOut {
  T* host = nullptr;
  T* p = nullptr;
  uint64_t count = 0;
  tcb::DBuf<T> tmp;
  DevOut(T* dst, uint64_t cnt, cudaStream_t s) : count(cnt) {
    if (!dst) return;
    if (is_device_ptr(dst)) {
      p = dst;
    } else {
      host = dst;
      tmp.alloc(cnt ? cnt : 1, s);
      p = tmp.get();
    }
  }
  void finish(cudaStream_t s) {
    if (host && count) tcb::copy_d2h(host, p, count * sizeof(T), s);
  }
};

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    TC_CUDA(cudaGetDevice(&prev));
    TC_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

tcb::PhaseLog::PhaseLog(cudaStream_t st) : s(st) {
  const char* e = getenv("TCB_PHASES");
  on = e && *e == '1';
  mark("start");
}
void tcb::PhaseLog::mark(const char* what) {
  if (!on || n >= kMax) return;
  cudaEventCreate(&ev[n]);
  cudaEventRecord(ev[n], s);
  name[n++] = what;
}
tcb::PhaseLog::~PhaseLog() {
  if (!on || n == 0) return;
  cudaEventSynchronize(ev[n - 1]);
  for (int i = 1; i < n; ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
    fprintf(stderr, "[tcb] %-22s %9.3f ms\n", name[i], ms);
  }
  for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
}

namespace {

tc_graph* new_handle(int device) {
  auto* g = new tc_graph();
  g->device = device;
  TC_CUDA(cudaStreamCreateWithFlags(&g->own_stream, cudaStreamNonBlocking));
  g->stream = g->own_stream;
  return g;
}

void destroy_handle(tc_graph* g) {
  if (!g) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(g->device);
  {
    // the handle's buffers were used on g->stream (possibly a caller's stream
    // that is gone by now): drain the device, then free on the own stream
    cudaDeviceSynchronize();
    cudaStream_t s = g->own_stream;
    auto rel = [s](auto& b) {  // every buffer goes back on the own stream (a caller's may be gone)
      b.s = s;
      b.release();
    };
    rel(g->off);
    rel(g->col);
    rel(g->src);
    rel(g->deg);
    rel(g->id_of);
    rel(g->rank_of);
    rel(g->colH);
    rel(g->offH);
    rel(g->inoff);
    rel(g->irec);
    rel(g->rowd);
    rel(g->cbits);
    rel(g->dine);
    rel(g->dsoff);
    rel(g->drow);
    rel(g->dseg);
    for (auto& b : g->part_kr) rel(b);
    g->part_kr.clear();
    for (auto& sc : g->scratch) sc.release(s);
    cudaStreamSynchronize(s);
  }
  if (g->own_stream) cudaStreamDestroy(g->own_stream);
  if (g->hi_stream) cudaStreamDestroy(g->hi_stream);
  if (g->lo_stream) cudaStreamDestroy(g->lo_stream);
  for (cudaEvent_t e : {g->fork_ev, g->join_hi, g->join_lo})
    if (e) cudaEventDestroy(e);
  delete g;
  cudaSetDevice(prev);
}

struct Timer {
  cudaEvent_t a, b;
  cudaStream_t s;
  explicit Timer(cudaStream_t st) : s(st) {
    TC_CUDA(cudaEventCreate(&a));
    TC_CUDA(cudaEventCreate(&b));
    TC_CUDA(cudaEventRecord(a, s));
  }
  double stop() {
    TC_CUDA(cudaEventRecord(b, s));
    TC_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  }
  ~Timer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

}  // namespace

extern "C" {

int tc_abi_version(void) { return TCB200_ABI_VERSION; }

const char* tc_last_error(void) { return g_last_error.c_str(); }

void tc_free(void* p) { std::free(p); }

uint64_t tc_release_cached_memory(int device) { return tcb::release_cached(device); }

tc_status tc_graph_build(const uint32_t* pairs, uint64_t m, uint32_t n_declared, int device, tc_graph** out,
                         tc_build_report* report) {
  if (!out) return set_error(TC_EINVAL, "tc_graph_build: out is NULL");
  if (m && !pairs) return set_error(TC_EINVAL, "tc_graph_build: pairs is NULL");
  tc_graph* g = nullptr;
  TC_API_TRY
  DeviceGuard dg(device);
  g = new_handle(device);
  try {
    Timer t(g->stream);
    DevIn<uint32_t> in(pairs, 2 * m, g->stream);
    tc_build_report rep{};
    tcb::build_from_pairs(*g, in.p, m, n_declared, &rep);
    g->build_ms = t.stop();
    if (report) *report = rep;
  } catch (...) {
    destroy_handle(g);
    throw;
  }
  *out = g;
  return TC_OK;
  TC_API_CATCH
}

namespace {
tc_status from_csr_impl(const uint64_t* row_offsets, const uint32_t* neighbors, uint32_t n, uint64_t num_edges,
                        int device, tc_graph** out, bool strict) {
  tc_graph* g = nullptr;
  TC_API_TRY
  DeviceGuard dg(device);
  g = new_handle(device);
  try {
    Timer t(g->stream);
    tcb::PhaseLog pl(g->stream);
    DevIn<uint64_t> off(row_offsets, (uint64_t)n + 1, g->stream);
    const uint64_t total = 2 * num_edges;
    if (total == 0 || is_device_ptr(neighbors)) {
      pl.mark("csr_h2d");
      tcb::build_from_csr(*g, off.p, neighbors, n, num_edges, strict);
    } else {
      // host neighbours: streamed in by the build, behind the orientation pass
      tcb::DBuf<uint32_t> nb(total, g->stream);
      const tcb::CsrFeed feed{neighbors, off.host() ? row_offsets : nullptr, nb.get()};
      pl.mark("csr_h2d_offsets");
      tcb::build_from_csr(*g, off.p, nb.get(), n, num_edges, strict, &feed);
    }
    g->build_ms = t.stop();
  } catch (...) {
    destroy_handle(g);
    throw;
  }
  *out = g;
  return TC_OK;
  TC_API_CATCH
}
}  // namespace

tc_status tc_graph_from_csr(const uint64_t* row_offsets, const uint32_t* neighbors, uint32_t n,
                            uint64_t num_edges, int device, tc_graph** out) {
  if (!out) return set_error(TC_EINVAL, "tc_graph_from_csr: out is NULL");
  if (!row_offsets || (num_edges && !neighbors)) return set_error(TC_EINVAL, "tc_graph_from_csr: NULL array");
  return from_csr_impl(row_offsets, neighbors, n, num_edges, device, out, false);
}

tc_status tc_graph_get_info(const tc_graph* g, tc_graph_info* info) {
  if (!g || !info) return set_error(TC_EINVAL, "tc_graph_get_info: NULL argument");
  info->num_vertices = g->n;
  info->num_edges = g->E;
  info->max_degree = g->max_deg;
  info->max_out_degree = g->max_dplus;
  info->device = g->device;
  info->build_ms = g->build_ms;
  info->core_ranks = g->core_words ? g->n - g->cb : 0;
  info->dense_rows = g->ndense;
  return TC_OK;
}

tc_status tc_graph_export_csr(tc_graph* g, uint64_t* row_offsets, uint32_t* neighbors) {
  if (!g || !row_offsets || (g->E && !neighbors)) return set_error(TC_EINVAL, "tc_graph_export_csr: NULL argument");
  TC_API_TRY
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  DevOut<uint64_t> off(row_offsets, (uint64_t)g->n + 1, g->stream);
  DevOut<uint32_t> nb(neighbors, 2 * g->E, g->stream);
  tcb::export_csr(*g, off.p, nb.p);
  off.finish(g->stream);
  nb.finish(g->stream);
  TC_CUDA(cudaStreamSynchronize(g->stream));
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_graph_degrees(tc_graph* g, uint32_t* degrees) {
  if (!g || (g->n && !degrees)) return set_error(TC_EINVAL, "tc_graph_degrees: NULL argument");
  TC_API_TRY
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  DevOut<uint32_t> d(degrees, g->n, g->stream);
  tcb::export_degrees(*g, d.p);
  d.finish(g->stream);
  TC_CUDA(cudaStreamSynchronize(g->stream));
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_graph_set_stream(tc_graph* g, void* stream) {
  if (!g) return set_error(TC_EINVAL, "tc_graph_set_stream: NULL graph");
  std::lock_guard<std::mutex> lk(g->mu);
  g->stream = stream ? static_cast<cudaStream_t>(stream) : g->own_stream;
  return TC_OK;
}

void tc_graph_destroy(tc_graph* g) { destroy_handle(g); }

tc_status tc_count(tc_graph* g, const tc_count_opts* opts, uint64_t* total, uint64_t* per_vertex,
                   tc_count_stats* stats) {
  if (!g || !total) return set_error(TC_EINVAL, "tc_count: NULL argument");
  tc_count_opts o{};
  if (opts) o = *opts;
  if (o.lookahead < 0 || o.lookahead > 2) return set_error(TC_EINVAL, "lookahead must be 0, 1, or 2");
  if (o.keep_listings) return set_error(TC_EUNSUPPORTED, "keep_listings is not supported on the GPU path");
  if (o.part_count > 1 && o.part_index >= o.part_count)
    return set_error(TC_EINVAL, "tc_count: part_index must be < part_count");
  TC_API_TRY
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  DevOut<uint64_t> t(total, 1, g->stream);
  DevOut<uint64_t> pv(per_vertex, g->n, g->stream);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  tcb::count_triangles(*g, o, t.p, per_vertex ? pv.p : nullptr, stats);
  t.finish(g->stream);
  pv.finish(g->stream);
  if (o.sync || t.host || pv.host || stats) TC_CUDA(cudaStreamSynchronize(g->stream));
  return TC_OK;
  TC_API_CATCH
}

namespace {
tc_status check_count_opts(const tc_count_opts& o) {
  if (o.lookahead < 0 || o.lookahead > 2) return set_error(TC_EINVAL, "lookahead must be 0, 1, or 2");
  if (o.keep_listings) return set_error(TC_EUNSUPPORTED, "keep_listings is not supported on the GPU path");
  return TC_OK;
}
}  // namespace

tc_status tc_comm_unique_id(void* id) {
  if (!id) return set_error(TC_EINVAL, "tc_comm_unique_id: NULL id");
  TC_API_TRY
  tcb::comm_unique_id(id);
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_comm_init_rank(const void* id, int nranks, int rank, int device, tc_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(TC_EINVAL, "tc_comm_init_rank: bad argument");
  TC_API_TRY
  *out = tcb::comm_init_rank(id, nranks, rank, device);
  return TC_OK;
  TC_API_CATCH
}

void tc_comm_destroy(tc_comm* comm) { tcb::comm_destroy(comm); }

tc_status tc_count_allreduce(tc_comm* comm, tc_graph* g, const tc_count_opts* opts, uint64_t* total,
                             uint64_t* per_vertex, tc_count_stats* stats) {
  if (!comm || !g || !total) return set_error(TC_EINVAL, "tc_count_allreduce: NULL argument");
  tc_count_opts o{};
  if (opts) o = *opts;
  if (tc_status st = check_count_opts(o)) return st;
  TC_API_TRY
  DeviceGuard dg(g->device);
  DevOut<uint64_t> t(total, 1, g->stream);
  DevOut<uint64_t> pv(per_vertex, g->n, g->stream);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  tcb::count_allreduce(comm, *g, o, t.p, per_vertex ? pv.p : nullptr, stats);
  t.finish(g->stream);
  pv.finish(g->stream);
  if (o.sync || t.host || pv.host || stats) TC_CUDA(cudaStreamSynchronize(g->stream));
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_multi_create(const int* devices, int nparts, tc_multi** out) {
  if (!devices || nparts < 1 || !out) return set_error(TC_EINVAL, "tc_multi_create: bad argument");
  TC_API_TRY
  *out = tcb::multi_create(devices, nparts);
  return TC_OK;
  TC_API_CATCH
}

void tc_multi_destroy(tc_multi* m) { tcb::multi_destroy(m); }

tc_status tc_count_multi(tc_multi* m, tc_graph* const* graphs, const tc_count_opts* opts, uint64_t* total,
                         uint64_t* per_vertex, tc_count_stats* stats) {
  if (!m || !graphs || !total) return set_error(TC_EINVAL, "tc_count_multi: NULL argument");
  const int P = tcb::multi_parts(m);
  for (int p = 0; p < P; ++p)
    if (!graphs[p]) return set_error(TC_EINVAL, "tc_count_multi: NULL graph");
  tc_count_opts o{};
  if (opts) o = *opts;
  if (tc_status st = check_count_opts(o)) return st;
  TC_API_TRY
  tc_graph* g0 = graphs[0];
  DeviceGuard dg(g0->device);
  DevOut<uint64_t> t(total, 1, g0->stream);
  DevOut<uint64_t> pv(per_vertex, g0->n, g0->stream);
  if (stats) std::memset(stats, 0, sizeof(*stats));
  tcb::count_multi(m, graphs, o, t.p, per_vertex ? pv.p : nullptr, stats);
  t.finish(g0->stream);
  pv.finish(g0->stream);
  TC_CUDA(cudaStreamSynchronize(g0->stream));
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_partition_bounds(tc_graph* g, uint32_t parts, uint64_t* bounds) {
  if (!g || !bounds || parts == 0) return set_error(TC_EINVAL, "tc_partition_bounds: bad argument");
  TC_API_TRY
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  const std::vector<uint64_t>& b = tcb::partition_bounds(*g, parts);
  std::memcpy(bounds, b.data(), ((size_t)parts + 1) * sizeof(uint64_t));
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_parse_matrix_market(const char* text, uint64_t len, uint32_t** pairs, uint64_t* m,
                                 uint32_t* n_declared) {
  if (!pairs || !m || !n_declared || (len && !text)) return set_error(TC_EINVAL, "tc_parse_matrix_market: NULL argument");
  TC_API_TRY
  std::vector<uint32_t> v;
  uint32_t n = 0;
  tcb::parse_matrix_market(text, len, v, n);
  uint32_t* p = static_cast<uint32_t*>(std::malloc(v.size() * sizeof(uint32_t) + 8));
  if (!p) return set_error(TC_ENOMEM, "host allocation failed");
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(uint32_t));
  *pairs = p;
  *m = v.size() / 2;
  *n_declared = n;
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_graph_load_matrix_market(const char* text, uint64_t len, int device, tc_graph** out,
                                      tc_build_report* report) {
  if (!out || (len && !text)) return set_error(TC_EINVAL, "tc_graph_load_matrix_market: NULL argument");
  tc_graph* g = nullptr;
  TC_API_TRY
  tcb::MmHeader h;
  tcb::parse_mm_header(text, len, h);  // banner + size line (host, a few bytes)
  if (h.nnz >= (1ull << 32)) return set_error(TC_ERANGE, "MatrixMarket: >= 2^32 entries");
  DeviceGuard dg(device);
  g = new_handle(device);
  try {
    Timer t(g->stream);
    const uint64_t blen = len - h.body;
    tcb::DBuf<unsigned char> body(blen ? blen : 1, g->stream);
    if (blen)
      TC_CUDA(cudaMemcpyAsync(body.get(), text + h.body, blen, cudaMemcpyHostToDevice, g->stream));
    tcb::DBuf<uint32_t> pairs;
    if (!tcb::mm_tokenize(body.get(), blen, h, pairs, device, g->stream)) {
      // malformed body: the host parser throws the reference's exact ParseError
      std::vector<uint32_t> v;
      uint32_t n = 0;
      tcb::parse_matrix_market(text, len, v, n);
      tcb::fail(TC_EPARSE, "MatrixMarket: device tokenizer and host parser disagree");
    }
    body.release();
    tc_build_report rep{};
    tcb::build_from_pairs(*g, pairs.get(), h.nnz, h.n_declared, &rep);
    g->build_ms = t.stop();
    if (report) *report = rep;
  } catch (...) {
    destroy_handle(g);
    throw;
  }
  *out = g;
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_list_triangles_range(tc_graph* g, uint64_t first_edge, uint64_t last_edge, uint32_t* rows,
                                  uint64_t capacity, uint64_t* count) {
  if (!g || !count || (capacity && !rows)) return set_error(TC_EINVAL, "tc_list_triangles: NULL argument");
  if (first_edge > last_edge || last_edge > g->E)
    return set_error(TC_EINVAL, "tc_list_triangles_range: edge range outside [0, num_edges]");
  TC_API_TRY
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg(g->device);
  DevOut<uint32_t> out(capacity ? rows : nullptr, 3 * capacity, g->stream);
  const uint64_t T = tcb::list_triangles(*g, out.p, capacity, first_edge, last_edge);
  if (capacity) {
    out.count = 3 * std::min<uint64_t>(T, capacity);
    out.finish(g->stream);
  }
  TC_CUDA(cudaStreamSynchronize(g->stream));
  *count = T;
  return TC_OK;
  TC_API_CATCH
}

tc_status tc_list_triangles(tc_graph* g, uint32_t* rows, uint64_t capacity, uint64_t* count) {
  if (!g) return set_error(TC_EINVAL, "tc_list_triangles: NULL argument");
  return tc_list_triangles_range(g, 0, g->E, rows, capacity, count);
}

tc_status tc_graph_csr_cache_size(const tc_graph* g, uint64_t* len) {
  if (!g || !len) return set_error(TC_EINVAL, "tc_graph_csr_cache_size: NULL argument");
  *len = 32 + 8 * ((uint64_t)g->n + 1) + 4 * (2 * g->E);
  return TC_OK;
}

tc_status tc_graph_write_csr_cache(tc_graph* g, void* bytes) {
  if (!g || !bytes) return set_error(TC_EINVAL, "tc_graph_write_csr_cache: NULL argument");
  if (reinterpret_cast<uintptr_t>(bytes) & 7) return set_error(TC_EINVAL, "tc_graph_write_csr_cache: buffer not 8-byte aligned");
  TC_API_TRY
  unsigned char* b = static_cast<unsigned char*>(bytes);
  static const char kMagic[8] = {'T', 'R', 'I', 'M', 'C', 'S', 'R', '1'};
  std::memcpy(b, kMagic, 8);
  const uint64_t hdr[3] = {1, g->n, g->E};  // version, num_vertices, num_edges (little-endian host)
  std::memcpy(b + 8, hdr, sizeof(hdr));
  return tc_graph_export_csr(g, reinterpret_cast<uint64_t*>(b + 32),
                             reinterpret_cast<uint32_t*>(b + 32 + 8 * ((uint64_t)g->n + 1)));
  TC_API_CATCH
}

tc_status tc_csr_cache_to_graph(const void* bytes, uint64_t len, int device, tc_graph** out) {
  if (!out || (len && !bytes)) return set_error(TC_EINVAL, "tc_csr_cache_to_graph: NULL argument");
  TC_API_TRY
  std::vector<uint64_t> aligned;
  const void* b = bytes;
  if (reinterpret_cast<uintptr_t>(bytes) & 7) {
    aligned.resize(len / 8 + 1);
    std::memcpy(aligned.data(), bytes, len);
    b = aligned.data();
  }
  tcb::CsrView v;
  tcb::parse_csr_cache(b, len, v);  // header checks; offsets and adjacency are validated on the device
  return from_csr_impl(v.offsets, v.nbrs, v.n, v.num_edges, device, out, true);
  TC_API_CATCH
}

uint64_t tc_gen_num_edges(int kind, int scale, int param) { return tcb::gen_num_edges(kind, scale, param); }

tc_status tc_generate(int kind, int scale, int param, int device, uint32_t* pairs) {
  if (!pairs) return set_error(TC_EINVAL, "tc_generate: pairs is NULL");
  TC_API_TRY
  DeviceGuard dg(device);
  const uint64_t m = tcb::gen_num_edges(kind, scale, param);
  cudaStream_t s;
  TC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  try {
    DevOut<uint32_t> out(pairs, 2 * m, s);
    tcb::generate(kind, scale, param, out.p, s);
    out.finish(s);
    TC_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    cudaStreamDestroy(s);
    throw;
  }
  cudaStreamDestroy(s);
  return TC_OK;
  TC_API_CATCH
}

}  // extern "C"
