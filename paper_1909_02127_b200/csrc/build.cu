// build.cu -- edge list / CSR -> degree-oriented device CSR (north_star (1)).
//
// Replaces trimatch::build_graph (graph.cpp:33-85): the reference counts both
// orientations, scatters, then std::sort + unique per vertex, serially.  Here:
//   k_canon        loop drop (graph.cpp:43-46), range check (graph.cpp:40-42),
//                  canonical key min<<b | max (both orientations collapse)
//   radix_sort_u64 hand-written LSD sort over 2b bits (prim.cu)
//   unique         fused flag+scan compaction; duplicates = m - loops - |E|
//                  (graph.cpp:67-73, :80-81)
//   k_degree       undirected degree (graph.cpp:87-91 degrees())
//   rank           stable radix sort of (deg<<32 | id) on the degree bits
//   k_orient       keep u->v iff rank(u) < rank(v): the (deg,id) orientation
//                  that replaces filter_candidates + the triangle UMO
//                  (matcher.cpp:46-87, query_plan.cpp:168-184)
//   radix_sort_u64 + run-count + scan -> oriented CSR (off/col/src)
#include <cuda_runtime.h>

#include <cstdlib>

#include "graph.cuh"
#include "prim.cuh"

namespace tcb {
namespace {

constexpr int kT = 256;

__global__ void k_canon(const uint32_t* __restrict__ pairs, uint64_t m, uint32_t n, int b,
                        uint64_t* __restrict__ keys, unsigned long long* __restrict__ loops,
                        int* __restrict__ bad) {
  const uint64_t sentinel = (b >= 32) ? ~0ull : ((1ull << (2 * b)) - 1);
  unsigned long long my_loops = 0;
  int my_bad = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 e = reinterpret_cast<const uint2*>(pairs)[i];
    uint64_t key = sentinel;
    if (e.x >= n || e.y >= n) {
      my_bad = 1;
    } else if (e.x == e.y) {
      ++my_loops;
    } else {
      const uint32_t lo = min(e.x, e.y), hi = max(e.x, e.y);
      key = ((uint64_t)lo << b) | hi;
    }
    keys[i] = key;
  }
  my_loops = warp_sum(my_loops);
  if (lane_id() == 0 && my_loops) atomicAdd(loops, my_loops);
  if (__any_sync(0xffffffffu, my_bad) && lane_id() == 0) atomicOr(bad, 1);
}

struct UniqueFlag {
  const uint64_t* k;
  uint64_t sentinel;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    const uint64_t x = k[i];
    return (x != sentinel && (i == 0 || k[i - 1] != x)) ? 1u : 0u;
  }
};

__global__ void k_unique_scatter(const uint64_t* __restrict__ k, uint64_t m, uint64_t sentinel,
                                 const uint32_t* __restrict__ pos, uint64_t* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = k[i];
    if (x != sentinel && (i == 0 || k[i - 1] != x)) out[pos[i]] = x;
  }
}

// Undirected degree of both endpoints; keys sorted by the low endpoint, so the
// low side is aggregated per warp with match_any (hub rows are long runs).
__global__ void k_degree(const uint64_t* __restrict__ k, uint64_t E, int b, uint32_t* __restrict__ deg) {
  const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < E; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool valid = i < E;
    const uint64_t x = valid ? k[i] : 0;
    const uint32_t lo = valid ? (uint32_t)(x >> b) : 0xffffffffu;
    const uint32_t hi = (uint32_t)(x & mask);
    const unsigned peers = __match_any_sync(0xffffffffu, lo);
    if (valid && lane_id() == (unsigned)(__ffs(peers) - 1)) atomicAdd(&deg[lo], (uint32_t)__popc(peers));
    if (valid) atomicAdd(&deg[hi], 1u);
  }
}

__global__ void k_max_u32(const uint32_t* __restrict__ a, uint64_t n, uint32_t* __restrict__ out) {
  uint32_t m = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, a[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane_id() == 0 && m) atomicMax(out, m);
}

__global__ void k_rank_keys(const uint32_t* __restrict__ deg, uint32_t n, uint64_t* __restrict__ keys) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    keys[v] = ((uint64_t)deg[v] << 32) | v;
}

__global__ void k_rank_maps(const uint64_t* __restrict__ sorted, uint32_t n, uint32_t* __restrict__ id_of,
                            uint32_t* __restrict__ rank_of, uint32_t* __restrict__ deg_r) {
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = sorted[r];
    const uint32_t id = (uint32_t)x;
    id_of[r] = id;
    rank_of[id] = (uint32_t)r;
    deg_r[r] = (uint32_t)(x >> 32);
  }
}

__global__ void k_orient(const uint64_t* __restrict__ k, uint64_t E, int b, const uint32_t* __restrict__ rank_of,
                         uint64_t* __restrict__ okeys) {
  const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t x = k[i];
    const uint32_t ra = rank_of[(uint32_t)(x >> b)], rb = rank_of[(uint32_t)(x & mask)];
    okeys[i] = ((uint64_t)min(ra, rb) << b) | max(ra, rb);
  }
}

// oriented keys (sorted) -> col/src + out-degree run counts
__global__ void k_split_oriented(const uint64_t* __restrict__ ok, uint64_t E, int b, uint32_t* __restrict__ col,
                                 uint32_t* __restrict__ src, uint32_t* __restrict__ dplus) {
  const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < E; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool valid = i < E;
    const uint64_t x = valid ? ok[i] : 0;
    const uint32_t s = valid ? (uint32_t)(x >> b) : 0xffffffffu;
    if (valid) {
      col[i] = (uint32_t)(x & mask);
      src[i] = s;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, s);
    if (valid && lane_id() == (unsigned)(__ffs(peers) - 1)) atomicAdd(&dplus[s], (uint32_t)__popc(peers));
  }
}

// CSR (sorted rows) -> canonical unique keys: entries (u,v) with v > u, in
// row order, are already sorted and unique.  row_of(i) comes from a scan of
// "rows ending at i" counts.
__global__ void k_row_ends(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ ends) {
  const uint64_t total = off[n];
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = off[u + 1];
    if (e < total) atomicAdd(&ends[e], 1u);
  }
}

struct RowOf {
  const uint32_t* excl;
  const uint32_t* ends;
};

struct UpperFlag {  // entry i of row r is kept iff nbrs[i] > r
  const uint32_t* nbrs;
  const uint32_t* row_excl;
  const uint32_t* ends;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    const uint32_t r = row_excl[i] + ends[i];
    return nbrs[i] > r ? 1u : 0u;
  }
};

__global__ void k_csr_keys(const uint32_t* __restrict__ nbrs, uint64_t total, const uint32_t* __restrict__ row_excl,
                           const uint32_t* __restrict__ ends, const uint32_t* __restrict__ pos, int b,
                           uint64_t* __restrict__ keys) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t r = row_excl[i] + ends[i];
    const uint32_t v = nbrs[i];
    if (v > r) keys[pos[i]] = ((uint64_t)r << b) | v;
  }
}

// export: oriented edge -> both directed keys in id space
__global__ void k_directed_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ col, uint64_t E,
                                const uint32_t* __restrict__ id_of, int b, uint64_t* __restrict__ keys) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = id_of[src[i]], c = id_of[col[i]];
    keys[2 * i] = ((uint64_t)a << b) | c;
    keys[2 * i + 1] = ((uint64_t)c << b) | a;
  }
}

__global__ void k_low_bits(const uint64_t* __restrict__ keys, uint64_t n, int b, uint32_t* __restrict__ out) {
  const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (uint32_t)(keys[i] & mask);
}

__global__ void k_gather_deg(const uint32_t* __restrict__ deg_r, const uint32_t* __restrict__ rank_of, uint32_t n,
                             uint32_t* __restrict__ out) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    out[v] = deg_r[rank_of[v]];
}

struct HotFlag {
  const uint32_t* col;
  uint32_t h0;
  __device__ __forceinline__ uint32_t operator()(uint64_t e) const { return col[e] >= h0 ? 1u : 0u; }
};

__global__ void k_hot_scatter(const uint32_t* __restrict__ col, uint64_t E, uint32_t h0,
                              const uint32_t* __restrict__ hp, uint16_t* __restrict__ colH) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = col[e];
    if (x >= h0) colH[hp[e]] = (uint16_t)(x - h0);
  }
}

__global__ void k_hot_offsets(const uint32_t* __restrict__ off, uint32_t n, uint64_t E,
                              const uint32_t* __restrict__ hp, uint32_t total_hot, uint32_t* __restrict__ offH) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u <= n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t o = off[u];
    offH[u] = o < E ? hp[o] : total_hot;
  }
}

struct DegLoad64 {
  const uint32_t* d;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const { return d[i]; }
};

unsigned grid_gs(uint64_t n, int device) {
  // grid-stride launches: a few waves of 148 SMs is plenty
  const uint64_t cap = (uint64_t)num_sms(device) * 16;
  uint64_t g = ceil_div64(n, kT);
  if (g < 1) g = 1;
  return (unsigned)(g < cap ? g : cap);
}

template <typename T>
T read_scalar(const T* d, cudaStream_t s) {
  T h;
  TC_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  return h;
}

// Shared tail: sorted unique canonical id-space keys -> ranks -> oriented CSR.
void finalize(tc_graph& g, DBuf<uint64_t>& ukeys, uint64_t E) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const int b = g.id_bits;
  const int dev = g.device;
  if (E >= (1ull << 32)) fail(TC_ERANGE, "graph has >= 2^32 undirected edges (u32 oriented offsets)");
  g.E = E;

  DBuf<uint32_t> deg(n ? n : 1, s);
  TC_CUDA(cudaMemsetAsync(deg.get(), 0, sizeof(uint32_t) * (n ? n : 1), s));
  if (E) {
    k_degree<<<grid_gs(E, dev), kT, 0, s>>>(ukeys.get(), E, b, deg.get());
    TC_LAUNCH();
  }
  DBuf<uint32_t> scal(2, s);
  TC_CUDA(cudaMemsetAsync(scal.get(), 0, 2 * sizeof(uint32_t), s));
  if (n) {
    k_max_u32<<<grid_gs(n, dev), kT, 0, s>>>(deg.get(), n, scal.get());
    TC_LAUNCH();
  }
  g.max_deg = read_scalar(scal.get(), s);

  // degree rank: stable sort of (deg<<32 | id) on the degree bits
  g.id_of.alloc(n ? n : 1, s);
  g.rank_of.alloc(n ? n : 1, s);
  g.deg.alloc(n ? n : 1, s);
  if (n) {
    DBuf<uint64_t> rk(n, s), rk2(n, s);
    k_rank_keys<<<grid_gs(n, dev), kT, 0, s>>>(deg.get(), n, rk.get());
    TC_LAUNCH();
    const int db = bits_for(g.max_deg);
    uint64_t* sorted = radix_sort_u64(rk.get(), rk2.get(), n, 32, 32 + ((db + 7) / 8) * 8, s);
    k_rank_maps<<<grid_gs(n, dev), kT, 0, s>>>(sorted, n, g.id_of.get(), g.rank_of.get(), g.deg.get());
    TC_LAUNCH();
  }
  deg.release();

  // orientation + oriented CSR
  g.col.alloc(E + 8, s);
  g.src.alloc(E ? E : 1, s);
  g.off.alloc((uint64_t)n + 1, s);
  TC_CUDA(cudaMemsetAsync(g.col.get(), 0xff, (E + 8) * sizeof(uint32_t), s));
  DBuf<uint32_t> dplus(n ? n : 1, s);
  TC_CUDA(cudaMemsetAsync(dplus.get(), 0, sizeof(uint32_t) * (n ? n : 1), s));
  if (E) {
    DBuf<uint64_t> ok(E, s);
    k_orient<<<grid_gs(E, dev), kT, 0, s>>>(ukeys.get(), E, b, g.rank_of.get(), ok.get());
    TC_LAUNCH();
    // reuse ukeys as the ping-pong buffer
    uint64_t* sorted = radix_sort_u64(ok.get(), ukeys.get(), E, 0, 2 * b, s);
    k_split_oriented<<<grid_gs(E, dev), kT, 0, s>>>(sorted, E, b, g.col.get(), g.src.get(), dplus.get());
    TC_LAUNCH();
  }
  ukeys.release();
  scan_exclusive<uint32_t>(LoadArray<uint32_t>{dplus.get()}, g.off.get(), n, g.off.get() + n, s);
  TC_CUDA(cudaMemsetAsync(scal.get(), 0, sizeof(uint32_t), s));
  if (n) {
    k_max_u32<<<grid_gs(n, dev), kT, 0, s>>>(dplus.get(), n, scal.get());
    TC_LAUNCH();
  }
  g.max_dplus = read_scalar(scal.get(), s);

  // hot window mirror (graph.cuh): 16-bit copy of every row's members >= h0
  {
    const char* hb = getenv("TCB_HOT_BITS");  // tests: shrink the window to drive the cold path
    uint32_t hot = hb ? (uint32_t)strtoul(hb, nullptr, 10) : kHotBits;
    if (hot < 32) hot = 32;
    if (hot > kHotBits) hot = kHotBits;
    g.h0 = n > hot ? n - hot : 0;
    DBuf<uint32_t> hp(E ? E : 1, s), th(1, s);
    scan_exclusive<uint32_t>(HotFlag{g.col.get(), g.h0}, hp.get(), E, th.get(), s);
    const uint32_t total_hot = E ? read_scalar(th.get(), s) : 0;
    g.colH.alloc((uint64_t)total_hot + 16, s);
    TC_CUDA(cudaMemsetAsync(g.colH.get(), 0, ((uint64_t)total_hot + 16) * sizeof(uint16_t), s));
    g.offH.alloc((uint64_t)n + 1, s);
    if (E) {
      k_hot_scatter<<<grid_gs(E, dev), kT, 0, s>>>(g.col.get(), E, g.h0, hp.get(), g.colH.get());
      TC_LAUNCH();
    }
    k_hot_offsets<<<grid_gs((uint64_t)n + 1, dev), kT, 0, s>>>(g.off.get(), n, E, hp.get(), total_hot,
                                                               g.offH.get());
    TC_LAUNCH();
  }
}

}  // namespace

void build_from_pairs(tc_graph& g, const uint32_t* d_pairs, uint64_t m, uint32_t n, tc_build_report* rep) {
  cudaStream_t s = g.stream;
  const int dev = g.device;
  g.n = n;
  g.id_bits = n > 1 ? bits_for((uint64_t)n - 1) : 1;
  const int b = g.id_bits;
  if (m >= (1ull << 32)) fail(TC_ERANGE, "edge list with >= 2^32 entries");
  if (n == 0 && m > 0) fail(TC_EINVAL, "build_graph: vertex id out of declared range");

  DBuf<unsigned long long> cnt(1, s);
  DBuf<int> bad(1, s);
  TC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
  TC_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  DBuf<uint64_t> keys(m ? m : 1, s), keys2(m ? m : 1, s);
  if (m) {
    k_canon<<<grid_gs(m, dev), kT, 0, s>>>(d_pairs, m, n, b, keys.get(), cnt.get(), bad.get());
    TC_LAUNCH();
  }
  if (read_scalar(bad.get(), s)) fail(TC_EINVAL, "build_graph: vertex id out of declared range");
  const uint64_t loops = read_scalar(cnt.get(), s);

  uint64_t* sorted = radix_sort_u64(keys.get(), keys2.get(), m, 0, 2 * b, s);
  const uint64_t sentinel = (b >= 32) ? ~0ull : ((1ull << (2 * b)) - 1);
  DBuf<uint32_t> pos(m ? m : 1, s);
  DBuf<uint32_t> ecount(1, s);
  scan_exclusive<uint32_t>(UniqueFlag{sorted, sentinel}, pos.get(), m, ecount.get(), s);
  const uint64_t E = m ? read_scalar(ecount.get(), s) : 0;
  DBuf<uint64_t> ukeys(E ? E : 1, s);
  if (m) {
    k_unique_scatter<<<grid_gs(m, dev), kT, 0, s>>>(sorted, m, sentinel, pos.get(), ukeys.get());
    TC_LAUNCH();
  }
  pos.release();
  keys.release();
  keys2.release();
  if (rep) {
    rep->self_loops_removed = loops;
    rep->duplicate_entries_removed = m - loops - E;
  }
  finalize(g, ukeys, E);
}

void build_from_csr(tc_graph& g, const uint64_t* d_off, const uint32_t* d_nbrs, uint32_t n, uint64_t num_edges) {
  cudaStream_t s = g.stream;
  const int dev = g.device;
  g.n = n;
  g.id_bits = n > 1 ? bits_for((uint64_t)n - 1) : 1;
  const int b = g.id_bits;
  const uint64_t total = 2 * num_edges;
  if (total >= (1ull << 32)) fail(TC_ERANGE, "CSR with >= 2^32 directed entries");
  DBuf<uint32_t> ends(total ? total : 1, s), row_excl(total ? total : 1, s), pos(total ? total : 1, s);
  DBuf<uint32_t> ecount(1, s);
  uint64_t E = 0;
  if (total) {
    TC_CUDA(cudaMemsetAsync(ends.get(), 0, total * sizeof(uint32_t), s));
    k_row_ends<<<grid_gs(n, dev), kT, 0, s>>>(d_off, n, ends.get());
    TC_LAUNCH();
    scan_exclusive<uint32_t>(LoadArray<uint32_t>{ends.get()}, row_excl.get(), total, (uint32_t*)nullptr, s);
    scan_exclusive<uint32_t>(UpperFlag{d_nbrs, row_excl.get(), ends.get()}, pos.get(), total, ecount.get(), s);
    E = read_scalar(ecount.get(), s);
    if (E != num_edges) fail(TC_EINVAL, "Graph: inconsistent CSR arrays (asymmetric adjacency)");
  }
  DBuf<uint64_t> ukeys(E ? E : 1, s);
  if (total) {
    k_csr_keys<<<grid_gs(total, dev), kT, 0, s>>>(d_nbrs, total, row_excl.get(), ends.get(), pos.get(), b,
                                                  ukeys.get());
    TC_LAUNCH();
  }
  ends.release();
  row_excl.release();
  pos.release();
  finalize(g, ukeys, E);
}

void export_csr(tc_graph& g, uint64_t* d_off, uint32_t* d_nbrs) {
  cudaStream_t s = g.stream;
  const int dev = g.device;
  const uint32_t n = g.n;
  const uint64_t E = g.E;
  const int b = g.id_bits;
  // offsets from degrees in id space (u64 scan)
  DBuf<uint32_t> deg(n ? n : 1, s);
  if (n) {
    k_gather_deg<<<grid_gs(n, dev), kT, 0, s>>>(g.deg.get(), g.rank_of.get(), n, deg.get());
    TC_LAUNCH();
  }
  scan_exclusive<uint64_t>(DegLoad64{deg.get()}, d_off, n, d_off + n, s);
  if (E == 0) return;
  if (2 * E >= (1ull << 32)) fail(TC_ERANGE, "export_csr: >= 2^32 directed entries");
  DBuf<uint64_t> k1(2 * E, s), k2(2 * E, s);
  k_directed_keys<<<grid_gs(E, dev), kT, 0, s>>>(g.src.get(), g.col.get(), E, g.id_of.get(), b, k1.get());
  TC_LAUNCH();
  uint64_t* sorted = radix_sort_u64(k1.get(), k2.get(), 2 * E, 0, 2 * b, s);
  k_low_bits<<<grid_gs(2 * E, dev), kT, 0, s>>>(sorted, 2 * E, b, d_nbrs);
  TC_LAUNCH();
}

void export_degrees(tc_graph& g, uint32_t* d_deg) {
  if (!g.n) return;
  k_gather_deg<<<grid_gs(g.n, g.device), kT, 0, g.stream>>>(g.deg.get(), g.rank_of.get(), g.n, d_deg);
  TC_LAUNCH();
}

}  // namespace tcb
