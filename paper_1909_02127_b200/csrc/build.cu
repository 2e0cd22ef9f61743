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

#include <algorithm>
#include <memory>
#include <cstdlib>
#include <vector>

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
// low side is aggregated per run of equal sorted keys (hub rows are long runs).
// Run aggregation over a warp's 32 consecutive entries of a sorted key
// stream: the first lane of each run of equal keys adds the run length (the
// valid lanes are a prefix).  Replaces match_any, whose MIO cost is high.
__device__ __forceinline__ void add_sorted_runs(uint32_t key, bool valid, uint32_t* __restrict__ cnt) {
  const unsigned lane = lane_id();
  const uint32_t up = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = valid && (lane == 0 || up != key);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const unsigned nvalid = __popc(__ballot_sync(0xffffffffu, valid));
  if (head) {
    const unsigned above = lane == 31 ? 0u : heads & ~((2u << lane) - 1u);
    const unsigned next = above ? (unsigned)(__ffs(above) - 1) : nvalid;
    atomicAdd(&cnt[key], next - lane);
  }
}

__global__ void k_degree(const uint64_t* __restrict__ k, uint64_t E, int b, uint32_t* __restrict__ deg) {
  const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < E; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool valid = i < E;
    const uint64_t x = valid ? k[i] : 0;
    const uint32_t lo = valid ? (uint32_t)(x >> b) : 0xffffffffu;
    const uint32_t hi = (uint32_t)(x & mask);
    add_sorted_runs(lo, valid, deg);  // keys are sorted: equal low ids are adjacent
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
    add_sorted_runs(s, valid, dplus);
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

// The directed entries whose source id is in [u_lo, u_hi), keyed
// (source - u_lo) << b | target, appended through one warp-aggregated counter
// (their order is restored by the sort).
__global__ void k_directed_keys_range(const uint32_t* __restrict__ src, const uint32_t* __restrict__ col, uint64_t E,
                                      const uint32_t* __restrict__ id_of, int b, uint32_t u_lo, uint32_t u_hi,
                                      uint64_t* __restrict__ keys, unsigned long long* __restrict__ cnt) {
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < E; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t a = 0, c = 0;
    if (i < E) {
      a = id_of[src[i]];
      c = id_of[col[i]];
    }
    const bool ka = i < E && a >= u_lo && a < u_hi, kc = i < E && c >= u_lo && c < u_hi;
    const uint32_t na = __popc(__ballot_sync(0xffffffffu, ka)), nc = __popc(__ballot_sync(0xffffffffu, kc));
    unsigned long long w = 0;
    if (lane_id() == 0 && na + nc) w = atomicAdd(cnt, (unsigned long long)(na + nc));
    w = __shfl_sync(0xffffffffu, w, 0);
    const uint32_t pa = __popc(__ballot_sync(0xffffffffu, ka) & lanemask_lt());
    const uint32_t pc = na + __popc(__ballot_sync(0xffffffffu, kc) & lanemask_lt());
    if (ka) keys[w + pa] = ((uint64_t)(a - u_lo) << b) | c;
    if (kc) keys[w + pc] = ((uint64_t)(c - u_lo) << b) | a;
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

// Hot-window mirror of the finished (sorted) rows: a row's hot members are its
// suffix >= h0, counted by binary search; entry e of row r = src[e] in that
// suffix lands at offH[r+1] - (off[r+1] - e).
__global__ void k_hot_counts(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, uint32_t n,
                             uint32_t h0, uint32_t* __restrict__ hcnt) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {  // 64-bit: n may be 2^32 - 1
    const uint32_t b = off[u + 1];
    uint32_t lo = off[u], hi = b;
    while (lo < hi) {
      const uint32_t mid = lo + ((hi - lo) >> 1);  // edge indices: lo + hi may pass 2^32
      if (col[mid] < h0) lo = mid + 1; else hi = mid;
    }
    hcnt[u] = b - lo;
  }
}

__global__ void k_hot_scatter(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                              const uint32_t* __restrict__ src, uint64_t E, uint32_t h0,
                              const uint32_t* __restrict__ offH, uint16_t* __restrict__ colH) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = col[e];
    if (x >= h0) {
      const uint32_t r = src[e];
      colH[offH[r + 1] - (off[r + 1] - (uint32_t)e)] = (uint16_t)(x - h0);
    }
  }
}

// ---- CSR route (tc_graph_from_csr): rank-space rows without a global sort ----
// The input rows are complete adjacency lists.  Before any neighbour arrives,
// the offsets alone give every vertex its rank and a padded rank-space slot of
// deg(u) entries (pad_off = scan of deg by rank).  Then ONE pass per id-row u
// -- a thread (short rows), a warp (<= kBigRow) or a warp per kBigRow chunk
// (hubs: count, chunk bases, write) -- keeps the entries with rank(v) >
// rank(u), packs them at the head of u's padded slot (ballot prefix,
// deterministic) and records d+(rank u).  Rows are independent, so the pass
// runs chunk by chunk behind the host->device copy of the neighbour array
// (build_from_csr); the row sorts then move every slot to its final place.
constexpr uint32_t kBigRow = 1024;
constexpr uint64_t kExportChunk = 1ull << 31;  // directed entries per export sort

__global__ void k_csr_deg(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ deg,
                          uint32_t* __restrict__ big, unsigned int* __restrict__ nbig, int* __restrict__ bad) {
  for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = off[u], b = off[u + 1];
    if (b < a) {
      atomicOr(bad, 1);
      deg[u] = 0;
      continue;
    }
    const uint32_t d = (uint32_t)(b - a);
    deg[u] = d;
    if (d > kBigRow) big[atomicAdd(nbig, 1u)] = (uint32_t)u;
  }
}

struct RowCtx {
  const uint64_t* off;
  const uint32_t* nbrs;
  const uint32_t* rank_of;
  uint32_t n;
  uint32_t* dplus;
  const uint64_t* pad_off;  // padded rank-space slots (deg entries each; 2E may exceed 2^32)
  uint32_t* pad;
  int strict;  // TRIMCSR1 ingest: also reject self-loops and non-ascending rows (io.cpp:211-216)
};

// validity bits of entry i (row u starting at a): 1 = id out of range,
// 2 = (strict) self-loop or not strictly ascending
__device__ __forceinline__ int entry_bad(const RowCtx& cx, uint64_t i, uint64_t a, uint32_t u, uint32_t v) {
  int bad = v >= cx.n ? 1 : 0;
  if (cx.strict && (v == u || (i > a && cx.nbrs[i - 1] >= v))) bad |= 2;
  return bad;
}

// One warp over id-row u; returns (in lane-summed form) the entries v > u.
__device__ __forceinline__ uint32_t warp_csr_row(const RowCtx& cx, uint32_t u, int& bad) {
  const unsigned lane = lane_id();
  const uint64_t a = cx.off[u], b = cx.off[u + 1];
  const uint32_t ru = cx.rank_of[u];
  uint32_t* out = cx.pad + cx.pad_off[ru];
  uint32_t run = 0, upper = 0;
  constexpr int kU = 4;
  for (uint64_t i0 = a; i0 < b; i0 += 32 * kU) {
    uint32_t v[kU], rv[kU];
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const uint64_t i = i0 + 32 * t + lane;
      v[t] = i < b ? cx.nbrs[i] : 0xffffffffu;
    }
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const bool valid = i0 + 32 * t + lane < b;
      if (valid) bad |= entry_bad(cx, i0 + 32 * t + lane, a, u, v[t]);
      rv[t] = (valid && v[t] < cx.n) ? cx.rank_of[v[t]] : 0u;
      upper += (valid && v[t] > u && v[t] < cx.n) ? 1u : 0u;
    }
#pragma unroll
    for (int t = 0; t < kU; ++t) {
      const bool valid = i0 + 32 * t + lane < b && v[t] < cx.n;
      const bool keep = valid && rv[t] > ru;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (keep) out[run + __popc(m & lanemask_lt())] = rv[t];
      run += __popc(m);
    }
  }
  if (lane == 0) cx.dplus[ru] = run;
  return upper;
}

// One thread over a short id-row u (<= kShortRow entries).
__device__ __forceinline__ uint32_t thread_csr_row(const RowCtx& cx, uint32_t u, uint64_t a, uint64_t b, int& bad) {
  const uint32_t ru = cx.rank_of[u];
  uint32_t* out = cx.pad + cx.pad_off[ru];
  uint32_t run = 0, upper = 0;
  for (uint64_t i0 = a; i0 < b; i0 += 4) {
    uint32_t v[4], rv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = i0 + t < b ? cx.nbrs[i0 + t] : 0xffffffffu;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool valid = i0 + t < b;
      if (valid) bad |= entry_bad(cx, i0 + t, a, u, v[t]);
      rv[t] = (valid && v[t] < cx.n) ? cx.rank_of[v[t]] : 0u;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool valid = i0 + t < b && v[t] < cx.n;
      upper += (valid && v[t] > u) ? 1u : 0u;
      if (valid && rv[t] > ru) out[run++] = rv[t];
    }
  }
  cx.dplus[ru] = run;
  return upper;
}

constexpr uint32_t kShortRow = 24;

// Id-rows [lo, hi) of at most kBigRow entries, groups of 32 from a queue (row
// lengths are skewed): short rows a thread each, the group's longer rows
// after, one at a time, warp-wide.
__global__ void __launch_bounds__(256) k_csr_rows(RowCtx cx, uint32_t lo, uint32_t hi,
                                                 unsigned int* __restrict__ queue,
                                                 unsigned long long* __restrict__ upper_total,
                                                 int* __restrict__ bad_flag) {
  uint32_t upper = 0;
  int bad = 0;
  while (true) {
    uint32_t g0 = 0;
    if (lane_id() == 0) g0 = atomicAdd(queue, 32u);
    g0 = __shfl_sync(0xffffffffu, g0, 0);
    if (g0 >= hi - lo) break;
    const uint32_t u0 = lo + g0;
    const uint32_t u = u0 + lane_id();
    const bool live = lane_id() < hi - u0;  // (u < hi without wrap-around)
    uint64_t a = 0, b = 0;
    if (live) {
      a = cx.off[u];
      b = cx.off[u + 1];
    }
    const bool is_short = live && b - a <= kShortRow;
    if (is_short) upper += thread_csr_row(cx, u, a, b, bad);
    uint32_t longs = __ballot_sync(0xffffffffu, live && !is_short && b - a <= kBigRow);
    while (longs) {
      const int j = __ffs(longs) - 1;
      longs &= longs - 1;
      upper += warp_csr_row(cx, u0 + j, bad);
    }
  }
  const unsigned long long w = warp_sum((unsigned long long)upper);
  if (lane_id() == 0 && w) atomicAdd(upper_total, w);
  bad = (int)__reduce_or_sync(0xffffffffu, (unsigned)bad);
  if (bad && lane_id() == 0) atomicOr(bad_flag, bad);
}

// Rows longer than kBigRow (hubs) are cut into chunks of kBigRow entries,
// chunk c = {u, first entry}; a warp per chunk.  Pass 0 adds each chunk's kept
// count to d+(rank u) and records it; k_chunk_bases turns the counts into
// per-chunk write bases within the row; pass 1 writes.  Only chunks of rows in
// [lo, hi) (the rows whose entries have arrived) are taken.
struct Chunk {
  uint32_t u, c0;  // row, first chunk of the row in the chunk list
  uint64_t a;      // first entry of the chunk
};

template <int kPass>
__global__ void __launch_bounds__(256) k_csr_chunks(RowCtx cx, const Chunk* __restrict__ chunks, uint32_t nchunks,
                                                    uint32_t lo, uint32_t hi, uint32_t* __restrict__ ccount,
                                                    const uint32_t* __restrict__ cbase,
                                                    unsigned long long* __restrict__ upper_total,
                                                    int* __restrict__ bad_flag) {
  const unsigned lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  uint32_t upper = 0;
  int bad = 0;
  for (uint32_t c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); c < nchunks; c += warps) {
    const Chunk ch = chunks[c];
    if (ch.u < lo || ch.u >= hi) continue;
    const uint64_t rowend = cx.off[ch.u + 1];
    const uint64_t a = ch.a, b = min(rowend, a + kBigRow);
    const uint32_t ru = cx.rank_of[ch.u];
    uint32_t* out = cx.pad + cx.pad_off[ru];
    uint32_t run = kPass ? cbase[c] : 0u, kept = 0;
    for (uint64_t i0 = a; i0 < b; i0 += 128) {
      uint32_t v[4], rv[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint64_t i = i0 + 32 * t + lane;
        v[t] = i < b ? cx.nbrs[i] : 0xffffffffu;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const bool valid = i0 + 32 * t + lane < b;
        if (!kPass && valid) bad |= entry_bad(cx, i0 + 32 * t + lane, cx.off[ch.u], ch.u, v[t]);
        rv[t] = (valid && v[t] < cx.n) ? cx.rank_of[v[t]] : 0u;
        upper += (valid && v[t] > ch.u && v[t] < cx.n) ? 1u : 0u;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const bool keep = i0 + 32 * t + lane < b && v[t] < cx.n && rv[t] > ru;
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        if (kPass && keep) out[run + __popc(m & lanemask_lt())] = rv[t];
        run += __popc(m);
        kept += __popc(m);
      }
    }
    if (!kPass && lane == 0) {
      ccount[c] = kept;
      if (kept) atomicAdd(&cx.dplus[ru], kept);
    }
  }
  if (!kPass) {
    const unsigned long long w = warp_sum((unsigned long long)upper);
    if (lane == 0 && w) atomicAdd(upper_total, w);
    bad = (int)__reduce_or_sync(0xffffffffu, (unsigned)bad);
    if (bad && lane == 0) atomicOr(bad_flag, bad);
  }
}

struct ChunkCount {
  const uint32_t* big;
  const uint64_t* off;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const {
    const uint32_t u = big[i];
    return (uint32_t)((off[u + 1] - off[u] + kBigRow - 1) / kBigRow);
  }
};

__global__ void k_chunk_fill(const uint32_t* __restrict__ big, uint32_t nbig, const uint64_t* __restrict__ off,
                             const uint32_t* __restrict__ choff, Chunk* __restrict__ chunks) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nbig; i += gridDim.x * blockDim.x) {
    const uint32_t u = big[i], c0 = choff[i];
    const uint64_t a = off[u], b = off[u + 1];
    uint32_t c = c0;
    for (uint64_t x = a; x < b; x += kBigRow) chunks[c++] = Chunk{u, c0, x};
  }
}

void kl_scan_chunks(const uint32_t* big, uint32_t nbig, const uint64_t* off, uint32_t* choff, cudaStream_t s) {
  scan_exclusive<uint32_t>(ChunkCount{big, off}, choff, nbig, choff + nbig, s);
}

// per big row (thread): exclusive prefix of its chunks' kept counts
__global__ void k_chunk_bases(const Chunk* __restrict__ chunks, uint32_t nchunks, uint32_t lo, uint32_t hi,
                              const uint32_t* __restrict__ ccount, uint32_t* __restrict__ cbase) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nchunks; c += gridDim.x * blockDim.x) {
    if (chunks[c].c0 != c || chunks[c].u < lo || chunks[c].u >= hi) continue;  // first chunk of an arrived row
    uint32_t run = 0;
    for (uint32_t k = c; k < nchunks && chunks[k].u == chunks[c].u; ++k) {
      cbase[k] = run;
      run += ccount[k];
    }
  }
}

// Row sorts.  Every rank-space row r is sorted IN its padded slot
// pad[pad_off[r], + d+(r)) as soon as its id-row has been oriented (piece by
// piece, behind the host copy), and its hot count hcnt[r] (members >= h0, the
// sorted suffix) recorded; after the last piece one compaction pass moves the
// slots to col/src and writes the hot mirror.  Rows of <= 16 entries are
// sorted by their lane (register bitonic network), rows of 17..32 by the warp
// (shuffle bitonic), 33..1024 by a warp through a conflict-free SMEM tile,
// longer rows by a CTA in SMEM; rows longer than sort_max are listed for the
// radix fallback.
struct SlotSort {
  const uint32_t* rank_of;
  const uint64_t* pad_off;
  uint32_t* pad;
  const uint32_t* dplus;
  uint32_t h0;
  uint32_t sort_max;
  uint32_t* hcnt;
  uint32_t* huge;  // rows over sort_max
  unsigned int* nhuge;
};

__device__ __forceinline__ void sort16(uint32_t (&x)[16]) {
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const bool asc = (i & k) == 0;
          const uint32_t a = x[i], b = x[l];
          x[i] = asc ? min(a, b) : max(a, b);
          x[l] = asc ? max(a, b) : min(a, b);
        }
      }
    }
  }
}

// The id-rows [lo, hi) of one piece, 32 per warp: their rank-space rows.
__global__ void __launch_bounds__(256) k_slot_sort_warp(SlotSort ss, uint32_t lo, uint32_t hi,
                                                        uint32_t* __restrict__ longrows,
                                                        unsigned int* __restrict__ nlong) {
  const unsigned lane = lane_id();
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint64_t u0 = lo + (uint64_t)(blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * 32; u0 < hi;
       u0 += (uint64_t)warps * 32) {
    uint32_t r = 0, d = 0;
    uint64_t po = 0;
    if (u0 + lane < hi) {
      r = ss.rank_of[u0 + lane];
      d = ss.dplus[r];
      po = ss.pad_off[r];
    }
    if (d > ss.sort_max) {
      ss.huge[atomicAdd(ss.nhuge, 1u)] = r;
      d = 0;
    } else if (d > 32) {
      longrows[atomicAdd(nlong, 1u)] = r;
      d = 0;
    }
    if (d >= 1 && d <= 16) {  // (hcnt is zeroed up front for empty rows)
      uint32_t x[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) x[i] = (uint32_t)i < d ? ss.pad[po + i] : 0xffffffffu;
      if (d >= 2) sort16(x);
      uint32_t h = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if ((uint32_t)i < d) {
          ss.pad[po + i] = x[i];
          h += x[i] >= ss.h0;
        }
      ss.hcnt[r] = h;
    }
    uint32_t mid = __ballot_sync(0xffffffffu, d > 16 && d <= 32);
    while (mid) {
      const int j = __ffs(mid) - 1;
      mid &= mid - 1;
      const uint32_t dj = __shfl_sync(0xffffffffu, d, j);
      const uint64_t pj = __shfl_sync(0xffffffffu, po, j);
      const uint32_t rj = __shfl_sync(0xffffffffu, r, j);
      uint32_t x = lane < dj ? ss.pad[pj + lane] : 0xffffffffu;
#pragma unroll
      for (uint32_t k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
          const uint32_t y = __shfl_xor_sync(0xffffffffu, x, jj);
          const bool asc = (lane & k) == 0, lower = (lane & jj) == 0;
          x = (lower == asc) ? min(x, y) : max(x, y);
        }
      }
      if (lane < dj) ss.pad[pj + lane] = x;
      const uint32_t h = __popc(__ballot_sync(0xffffffffu, lane < dj && x >= ss.h0));
      if (lane == 0) ss.hcnt[rj] = h;
    }
  }
}

// In-lane bitonic stage j (< kE) of merge size k over a lane's kE registers.
template <int kE, int J>
__device__ __forceinline__ void lane_stage(uint32_t (&x)[kE], uint32_t pb, uint32_t k) {
  if constexpr (J < kE) {
#pragma unroll
    for (int i = 0; i < kE; ++i) {
      const int l = i ^ J;
      if (l > i && l < kE) {
        const bool asc = ((pb + i) & k) == 0;
        const uint32_t a = x[i], b = x[l];
        x[i] = asc ? min(a, b) : max(a, b);
        x[l] = asc ? max(a, b) : min(a, b);
      }
    }
  }
}

// Listed rows of 33..1024 entries: a warp each, kE = 2..32 entries per lane
// in registers (position p = lane*kE + i), bitonic network over 32*kE: in-lane
// stages for j < kE, shuffles for j >= kE.  The row goes through a per-warp
// SMEM tile (index p + p/32: conflict-free both ways) so that global loads and
// stores stay coalesced.  Sorted in place; returns the row's hot count.
template <int kE>
__device__ __forceinline__ uint32_t warp_sort_row(uint32_t* __restrict__ row, uint32_t d, uint32_t h0,
                                                  uint32_t* __restrict__ sm) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int m = 0; m < kE; ++m) {
    const uint32_t t = m * 32 + lane;
    sm[t + m] = t < d ? row[t] : 0xffffffffu;
  }
  __syncwarp();
  uint32_t x[kE];
#pragma unroll
  for (int i = 0; i < kE; ++i) {
    const uint32_t p = lane * kE + i;
    x[i] = sm[p + (p >> 5)];
  }
  // Networks up to 256 are fully unrolled; above, k stays a runtime loop (a
  // fully unrolled network of 1024 is ~20k instructions and the warps stall
  // on instruction fetch: 4.6 -> 1.4 ms for the 257..1024 rows at C4).
  const uint32_t pb = lane * kE;
  if constexpr (kE <= 8) {
#pragma unroll
    for (uint32_t k = 2; k <= 32u * kE; k <<= 1) {
#pragma unroll
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        if (j >= (uint32_t)kE) {
          const bool lower = (pb & j) == 0;
#pragma unroll
          for (int i = 0; i < kE; ++i) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, x[i], j / kE);
            const bool asc = ((pb + i) & k) == 0;
            x[i] = (lower == asc) ? min(x[i], y) : max(x[i], y);
          }
        } else if (j == 4) {
          lane_stage<kE, 4>(x, pb, k);
        } else if (j == 2) {
          lane_stage<kE, 2>(x, pb, k);
        } else {
          lane_stage<kE, 1>(x, pb, k);
        }
      }
    }
  } else {
#pragma unroll 1
    for (uint32_t k = 2; k <= 32u * kE; k <<= 1) {
      uint32_t j = k >> 1;
#pragma unroll 1
      for (; j >= (uint32_t)kE; j >>= 1) {
        const bool lower = (pb & j) == 0;  // j >= kE: partner is lane ^ (j / kE)
#pragma unroll
        for (int i = 0; i < kE; ++i) {
          const uint32_t y = __shfl_xor_sync(0xffffffffu, x[i], j / kE);
          const bool asc = ((pb + i) & k) == 0;
          x[i] = (lower == asc) ? min(x[i], y) : max(x[i], y);
        }
      }
      if (j == 16) { lane_stage<kE, 16>(x, pb, k); j = 8; }
      if (j == 8) { lane_stage<kE, 8>(x, pb, k); j = 4; }
      if (j == 4) { lane_stage<kE, 4>(x, pb, k); j = 2; }
      if (j == 2) { lane_stage<kE, 2>(x, pb, k); j = 1; }
      if (j == 1) lane_stage<kE, 1>(x, pb, k);
    }
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < kE; ++i) {
    const uint32_t p = lane * kE + i;
    sm[p + (p >> 5)] = x[i];
  }
  __syncwarp();
  uint32_t h = 0;
#pragma unroll
  for (int m = 0; m < kE; ++m) {
    const uint32_t t = m * 32 + lane;
    if (t < d) {
      const uint32_t y = sm[t + m];
      row[t] = y;
      h += y >= h0;
    }
  }
  __syncwarp();
  return warp_sum(h);
}

__global__ void __launch_bounds__(256) k_slot_sort_mid(SlotSort ss, const uint32_t* __restrict__ rows,
                                                       const unsigned int* __restrict__ nrows,
                                                       uint32_t* __restrict__ longrows,
                                                       unsigned int* __restrict__ nlong) {
  __shared__ uint32_t tile[8][8 * 33];
  uint32_t* sm = tile[threadIdx.x >> 5];
  const uint32_t nr = *nrows;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t idx = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); idx < nr; idx += warps) {
    const uint32_t r = rows[idx], d = ss.dplus[r];
    uint32_t* row = ss.pad + ss.pad_off[r];
    uint32_t h = 0;
    if (d <= 64) h = warp_sort_row<2>(row, d, ss.h0, sm);
    else if (d <= 128) h = warp_sort_row<4>(row, d, ss.h0, sm);
    else if (d <= 256) h = warp_sort_row<8>(row, d, ss.h0, sm);
    else {
      if (lane_id() == 0) longrows[atomicAdd(nlong, 1u)] = r;
      continue;
    }
    if (lane_id() == 0) ss.hcnt[r] = h;
  }
}

// Rows of 257..1024 entries (16/32 per lane, its own kernel for the register
// budget); longer rows are re-listed for the CTA sort.
__global__ void __launch_bounds__(128) k_slot_sort_mid2(SlotSort ss, const uint32_t* __restrict__ rows,
                                                        const unsigned int* __restrict__ nrows,
                                                        uint32_t* __restrict__ longrows,
                                                        unsigned int* __restrict__ nlong) {
  __shared__ uint32_t tile[4][32 * 33];
  uint32_t* sm = tile[threadIdx.x >> 5];
  const uint32_t nr = *nrows;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint32_t idx = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); idx < nr; idx += warps) {
    const uint32_t r = rows[idx], d = ss.dplus[r];
    uint32_t* row = ss.pad + ss.pad_off[r];
    uint32_t h = 0;
    if (d <= 512) h = warp_sort_row<16>(row, d, ss.h0, sm);
    else if (d <= 1024) h = warp_sort_row<32>(row, d, ss.h0, sm);
    else {
      if (lane_id() == 0) longrows[atomicAdd(nlong, 1u)] = r;
      continue;
    }
    if (lane_id() == 0) ss.hcnt[r] = h;
  }
}

// Listed rows (<= sort_max entries): one CTA each, SMEM bitonic sort over the
// next power of two.
constexpr uint32_t kSortMax = 16384;
__global__ void __launch_bounds__(256) k_slot_sort_block(SlotSort ss, const uint32_t* __restrict__ rows,
                                                         const unsigned int* __restrict__ nrows) {
  extern __shared__ uint32_t sk[];
  __shared__ uint32_t s_h;
  const uint32_t nr = *nrows;
  for (uint32_t idx = blockIdx.x; idx < nr; idx += gridDim.x) {
    const uint32_t r = rows[idx], d = ss.dplus[r];
    uint32_t* row = ss.pad + ss.pad_off[r];
    uint32_t P = 64;
    while (P < d) P <<= 1;
    if (threadIdx.x == 0) s_h = 0;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) sk[i] = i < d ? row[i] : 0xffffffffu;
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t t = threadIdx.x; t < P / 2; t += blockDim.x) {
          const uint32_t i = ((t & ~(j - 1)) << 1) | (t & (j - 1)), l = i + j;  // j is a power of two
          const uint32_t xi = sk[i], xl = sk[l];
          if ((xi > xl) == ((i & k) == 0)) {
            sk[i] = xl;
            sk[l] = xi;
          }
        }
        __syncthreads();
      }
    }
    uint32_t h = 0;
    for (uint32_t i = threadIdx.x; i < d; i += blockDim.x) {
      row[i] = sk[i];
      h += sk[i] >= ss.h0;
    }
    h = warp_sum(h);
    if (lane_id() == 0 && h) atomicAdd(&s_h, h);
    __syncthreads();
    if (threadIdx.x == 0) ss.hcnt[r] = s_h;
  }
}

// Every slot -> col[off[r], off[r+1]) with src = r, and (hot: its sorted
// suffix >= h0) -> colH[offH[r], offH[r+1]) as 16-bit offsets.  A warp takes
// 32 consecutive rows, whose outputs are one contiguous range of col: lanes
// walk that range 32 positions at a time (coalesced stores) and find their row
// by a 5-step search over the group's offsets in SMEM.
__global__ void __launch_bounds__(256) k_slot_compact(const uint32_t* __restrict__ off,
                                                      const uint64_t* __restrict__ pad_off,
                                                      const uint32_t* __restrict__ pad, uint32_t n,
                                                      uint32_t* __restrict__ col, uint32_t* __restrict__ src,
                                                      const uint32_t* __restrict__ offH, uint32_t h0,
                                                      uint16_t* __restrict__ colH) {
  __shared__ uint32_t s_off[8][33], s_hb[8][32], s_hs[8][32];
  __shared__ uint64_t s_po[8][32];
  const unsigned lane = lane_id(), w = threadIdx.x >> 5;
  const uint32_t warps = gridDim.x * (blockDim.x / 32);
  for (uint64_t r00 = (uint64_t)(blockIdx.x * (blockDim.x / 32) + w) * 32; r00 < n; r00 += (uint64_t)warps * 32) {
    const uint64_t r = r00 + lane;
    const uint32_t rr = r < n ? (uint32_t)r : n;
    const uint32_t o = off[rr];
    s_off[w][lane] = o;
    if (lane == 31) s_off[w][32] = off[r00 + 32 < n ? (uint32_t)(r00 + 32) : n];
    uint32_t hb = 0, hs = 0xffffffffu;
    uint64_t po = 0;
    if (r < n) {
      po = pad_off[rr];
      if (colH) {
        hb = offH[rr];
        hs = (off[rr + 1] - o) - (offH[rr + 1] - hb);  // first hot position of the row
      }
    }
    s_po[w][lane] = po;
    s_hb[w][lane] = hb;
    s_hs[w][lane] = hs;
    __syncwarp();
    const uint32_t a = s_off[w][0], b = s_off[w][32];
    for (uint32_t p0 = a + lane; p0 < b; p0 += 32 * 4) {  // 4 independent positions in flight
      uint32_t j[4], i[4], x[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t p = p0 + 32 * t;
        uint32_t jj = 0;
#pragma unroll
        for (uint32_t st = 16; st > 0; st >>= 1)
          if (s_off[w][jj + st] <= p) jj += st;
        j[t] = jj;
        i[t] = p - s_off[w][jj];
        x[t] = p < b ? pad[s_po[w][jj] + i[t]] : 0u;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t p = p0 + 32 * t;
        if (p >= b) break;
        col[p] = x[t];
        src[p] = (uint32_t)r00 + j[t];
        if (colH && i[t] >= s_hs[w][j[t]]) colH[s_hb[w][j[t]] + i[t] - s_hs[w][j[t]]] = (uint16_t)(x[t] - h0);
      }
    }
    __syncwarp();
  }
}

__global__ void k_pack_oriented(const uint32_t* __restrict__ src, const uint32_t* __restrict__ col, uint64_t E,
                                int b, uint64_t* __restrict__ keys) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = ((uint64_t)src[i] << b) | col[i];
}

__global__ void k_unpack_col(const uint64_t* __restrict__ keys, uint64_t E, int b, uint32_t* __restrict__ col) {
  const uint64_t mask = (b >= 32) ? 0xffffffffull : ((1ull << b) - 1);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E;
       i += (uint64_t)gridDim.x * blockDim.x)
    col[i] = (uint32_t)(keys[i] & mask);
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

// Degree rank from id-space undirected degrees: stable sort of (deg<<32 | id)
// on the degree bits -> id_of, rank_of, deg (by rank), max_deg.
void rank_vertices(tc_graph& g, const uint32_t* deg) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const int dev = g.device;
  DBuf<uint32_t> scal(1, s);
  TC_CUDA(cudaMemsetAsync(scal.get(), 0, sizeof(uint32_t), s));
  if (n) {
    k_max_u32<<<grid_gs(n, dev), kT, 0, s>>>(deg, n, scal.get());
    TC_LAUNCH();
  }
  g.max_deg = read_scalar(scal.get(), s);
  g.id_of.alloc(n ? n : 1, s);
  g.rank_of.alloc(n ? n : 1, s);
  g.deg.alloc(n ? n : 1, s);
  if (n) {
    DBuf<uint64_t> rk(n, s), rk2(n, s);
    k_rank_keys<<<grid_gs(n, dev), kT, 0, s>>>(deg, n, rk.get());
    TC_LAUNCH();
    const int db = bits_for(g.max_deg);
    uint64_t* sorted = radix_sort_u64(rk.get(), rk2.get(), n, 32, 32 + ((db + 7) / 8) * 8, s);
    k_rank_maps<<<grid_gs(n, dev), kT, 0, s>>>(sorted, n, g.id_of.get(), g.rank_of.get(), g.deg.get());
    TC_LAUNCH();
  }
}

// out-degrees by rank -> row offsets (g.off) and max d+
void row_offsets(tc_graph& g, const uint32_t* dplus) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  scan_exclusive<uint32_t>(LoadArray<uint32_t>{dplus}, g.off.get(), n, g.off.get() + n, s);
  DBuf<uint32_t> scal(1, s);
  TC_CUDA(cudaMemsetAsync(scal.get(), 0, sizeof(uint32_t), s));
  if (n) {
    k_max_u32<<<grid_gs(n, g.device), kT, 0, s>>>(dplus, n, scal.get());
    TC_LAUNCH();
  }
  g.max_dplus = read_scalar(scal.get(), s);
}

// Shared tail: the hot-window mirror of the finished oriented CSR.
// First rank of the hot window [h0, n) (graph.cuh).
uint32_t hot_window_start(uint32_t n) {
  const char* hb = getenv("TCB_HOT_BITS");  // tests: shrink the window to drive the cold path
  uint32_t hot = hb ? (uint32_t)strtoul(hb, nullptr, 10) : kHotBits;
  if (hot < 32) hot = 32;
  if (hot > kHotBits) hot = kHotBits;
  return n > hot ? n - hot : 0;
}

void finish_rows(tc_graph& g) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const uint64_t E = g.E;
  const int dev = g.device;
  // hot window mirror (graph.cuh): 16-bit copy of every row's members >= h0
  g.h0 = hot_window_start(n);
  g.offH.alloc((uint64_t)n + 1, s);
  {
    DBuf<uint32_t> hcnt(n ? n : 1, s);
    if (n) {
      k_hot_counts<<<grid_gs(n, dev), kT, 0, s>>>(g.off.get(), g.col.get(), n, g.h0, hcnt.get());
      TC_LAUNCH();
    }
    scan_exclusive<uint32_t>(LoadArray<uint32_t>{hcnt.get()}, g.offH.get(), n, g.offH.get() + n, s);
  }
  const uint32_t total_hot = n ? read_scalar(g.offH.get() + n, s) : 0;
  g.colH.alloc((uint64_t)total_hot + 16, s);
  TC_CUDA(cudaMemsetAsync(g.colH.get() + total_hot, 0, 16 * sizeof(uint16_t), s));
  if (E) {
    k_hot_scatter<<<grid_gs(E, dev), kT, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), E, g.h0, g.offH.get(),
                                                 g.colH.get());
    TC_LAUNCH();
  }
}

void alloc_rows(tc_graph& g) {
  cudaStream_t s = g.stream;
  g.col.alloc(g.E + 8, s);
  g.src.alloc(g.E ? g.E : 1, s);
  g.off.alloc((uint64_t)g.n + 1, s);
  // every col[0, E) is written by the build; the 8-word tail pad reads as "no id"
  TC_CUDA(cudaMemsetAsync(g.col.get() + g.E, 0xff, 8 * sizeof(uint32_t), s));
}

// ---- in-edge index (graph.cuh tc_graph::ine) ----------------------------------
// din(v) = deg(v) - d+(v): the in-edges of rank v, no edge pass.
struct InDeg {
  const uint32_t* off;
  const uint32_t* deg;
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const { return deg[v] - (off[v + 1] - off[v]); }
};

// max over pivots of deg(v) - d+(v) (the in-degree)
__global__ void k_max_din(const uint32_t* __restrict__ inoff, uint32_t n, unsigned int* __restrict__ out) {
  uint32_t m = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x)
    m = max(m, inoff[v + 1] - inoff[v]);
  m = __reduce_max_sync(0xffffffffu, m);
  if ((threadIdx.x & 31u) == 0 && m) atomicMax(out, m);
}

// Every oriented edge e = u->v to its head's slot (one atomic per edge: a
// warp's 32 edges come from one or two rows, so their heads rarely repeat),
// as a 32-byte level-1 item record
// (graph.cuh irec, one 256-bit store): the suffix geometry comes from u's row descriptor, read in
// edge order (consecutive edges share their row).  With ccnt (rows [r0, n):
// core members of a dense row, else 0), bit `slot` of dbits marks a dense
// item: u's row is dense and e is not its last edge.
// The slot atomics of the hub heads (the top `nhub` ranks: degrees ascend
// with rank, so these take the largest share of the in-edges) are aggregated
// per CTA tile in shared memory: one global atomic per (tile, hub head) claims
// the tile's run of slots, the per-edge SMEM atomic's return value places the
// edge inside it.  Other heads take one global atomic per edge.  Measured
// at C4 (profiles/README.md): 10.0 -> 7.4 ms with 512 hub counters (4096:
// 8.3 ms, the per-tile reset and the SMEM footprint start to cost).
template <int kInEdges>
__global__ void __launch_bounds__(256) k_in_scatter(const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
                                                    uint64_t E, uint32_t* __restrict__ cur,
                                                    const uint4* __restrict__ rowd, uint32_t r0,
                                                    uint4* __restrict__ irec, const uint32_t* __restrict__ ccnt,
                                                    uint32_t* __restrict__ dbits, uint32_t hub_lo, uint32_t nhub) {
  // kInEdges independent edges per thread per tile (coalesced per k).  The
  // row descriptor loads (which need only u) are issued next to the slot
  // atomics: two dependent round trips per tile, not three.
  extern __shared__ uint32_t s_hub[];  // [nhub] counts, then bases
  __shared__ uint32_t s_list[256 * kInEdges];
  __shared__ uint32_t s_nlist;
  for (uint32_t i = threadIdx.x; i < nhub; i += blockDim.x) s_hub[i] = 0;
  if (threadIdx.x == 0) s_nlist = 0;
  __syncthreads();
  const uint64_t tile = (uint64_t)blockDim.x * kInEdges;
  for (uint64_t base = (uint64_t)blockIdx.x * tile; base < E; base += (uint64_t)gridDim.x * tile) {
    uint32_t v[kInEdges], u[kInEdges], slot[kInEdges], cc[kInEdges];
    uint4 d0[kInEdges], d1[kInEdges];
    bool ok[kInEdges];
#pragma unroll
    for (int k = 0; k < kInEdges; ++k) {
      const uint64_t e = base + (uint64_t)k * blockDim.x + threadIdx.x;
      ok[k] = e < E;
      v[k] = ok[k] ? col[e] : 0u;
      u[k] = ok[k] ? src[e] : r0;
    }
#pragma unroll
    for (int k = 0; k < kInEdges; ++k) {
      const uint64_t i = u[k] - r0;
      d0[k] = rowd[2 * i];
      d1[k] = rowd[2 * i + 1];
      cc[k] = dbits ? ccnt[i] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kInEdges; ++k) {
      slot[k] = 0;
      if (!ok[k]) continue;
      if (v[k] >= hub_lo) {
        const uint32_t h = v[k] - hub_lo;
        slot[k] = atomicAdd(&s_hub[h], 1u);
        if (slot[k] == 0) s_list[atomicAdd(&s_nlist, 1u)] = h;
      } else {
        slot[k] = atomicAdd(&cur[v[k]], 1u);
      }
    }
    if (nhub) {
      __syncthreads();
      const uint32_t nl = s_nlist;
      for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
        const uint32_t h = s_list[i];
        s_hub[h] = atomicAdd(&cur[hub_lo + h], s_hub[h]);
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kInEdges; ++k)
        if (ok[k] && v[k] >= hub_lo) slot[k] += s_hub[v[k] - hub_lo];
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) s_hub[s_list[i]] = 0;
      if (threadIdx.x == 0) s_nlist = 0;
      __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < kInEdges; ++k) {
      if (!ok[k]) continue;
      const uint64_t e = base + (uint64_t)k * blockDim.x + threadIdx.x;
      const RowGeo r(d0[k], d1[k]);
      uint4 geo = make_uint4(0, 0, 0, 0);
      uint64_t mo = 0;
      const uint32_t a = (uint32_t)e + 1;
      if (a < r.end) {
        const uint32_t ce = r.cold_end();
        geo = a >= ce ? make_uint4(r.O + (a - ce), r.Ht, 0, 0) : make_uint4(r.O, r.Ht, a, ce);
        if (geo.y > geo.x) mo = r.rowbase + r.masks().P((uint32_t)e - r.beg);
      }
      st256(irec + 2 * (uint64_t)slot[k], geo, make_uint4((uint32_t)e, u[k], (uint32_t)mo, (uint32_t)(mo >> 32)));
      if (a < r.end && cc[k] != 0) atomicOr(&dbits[slot[k] >> 5], 1u << (slot[k] & 31));
    }
  }
}

// ---- dense core (graph.cuh RowGeo) -------------------------------------------
// Core members of row u: its hot suffix entries >= cb - h0 (colH is sorted
// per row), found by binary search; the row is dense with >= core_min.
// ccnt[u - r0] = core members if dense, else 0.
__global__ void k_core_rows(const uint32_t* __restrict__ offH, const uint16_t* __restrict__ colH, uint32_t r0,
                            uint32_t n, uint32_t cbh, uint32_t core_min, uint32_t* __restrict__ ccnt) {
  for (uint64_t u = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = offH[u], hi = offH[u + 1];
    const uint32_t end = hi;
    while (lo < hi) {
      const uint32_t m = lo + ((hi - lo) >> 1);  // entry indices: lo + hi may pass 2^32
      if (colH[m] < cbh) lo = m + 1; else hi = m;
    }
    const uint32_t c = end - lo;
    ccnt[u - r0] = (c >= core_min && c > 0) ? c : 0u;
  }
}

struct DenseFlag {
  const uint32_t* ccnt;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return ccnt[i] ? 1u : 0u; }
};

// Row descriptors (32 bytes per rank, graph.cuh RowGeo), without rowbase.
__global__ void k_rowdesc(const uint32_t* __restrict__ off, const uint32_t* __restrict__ offH, uint32_t r0,
                          uint32_t n, const uint32_t* __restrict__ ccnt, const uint32_t* __restrict__ dpos,
                          uint4* __restrict__ rowd) {
  for (uint64_t u = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = ccnt ? ccnt[u - r0] : 0u;
    const uint32_t Hf = offH[u + 1];
    rowd[2 * (u - r0)] = make_uint4(off[u], off[u + 1], offH[u], Hf - c);
    rowd[2 * (u - r0) + 1] = make_uint4(Hf, c ? dpos[u - r0] : kNoDense, 0, 0);
  }
}

// Mask bytes of row r0 + i (the sparse hot part, RowGeo::masks).
struct RowBytesGeo {
  const uint4* rowd;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    return RowGeo(rowd[2 * i], rowd[2 * i + 1]).masks().total();
  }
};
__global__ void k_rowbase_put(const uint64_t* __restrict__ rb, uint32_t nr, uint4* __restrict__ rowd) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 b = rowd[2 * i + 1];
    b.z = (uint32_t)rb[i];
    b.w = (uint32_t)(rb[i] >> 32);
    rowd[2 * i + 1] = b;
  }
}

// Dense in-edge list: in-edge i = {e, u} of pivot v is a dense item when u's
// row is dense and its suffix after v is non-empty (dflag, k_in_scatter).
// Dense-item flags as a bit array over the in-edge slots (E bits: L2-resident
// while the in-edge scatter sets them) and their word popcount prefix wp: the
// dense-list position of slot i is wp[i / 32] + the set bits below it.
struct WordPopc {
  const uint32_t* w;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return __popc(w[i]); }
};
__device__ __forceinline__ uint32_t dense_pos(const uint32_t* __restrict__ dbits, const uint32_t* __restrict__ wp,
                                              uint64_t i) {
  return wp[i >> 5] + __popc(dbits[i >> 5] & ((1u << (i & 31)) - 1u));
}
__global__ void k_dense_scatter(const uint4* __restrict__ irec, uint64_t E, const uint32_t* __restrict__ dbits,
                                const uint32_t* __restrict__ wp, const uint32_t* __restrict__ dpos, uint32_t r0,
                                uint32_t* __restrict__ dine) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t w = dbits[i >> 5];
    if ((w >> (i & 31)) & 1u) dine[wp[i >> 5] + __popc(w & ((1u << (i & 31)) - 1u))] = dpos[irec[2 * i + 1].y - r0];
  }
}
// Dense segments of pivot v: its dense items [pos(inoff[v]), pos(inoff[v+1]))
struct DenseSegs {
  const uint32_t* inoff;
  const uint32_t* dbits;
  const uint32_t* wp;
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const {
    const uint32_t c = dense_pos(dbits, wp, inoff[v + 1]) - dense_pos(dbits, wp, inoff[v]);
    return (c + kDenseSeg - 1) / kDenseSeg;
  }
};
__global__ void k_dense_segs(const uint32_t* __restrict__ inoff, const uint32_t* __restrict__ dbits,
                             const uint32_t* __restrict__ wp, uint32_t n, const uint32_t* __restrict__ dsoff,
                             uint4* __restrict__ dseg) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = dense_pos(dbits, wp, inoff[v]), b = dense_pos(dbits, wp, inoff[v + 1]);
    uint32_t s = dsoff[v];
    for (uint32_t i = a; i < b; i += kDenseSeg) dseg[s++] = make_uint4((uint32_t)v, i, min(i + kDenseSeg, b), 0);
  }
}
__global__ void k_dense_rows(const uint4* __restrict__ rowd, uint32_t r0, uint32_t nr, uint32_t* __restrict__ drow) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t didx = rowd[2 * i + 1].y;
    if (didx != kNoDense) drow[didx] = r0 + (uint32_t)i;
  }
}

// Core bitmaps: one warp per dense row sets the bits of its core members.
__global__ void k_core_fill(const uint4* __restrict__ rowd, uint32_t nr, const uint16_t* __restrict__ colH,
                            uint32_t cbh, uint32_t words, uint32_t* __restrict__ cbits) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nr;
       i += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const RowGeo r(rowd[2 * i], rowd[2 * i + 1]);
    if (r.didx == kNoDense) continue;
    uint32_t* bm = cbits + (uint64_t)r.didx * words;
    for (uint32_t p = r.Ht + lane; p < r.Hf; p += 32) {
      const uint32_t y = colH[p] - cbh;
      atomicOr(&bm[y >> 5], 1u << (y & 31));
    }
  }
}

// First rank with deg > 0 (degrees ascend with rank): the isolated vertices
// are ranks [0, r0).
__global__ void k_first_nonisolated(const uint32_t* __restrict__ deg, uint32_t n, uint32_t* __restrict__ r0) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t m = lo + (hi - lo) / 2;
    if (deg[m] < 1) lo = m + 1; else hi = m;
  }
  *r0 = lo;
}

// Plan capacities: work segments per pivot class (per-vertex superset: d+ = 0
// pivots in the warp bin).
__global__ void k_plan_caps(PivotClass pc, uint32_t r0, uint32_t n, unsigned long long* __restrict__ tot) {
  unsigned long long t[4] = {0, 0, 0, 0};
  for (uint64_t v = r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t din = 0;
    const int c = pc((uint32_t)v, din);
    if (c >= 0) {
      const uint32_t per = segs_per_class(c);
      const unsigned long long ns = (din + per - 1) / per;
      t[0] += c == 0 ? ns : 0;
      t[1] += c == 1 ? ns : 0;
      t[2] += c == 2 ? ns : 0;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long w = warp_sum(t[i]);
    if ((threadIdx.x & 31u) == 0 && w) atomicAdd(&tot[i], w);
  }
}

// Sorted unique canonical id-space keys (edge-list route) -> ranks ->
// oriented CSR: orient each key by rank, radix sort, split.
void finalize(tc_graph& g, DBuf<uint64_t>& ukeys, uint64_t E) {
  cudaStream_t s = g.stream;
  PhaseLog pl(s);
  const uint32_t n = g.n;
  const int b = g.id_bits;
  const int dev = g.device;
  if (E >= (1ull << 32)) fail(TC_ERANGE, "graph has >= 2^32 undirected edges (u32 oriented offsets)");
  g.E = E;
  {
    DBuf<uint32_t> deg(n ? n : 1, s);
    TC_CUDA(cudaMemsetAsync(deg.get(), 0, sizeof(uint32_t) * (n ? n : 1), s));
    if (E) {
      k_degree<<<grid_gs(E, dev), kT, 0, s>>>(ukeys.get(), E, b, deg.get());
      TC_LAUNCH();
    }
    rank_vertices(g, deg.get());
  }
  pl.mark("fin_rank");
  alloc_rows(g);
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
  pl.mark("fin_orient_sort");
  row_offsets(g, dplus.get());
  finish_rows(g);
  pl.mark("fin_rows");
}

// Shared tail of both build routes: the in-edge index and the count-plan
// capacities (one small read-back; the count itself never synchronises).
void finish_graph(tc_graph& g) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const uint64_t E = g.E;
  const int dev = g.device;
  PhaseLog pl(s);
  g.r0 = 0;
  if (n) {
    DBuf<uint32_t> r0(1, s);
    k_first_nonisolated<<<1, 1, 0, s>>>(g.deg.get(), n, r0.get());
    TC_LAUNCH();
    g.r0 = read_scalar(r0.get(), s);
  }
  const uint32_t nr = n - g.r0;
  // dense core: rows with >= core_min members among the top core_bits ranks
  // (TCB_CORE_BITS / TCB_CORE_MIN: tests shrink the core to drive the dense
  // path on small graphs; TCB_CORE_BITS=0 disables it)
  // default: kCoreBits; half of it for small graphs (n <= 2^17), where the
  // core rows are few and short (C1 0.149 -> 0.140 ms per count; C3 and C4
  // are fastest at kCoreBits: profiles/README.md)
  uint32_t core_bits = env_u32("TCB_CORE_BITS", n <= (1u << 17) ? kCoreBits / 2 : kCoreBits) & ~31u;
  if (core_bits > 32u * 32u * kCoreWordsMax) core_bits = 32u * 32u * kCoreWordsMax;
  const uint32_t core_min = std::max<uint32_t>(1, env_u32("TCB_CORE_MIN", core_bits / 32));
  g.cb = 0;
  g.core_words = 0;
  g.ndense = 0;
  g.cbits.release();
  DBuf<uint32_t> ccnt, dpos;
  if (nr && core_bits && n >= core_bits && n - core_bits >= g.h0) {
    // core = ranks [cb, n), cb - h0 a multiple of 32 so the core words are
    // words of the joins' hot bitmap; n - cb <= core_bits
    const uint32_t cbh = (n - core_bits - g.h0 + 31) & ~31u, cb = g.h0 + cbh;
    ccnt.alloc(nr, s);
    dpos.alloc((uint64_t)nr + 1, s);
    k_core_rows<<<grid_gs(nr, dev), kT, 0, s>>>(g.offH.get(), g.colH.get(), g.r0, n, cbh, core_min, ccnt.get());
    TC_LAUNCH();
    scan_exclusive<uint32_t>(DenseFlag{ccnt.get()}, dpos.get(), nr, dpos.get() + nr, s);
    const uint32_t nd = read_scalar(dpos.get() + nr, s);
    if (nd > 0) {
      g.cb = cb;
      g.core_words = (n - cb + 31) / 32;
      g.ndense = nd;
      g.core_min = core_min;
    } else {
      ccnt.release();  // no dense rows: every row stays sparse
    }
  }
  pl.mark("fin_core_rows");
  g.rowd.alloc(2 * (uint64_t)(nr ? nr : 1), s);
  if (nr) {
    k_rowdesc<<<grid_gs(nr, dev), kT, 0, s>>>(g.off.get(), g.offH.get(), g.r0, n, g.ndense ? ccnt.get() : nullptr,
                                              dpos.get(), g.rowd.get());
    TC_LAUNCH();
  }
  if (g.ndense) {
    g.cbits.alloc((uint64_t)g.ndense * g.core_words, s);
    TC_CUDA(cudaMemsetAsync(g.cbits.get(), 0, sizeof(uint32_t) * (uint64_t)g.ndense * g.core_words, s));
    k_core_fill<<<grid_gs(32 * (uint64_t)nr, dev), kT, 0, s>>>(g.rowd.get(), nr, g.colH.get(), g.cb - g.h0,
                                                                g.core_words, g.cbits.get());
    TC_LAUNCH();
  }
  pl.mark("fin_rowdesc_cbits");
  // per-vertex mask base of every row (graph property; RowGeo::rowbase)
  g.mask_total = 0;
  if (nr) {
    DBuf<uint64_t> rb((uint64_t)nr + 1, s);
    scan_exclusive<uint64_t>(RowBytesGeo{g.rowd.get()}, rb.get(), nr, rb.get() + nr, s);
    k_rowbase_put<<<grid_gs(nr, dev), kT, 0, s>>>(rb.get(), nr, g.rowd.get());
    TC_LAUNCH();
    g.mask_total = read_scalar(rb.get() + nr, s);
  }
  pl.mark("fin_rowbase");
  // in-edge index (+ the dense-item flag of every slot)
  g.inoff.alloc((uint64_t)n + 1, s);
  scan_exclusive<uint32_t>(InDeg{g.off.get(), g.deg.get()}, g.inoff.get(), n, g.inoff.get() + n, s);
  g.irec.alloc(2 * (E ? E : 1), s);
  g.max_din = 0;
  if (n) {
    DBuf<unsigned int> md(1, s);
    TC_CUDA(cudaMemsetAsync(md.get(), 0, sizeof(unsigned int), s));
    k_max_din<<<grid_gs(n, dev), kT, 0, s>>>(g.inoff.get(), n, md.get());
    TC_LAUNCH();
    g.max_din = read_scalar(md.get(), s);
  }
  DBuf<uint32_t> dbits;
  const uint64_t nwords = (E + 31) / 32;
  if (E) {
    if (g.ndense) {
      dbits.alloc(nwords + 1, s);
      TC_CUDA(cudaMemsetAsync(dbits.get(), 0, sizeof(uint32_t) * (nwords + 1), s));
    }
    DBuf<uint32_t> cur(n, s);
    TC_CUDA(cudaMemcpyAsync(cur.get(), g.inoff.get(), sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    const uint32_t ik = env_u32("TCB_INSC_K", 4);
    const uint32_t nhub = std::min<uint32_t>(n, env_u32("TCB_INSC_HUB", 512));
    auto insc = ik >= 8 ? k_in_scatter<8> : ik >= 2 ? k_in_scatter<4> : k_in_scatter<1>;
    const size_t hub_smem = sizeof(uint32_t) * nhub;
    if (hub_smem > 48 * 1024)
      TC_CUDA(cudaFuncSetAttribute(insc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hub_smem));
    insc<<<grid_gs(E, dev), kT, hub_smem, s>>>(g.col.get(), g.src.get(), E, cur.get(), g.rowd.get(), g.r0,
                                               g.irec.get(), g.ndense ? ccnt.get() : nullptr, dbits.get(),
                                               n - nhub, nhub);
    TC_LAUNCH();
  }
  pl.mark("fin_in_scatter");
  // dense in-edge list and its segments (k_join_dense)
  g.dine.release();
  g.dseg.release();
  g.drow.release();
  g.ndine = 0;
  g.dsoff.alloc((uint64_t)n + 1, s);
  TC_CUDA(cudaMemsetAsync(g.dsoff.get(), 0, sizeof(uint32_t) * ((uint64_t)n + 1), s));
  if (g.ndense && E) {
    DBuf<uint32_t> wp(nwords + 2, s);
    scan_exclusive<uint32_t>(WordPopc{dbits.get()}, wp.get(), nwords + 1, wp.get() + nwords + 1, s);
    g.ndine = read_scalar(wp.get() + nwords + 1, s);
    g.dine.alloc(g.ndine ? g.ndine : 1, s);
    if (g.ndine) {
      k_dense_scatter<<<grid_gs(E, dev), kT, 0, s>>>(g.irec.get(), E, dbits.get(), wp.get(), dpos.get(), g.r0,
                                                     g.dine.get());
      TC_LAUNCH();
    }
    scan_exclusive<uint32_t>(DenseSegs{g.inoff.get(), dbits.get(), wp.get()}, g.dsoff.get(), n, g.dsoff.get() + n,
                             s);
    const uint32_t nseg = read_scalar(g.dsoff.get() + n, s);
    g.dseg.alloc(nseg ? nseg : 1, s);
    if (nseg) {
      k_dense_segs<<<grid_gs(n, dev), kT, 0, s>>>(g.inoff.get(), dbits.get(), wp.get(), n, g.dsoff.get(),
                                                  g.dseg.get());
      TC_LAUNCH();
    }
    dbits.release();
    g.drow.alloc(g.ndense, s);
    k_dense_rows<<<grid_gs(nr, dev), kT, 0, s>>>(g.rowd.get(), g.r0, nr, g.drow.get());
    TC_LAUNCH();
  }
  ccnt.release();
  dpos.release();
  pl.mark("fin_dense_list");
  DBuf<unsigned long long> tot(4, s);
  TC_CUDA(cudaMemsetAsync(tot.get(), 0, 4 * sizeof(unsigned long long), s));
  if (nr) {
    k_plan_caps<<<grid_gs(nr, dev), kT, 0, s>>>(PivotClass{g.off.get(), g.offH.get(), g.inoff.get(), true}, g.r0,
                                               n, tot.get());
    TC_LAUNCH();
  }
  unsigned long long h[4];
  TC_CUDA(cudaMemcpyAsync(h, tot.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  for (int c = 0; c < 3; ++c) g.seg_cap[c] = h[c];
  g.part_bounds.clear();
  g.part_bounds_P = 0;
  g.part_kr.clear();
  g.part_kr_P = 0;
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
  finish_graph(g);
}

void build_from_csr(tc_graph& g, const uint64_t* d_off, const uint32_t* d_nbrs, uint32_t n, uint64_t num_edges,
                    bool strict, const CsrFeed* feed) {
  cudaStream_t s = g.stream;
  const int dev = g.device;
  g.n = n;
  g.id_bits = n > 1 ? bits_for((uint64_t)n - 1) : 1;
  const uint64_t total = 2 * num_edges;  // may exceed 2^32: slot offsets are u64
  if (num_edges >= (1ull << 32)) fail(TC_ERANGE, "graph has >= 2^32 undirected edges (u32 oriented offsets)");
  PhaseLog pl(s);
  // The neighbour array streams in behind everything that needs only the
  // offsets: pieces of kFeedChunk entries (8 M from pageable memory, which
  // goes through pinned bounce slots), one event each (feed.cu).
  const bool stream_in = feed && total;
  const char* fc = getenv("TCB_FEED_CHUNK");  // tests: many small pieces
  uint64_t chunk = fc ? std::max<uint64_t>(1, strtoull(fc, nullptr, 10)) : kFeedChunk;
  std::unique_ptr<PieceFeed> pf;
  uint64_t piece = total ? total : 1;
  if (stream_in) {
    if (!fc && pageable_host(feed->h_nbrs)) chunk = std::min<uint64_t>(chunk, 1ull << 23);
    piece = feed->h_off ? chunk : total;
    pf.reset(new PieceFeed(feed->h_nbrs, feed->d_dst, total, piece, s));
  }
  const uint32_t K = pf ? pf->pieces() : 1;
  const uint32_t nn = n ? n : 1;
  DBuf<uint32_t> deg(nn, s), big(total / kBigRow + 1, s);
  DBuf<unsigned int> cnts(2, s);  // big rows / long rank-space rows
  DBuf<unsigned int> queues(K, s);
  DBuf<int> bad(1, s);
  DBuf<unsigned long long> upper(1, s);
  TC_CUDA(cudaMemsetAsync(cnts.get(), 0, 2 * sizeof(unsigned int), s));
  TC_CUDA(cudaMemsetAsync(queues.get(), 0, K * sizeof(unsigned int), s));
  TC_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  TC_CUDA(cudaMemsetAsync(upper.get(), 0, sizeof(unsigned long long), s));
  if (n) {
    k_csr_deg<<<grid_gs(n, dev), kT, 0, s>>>(d_off, n, deg.get(), big.get(), cnts.get(), bad.get());
    TC_LAUNCH();
  }
  const uint64_t off_n = n ? read_scalar(d_off + n, s) : 0;
  if (read_scalar(bad.get(), s) || off_n != total || (n && read_scalar(d_off, s) != 0)) {
    if (strict) fail(TC_EPARSE, "corrupt CSR cache offsets (line 1)");
    fail(TC_EINVAL, "Graph: inconsistent CSR arrays");
  }
  // hub rows -> chunk list (device: chunk counts, scan, fill)
  const uint32_t nbig = read_scalar(cnts.get(), s);
  DBuf<uint32_t> choff((uint64_t)nbig + 1, s);
  uint32_t nch = 0;
  if (nbig) {
    kl_scan_chunks(big.get(), nbig, d_off, choff.get(), s);
    nch = read_scalar(choff.get() + nbig, s);
  }
  DBuf<Chunk> chunks(nch ? nch : 1, s);
  DBuf<uint32_t> ccount(nch ? nch : 1, s), cbase(nch ? nch : 1, s);
  if (nch) {
    k_chunk_fill<<<ceil_div(nbig, 256), 256, 0, s>>>(big.get(), nbig, d_off, choff.get(), chunks.get());
    TC_LAUNCH();
  }
  rank_vertices(g, deg.get());
  deg.release();
  // padded rank-space slots: deg(u) entries each, by rank
  DBuf<uint64_t> pad_off((uint64_t)nn + 1, s);
  DBuf<uint32_t> pad(total ? total : 1, s);
  scan_exclusive<uint64_t>(DegLoad64{g.deg.get()}, pad_off.get(), n, pad_off.get() + n, s);
  DBuf<uint32_t> dplus(nn, s);
  TC_CUDA(cudaMemsetAsync(dplus.get(), 0, sizeof(uint32_t) * nn, s));
  pl.mark("csr_rank");
  RowCtx cx{d_off, d_nbrs, g.rank_of.get(), n, dplus.get(), pad_off.get(), pad.get(), strict ? 1 : 0};
  // per piece: orient its rows, then sort their slots in place (hot counts)
  g.h0 = hot_window_start(n);
  const char* smx = getenv("TCB_ROWSORT_MAX");  // tests: force the radix fallback on small graphs
  const uint32_t sort_max = std::min<uint32_t>(smx ? (uint32_t)strtoul(smx, nullptr, 10) : kSortMax, kSortMax);
  DBuf<uint32_t> hcnt(nn, s), huge(nn, s), rows_a(nn, s), rows_b(nn, s);
  DBuf<unsigned int> lists(3 * K + 1, s);  // per piece: mid / long / CTA list counts; + huge count
  TC_CUDA(cudaMemsetAsync(hcnt.get(), 0, sizeof(uint32_t) * nn, s));
  TC_CUDA(cudaMemsetAsync(lists.get(), 0, (3 * K + 1) * sizeof(unsigned int), s));
  const SlotSort ss{g.rank_of.get(), pad_off.get(), pad.get(), dplus.get(), g.h0, sort_max, hcnt.get(),
                    huge.get(), lists.get() + 3 * K};
  uint32_t Pb = 64;
  while (Pb < sort_max) Pb <<= 1;
  TC_CUDA(cudaFuncSetAttribute(k_slot_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(Pb * sizeof(uint32_t))));
  const unsigned gw = (unsigned)num_sms(dev) * 8;
  uint32_t lo = 0;
  for (uint32_t k = 0; k < K && total; ++k) {
    // rows whose entries all lie in the first k+1 pieces
    uint32_t hi = n;
    if (stream_in && k + 1 < K) {
      const uint64_t e = (uint64_t)(k + 1) * piece;
      hi = (uint32_t)(std::upper_bound(feed->h_off, feed->h_off + (uint64_t)n + 1, e) - feed->h_off) - 1;
    }
    if (pf) pf->wait_piece(k, s);
    if (hi > lo) {
      k_csr_rows<<<gw, 256, 0, s>>>(cx, lo, hi, queues.get() + k, upper.get(), bad.get());
      TC_LAUNCH();
      if (nch) {
        k_csr_chunks<0><<<gw, 256, 0, s>>>(cx, chunks.get(), nch, lo, hi, ccount.get(), cbase.get(), upper.get(),
                                           bad.get());
        TC_LAUNCH();
        k_chunk_bases<<<ceil_div(nch, 256), 256, 0, s>>>(chunks.get(), nch, lo, hi, ccount.get(), cbase.get());
        TC_LAUNCH();
        k_csr_chunks<1><<<gw, 256, 0, s>>>(cx, chunks.get(), nch, lo, hi, ccount.get(), cbase.get(), upper.get(),
                                           bad.get());
        TC_LAUNCH();
      }
      unsigned int* cnt3 = lists.get() + 3 * k;
      k_slot_sort_warp<<<gw, 256, 0, s>>>(ss, lo, hi, rows_a.get(), cnt3);
      TC_LAUNCH();
      k_slot_sort_mid<<<gw, 256, 0, s>>>(ss, rows_a.get(), cnt3, rows_b.get(), cnt3 + 1);
      TC_LAUNCH();
      k_slot_sort_mid2<<<gw * 2, 128, 0, s>>>(ss, rows_b.get(), cnt3 + 1, rows_a.get(), cnt3 + 2);
      TC_LAUNCH();
      k_slot_sort_block<<<gw, 256, Pb * sizeof(uint32_t), s>>>(ss, rows_a.get(), cnt3 + 2);
      TC_LAUNCH();
    }
    lo = hi;
  }
  pl.mark("csr_orient_sort");
  const uint64_t E = read_scalar(upper.get(), s);
  const int badv = read_scalar(bad.get(), s);
  if (badv && strict) fail(TC_EPARSE, "corrupt CSR cache adjacency (line 1)");
  if (badv) fail(TC_EINVAL, "Graph: neighbor id out of range");
  if (E != num_edges) fail(TC_EINVAL, "Graph: inconsistent CSR arrays (asymmetric adjacency)");
  g.E = E;
  alloc_rows(g);
  row_offsets(g, dplus.get());
  if (n && read_scalar(g.off.get() + n, s) != E)
    fail(TC_EINVAL, "Graph: inconsistent CSR arrays (asymmetric adjacency)");
  const uint32_t nhuge = read_scalar(lists.get() + 3 * K, s);
  pl.mark("csr_offsets");
  if (nhuge == 0) {
    // slots -> col/src + the hot mirror in one pass
    g.offH.alloc((uint64_t)n + 1, s);
    scan_exclusive<uint32_t>(LoadArray<uint32_t>{hcnt.get()}, g.offH.get(), n, g.offH.get() + n, s);
    const uint32_t total_hot = n ? read_scalar(g.offH.get() + n, s) : 0;
    g.colH.alloc((uint64_t)total_hot + 16, s);
    TC_CUDA(cudaMemsetAsync(g.colH.get() + total_hot, 0, 16 * sizeof(uint16_t), s));
    pl.mark("csr_hot_offsets");
    if (E) {
      k_slot_compact<<<gw, 256, 0, s>>>(g.off.get(), pad_off.get(), pad.get(), n, g.col.get(), g.src.get(),
                                        g.offH.get(), g.h0, g.colH.get());
      TC_LAUNCH();
    }
    pl.mark("csr_compact_hot");
  } else {
    // rows longer than the CTA sort: move the slots, one global radix sort
    k_slot_compact<<<gw, 256, 0, s>>>(g.off.get(), pad_off.get(), pad.get(), n, g.col.get(), g.src.get(), nullptr,
                                      0, nullptr);
    TC_LAUNCH();
    DBuf<uint64_t> k1(E, s), k2(E, s);
    k_pack_oriented<<<grid_gs(E, dev), kT, 0, s>>>(g.src.get(), g.col.get(), E, g.id_bits, k1.get());
    TC_LAUNCH();
    uint64_t* sorted = radix_sort_u64(k1.get(), k2.get(), E, 0, 2 * g.id_bits, s);
    k_unpack_col<<<grid_gs(E, dev), kT, 0, s>>>(sorted, E, g.id_bits, g.col.get());
    TC_LAUNCH();
    k1.release();
    k2.release();
    pad.release();
    finish_rows(g);
    pl.mark("csr_radix_fallback");
  }
  finish_graph(g);
  pl.mark("csr_in_index");
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
  // > kExportChunk directed entries (TCB_EXPORT_CHUNK for tests): source-id
  // ranges of at most that many entries, each keyed, sorted and written on
  // its own (radix_sort_u64 sorts < 2^32 keys)
  const uint64_t cmax = std::max<uint64_t>(1, std::min<uint64_t>(env_u32("TCB_EXPORT_CHUNK", kExportChunk),
                                                                 kExportChunk));
  if (2 * E > cmax) {
    std::vector<uint64_t> ho((uint64_t)n + 1);
    TC_CUDA(cudaMemcpyAsync(ho.data(), d_off, ho.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    DBuf<uint64_t> k1(cmax, s), k2(cmax, s);
    DBuf<unsigned long long> cnt(1, s);
    uint32_t u_lo = 0;
    while (u_lo < n) {
      // largest u_hi with off[u_hi] - off[u_lo] <= cmax (a row longer than cmax alone)
      uint32_t u_hi = (uint32_t)(std::upper_bound(ho.begin() + u_lo, ho.end(), ho[u_lo] + cmax) - ho.begin()) - 1;
      if (u_hi <= u_lo) u_hi = u_lo + 1;
      const uint64_t base = ho[u_lo], m = ho[u_hi] - base;
      if (m > cmax) fail(TC_ERANGE, "export_csr: a row longer than the export chunk");
      if (m) {
        TC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(unsigned long long), s));
        k_directed_keys_range<<<grid_gs(E, dev), kT, 0, s>>>(g.src.get(), g.col.get(), E, g.id_of.get(), b, u_lo,
                                                             u_hi, k1.get(), cnt.get());
        TC_LAUNCH();
        uint64_t* sorted = radix_sort_u64(k1.get(), k2.get(), m, 0, b + bits_for(u_hi - u_lo - 1 ? u_hi - u_lo - 1 : 1), s);
        k_low_bits<<<grid_gs(m, dev), kT, 0, s>>>(sorted, m, b, d_nbrs + base);
        TC_LAUNCH();
      }
      u_lo = u_hi;
    }
    return;
  }
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
