// count.cu -- the hot path: degree-binned advance and fused SMEM join over the
// level-1 frontier index, warp-shuffle/atomic reduction (north_star (2)-(4)).
//
// Reference path replaced (matcher.cpp): count_triangles :301-303 -> match
// :249-299 -> count_final_level :204-245, whose inner loop visits every x in
// N(u) for each level-1 row (u,w) and tests has_edge(w,x) by binary search
// (graph.cpp:23-31).
//
// Formulation on the (deg,id)-ordered DAG in rank space:
//   every triangle a<b<c (ranks) has oriented edges a->b, a->c, b->c and is
//   found exactly once with PIVOT v=b: for each in-edge u->v (u=a, a
//   frontier item, frontier.cu) the advance expands the candidate wedges
//   x = the suffix of N+(u) after v (x=c is in it), and the join keeps x iff
//   x in N+(v).  Candidate wedges J = sum_u C(d+(u),2) (4.2e10 at RMAT s24)
//   instead of the reference's sum_rows deg(u), and 4.4x fewer than the
//   wedge-stream W.
// Bins (by d+(v)):
//   warp bin  d+(v) <= kWarpMaxDeg: one warp per segment, warp-private hash;
//             items are (b,e) ranges of the 32-bit col[]
//   CTA bin   larger: the CTA stages N+(v) once per segment -- members in the
//             hot window [h0,n) as a bitmap, the rest in a hash -- and its
//             warps share it.  Items are {hb,he,cb,ce}: the suffix split into
//             its hot part (16-bit colH, graph.cuh) and cold part (32-bit col)
// Chunks: suffixes are streamed as 16-byte int4 loads (8 hot / 4 cold ids),
//   load-balanced across lanes by a ballot/redux start mask, segment chunks
//   split evenly across warps.
// Per-vertex counts (t[a],t[b],t[c] += 1 per triangle): t[a] per item, t[b]
//   per segment, t[c] per hit into SMEM counters for the top ranks (global
//   atomics below them).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "graph.cuh"
#include "prim.cuh"

namespace tcb {
namespace {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kJoinThreads = 256;
constexpr int kJoinWarps = kJoinThreads / 32;
constexpr uint32_t kWarpTable = 128;         // warp-bin hash slots (d+ <= 48)
constexpr uint32_t kTopCounters = 1u << 13;  // per-vertex SMEM counters (16-bit halves: 16 KB)
constexpr uint32_t kCtaSmemSlots = 1024;     // cold-member hash table in SMEM (4 KB)

__host__ __device__ __forceinline__ uint32_t table_size_for(uint32_t members) {
  uint32_t t = 32;  // load factor <= 1/2
  while (t < 2 * members) t <<= 1;
  return t;
}

__host__ __device__ __forceinline__ uint32_t log2_pow2(uint32_t ts) {
  uint32_t l = 0;
  while ((1u << l) < ts) ++l;
  return l;
}

// ---- multi-GPU partition -------------------------------------------------------

// Prefix of per-edge cost (wedge work + a per-item overhead) over the oriented
// edges, then P-1 binary searches.  Contiguous edge ranges = contiguous source
// ranges of the degree-ordered DAG: the north-star "degree-weighted ranges".
struct EdgeCost {
  const uint32_t* off;
  const uint32_t* col;
  const uint32_t* src;
  __device__ __forceinline__ uint64_t operator()(uint64_t e) const {
    const uint32_t v = col[e];
    const uint32_t dv = off[v + 1] - off[v];
    const uint32_t end = off[src[e] + 1];
    return (dv > 0 && e + 1 < end) ? (uint64_t)(end - (uint32_t)(e + 1)) + 8 : 0ull;
  }
};

__global__ void k_part_bounds(const uint64_t* __restrict__ prefix, uint64_t E, uint64_t total, uint32_t parts,
                              uint64_t* __restrict__ bounds) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  if (p == 0) {
    bounds[0] = 0;
    return;
  }
  if (p == parts) {
    bounds[parts] = E;
    return;
  }
  const uint64_t target = (uint64_t)((double)total * p / parts);
  uint64_t lo = 0, hi = E;  // first e with prefix[e] >= target
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (prefix[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[p] = lo;
}

// ---- membership structures -------------------------------------------------

// Multiplicative (Fibonacci) hashing: scatters runs of consecutive ranks, so
// linear-probe clusters stay short (identity hashing of dense rank runs gave
// long, divergent probe chains: profiles/README.md, join v1).
__device__ __forceinline__ uint32_t hslot(uint32_t x, uint32_t shift) { return (x * 0x9E3779B1u) >> shift; }

__device__ __forceinline__ bool hash_find(const uint32_t* tab, uint32_t mask, uint32_t shift, uint32_t x) {
  uint32_t s = hslot(x, shift) & mask;
  while (true) {
    const uint32_t k = tab[s];
    if (k == x) return true;
    if (k == kEmpty) return false;
    s = (s + 1) & mask;
  }
}

__device__ __forceinline__ void hash_insert(uint32_t* tab, uint32_t mask, uint32_t shift, uint32_t x) {
  uint32_t s = hslot(x, shift) & mask;
  while (atomicCAS(&tab[s], kEmpty, x) != kEmpty) s = (s + 1) & mask;
}

// Per-vertex hits t[x]: SMEM counters for the top ranks [rc, n) (flushed once
// per CTA), global atomics below them.
__device__ uint32_t g_pv_dbg = 0;

// kHalf: counters are 16-bit halves of 32-bit words (twice the window per
// byte, which keeps 4 CTAs/SM resident).  The increments stay fire-and-forget
// (RED, no return value); the CTA kernel flushes before any half could wrap
// (a segment adds at most its item count to one counter).
template <bool kHalf>
struct PvSink {
  uint32_t* top;
  uint32_t rc;
  unsigned long long* t_rank;
  uint32_t dbg;  // diagnostics (TCB_PV_DBG): bit0 skip t[x], bit1 skip global atomics
  __device__ __forceinline__ void hit(uint32_t x) const {
    if (dbg & 1) return;
    if (x >= rc) {
      const uint32_t i = x - rc;
      if (kHalf) atomicAdd(&top[i >> 1], 1u << ((i & 1u) << 4));
      else atomicAdd(&top[i], 1u);
    } else if (!(dbg & 2)) {
      atomicAdd(&t_rank[x], 1ull);
    }
  }
};

// Add the SMEM counters [rc, rc+ncnt) into t_rank and zero them.
template <bool kHalf>
__device__ __forceinline__ void flush_top(uint32_t* top, uint32_t ncnt, uint32_t rc, unsigned long long* t_rank) {
  if (kHalf) {
    for (uint32_t j = threadIdx.x; j < ncnt / 2; j += blockDim.x) {
      const uint32_t w = top[j];
      if (!w) continue;
      top[j] = 0;
      if (w & 0xffffu) atomicAdd(&t_rank[rc + 2 * j], (unsigned long long)(w & 0xffffu));
      if (w >> 16) atomicAdd(&t_rank[rc + 2 * j + 1], (unsigned long long)(w >> 16));
    }
  } else {
    for (uint32_t j = threadIdx.x; j < ncnt; j += blockDim.x) {
      const uint32_t w = top[j];
      if (!w) continue;
      top[j] = 0;
      atomicAdd(&t_rank[rc + j], (unsigned long long)w);
    }
  }
}

// ---- chunk decoders ----------------------------------------------------------

// 8 hot ids (16-bit offsets from h0) per 16-byte chunk: bitmap probes.
__device__ __forceinline__ uint32_t hot_u16(const uint4& q, int i) {
  const uint32_t w = (i < 2) ? q.x : (i < 4) ? q.y : (i < 6) ? q.z : q.w;
  return (i & 1) ? (w >> 16) : (w & 0xffffu);
}

template <bool kPerVertex, typename Sink>
__device__ __forceinline__ uint32_t probe_hot(const uint4& q, uint32_t c, uint32_t b, uint32_t e,
                                              const uint32_t* bm, uint32_t h0, const Sink& sink) {
  const uint32_t p0 = c << 3;
  const uint32_t lo = b > p0 ? b - p0 : 0u;
  const uint32_t hi = e - p0 < 8u ? e - p0 : 8u;
  const uint32_t valid = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
  uint32_t hits = 0;
  uint32_t y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    y[i] = hot_u16(q, i);
    hits |= ((bm[y[i] >> 5] >> (y[i] & 31)) & 1u) << i;
  }
  hits &= valid;
  if (kPerVertex && hits) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (hits & (1u << i)) sink.hit(y[i] + h0);
  }
  return __popc(hits);
}

// 4 cold ids (32-bit) per chunk: hash probes.
template <bool kPerVertex, typename Sink>
__device__ __forceinline__ uint32_t probe_cold(const uint4& q, uint32_t c, uint32_t b, uint32_t e,
                                               const uint32_t* tab, uint32_t mask, uint32_t shift,
                                               const Sink& sink) {
  const uint32_t xs[4] = {q.x, q.y, q.z, q.w};
  const uint32_t p0 = c << 2;
  uint32_t h = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t p = p0 + t;
    if (p >= b && p < e && hash_find(tab, mask, shift, xs[t])) {
      ++h;
      if (kPerVertex) sink.hit(xs[t]);
    }
  }
  return h;
}

// ---- load balancing ----------------------------------------------------------

// Item each lane's chunk w+lane belongs to, for items whose chunk starts are
// given per lane (start/pre = exclusive/inclusive prefix, nch >= 1).
__device__ __forceinline__ uint32_t item_of(uint32_t w, uint32_t nch, uint32_t pre, uint32_t start) {
  const unsigned lane = lane_id();
  const uint32_t kb = __popc(__ballot_sync(0xffffffffu, nch && pre <= w));
  const uint32_t bit = (nch && start > w && start < w + 32) ? (1u << (start - w)) : 0u;
  const uint32_t smask = __reduce_or_sync(0xffffffffu, bit);
  const uint32_t k = kb + __popc(smask & ((2u << lane) - 1u));
  return k < 32 ? k : 31;
}

// Per-item hit counts of one chunk window: lanes holding chunks of the same
// item are a contiguous run (item index is non-decreasing in the lane), so a
// 5-step segmented suffix sum leaves each run's total in its head lane -- one
// SMEM atomic per item run instead of one per lane.
__device__ __forceinline__ void add_item_counts(uint32_t* cnt, const uint16_t* sidx, bool valid, uint32_t k,
                                                uint32_t x) {
  const unsigned lane = lane_id();
  const uint32_t key = valid ? k : 0xffffffffu;
  uint32_t v = valid ? x : 0u;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_down_sync(0xffffffffu, v, d);
    const uint32_t k2 = __shfl_down_sync(0xffffffffu, key, d);
    if (lane + d < 32 && k2 == key) v += t;
  }
  const uint32_t kp = __shfl_up_sync(0xffffffffu, key, 1);
  if (valid && v && (lane == 0 || kp != key)) atomicAdd(&cnt[sidx ? sidx[k] : k], v);
}

// A warp walks chunk range [fb, fe) of a segment list staged in SMEM (item i:
// chunk start pre[i] (pre[ni] = total), element range [sb[i], se[i]), original
// index sidx[i]), two chunks per lane in flight.  fn(q, c, b, e) -> hits.
template <int kIdsPerChunk, typename T, typename ChunkFn>
__device__ __forceinline__ uint32_t warp_walk(uint32_t fb, uint32_t fe, uint32_t ni, const uint32_t* pre,
                                              const uint32_t* sb, const uint32_t* se, const uint16_t* sidx,
                                              uint32_t* icnt, const T* base, ChunkFn fn) {
  constexpr uint32_t kShift = kIdsPerChunk == 8 ? 3 : 2;
  const unsigned lane = lane_id();
  const uint4* base4 = reinterpret_cast<const uint4*>(base);
  uint32_t h = 0;
  if (fb >= fe) return 0;
  uint32_t lo = 0, hi = ni;  // item containing chunk fb: last i with pre[i] <= fb
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (pre[mid] <= fb) lo = mid; else hi = mid;
  }
  uint32_t k0 = lo;
  for (uint32_t f = fb; f < fe; f += 64) {
    // window A = [f, f+32), window B = [f+32, f+64)
    uint32_t j = k0 + 1 + lane;
    uint32_t st = pre[min(j, ni)];
    uint32_t bit = (j < ni && st < f + 32) ? (1u << (st - f)) : 0u;
    const uint32_t mA = __reduce_or_sync(0xffffffffu, bit);
    const uint32_t kA = k0 + __popc(mA & ((2u << lane) - 1u));
    const uint32_t k1 = k0 + __popc(__ballot_sync(0xffffffffu, j < ni && st <= f + 32));
    j = k1 + 1 + lane;
    st = pre[min(j, ni)];
    bit = (j < ni && st < f + 64) ? (1u << (st - f - 32)) : 0u;
    const uint32_t mB = __reduce_or_sync(0xffffffffu, bit);
    const uint32_t kB = k1 + __popc(mB & ((2u << lane) - 1u));
    k0 = k1 + __popc(__ballot_sync(0xffffffffu, j < ni && st <= f + 64));
    const uint32_t fA = f + lane, fB = f + 32 + lane;
    const bool vA = fA < fe, vB = fB < fe;
    const uint32_t kAc = vA ? kA : 0, kBc = vB ? kB : 0;
    const uint32_t bA = sb[kAc], eA = se[kAc], cA = (bA >> kShift) + (fA - pre[kAc]);
    const uint32_t bB = sb[kBc], eB = se[kBc], cB = (bB >> kShift) + (fB - pre[kBc]);
    uint4 qA = make_uint4(0, 0, 0, 0), qB = make_uint4(0, 0, 0, 0);
    if (vA) qA = __ldg(base4 + cA);
    if (vB) qB = __ldg(base4 + cB);
    if (vA) {
      const uint32_t x = fn(qA, cA, bA, eA);
      h += x;
      if (icnt && x) atomicAdd(&icnt[sidx[kAc]], x);
    }
    if (vB) {
      const uint32_t x = fn(qB, cB, bB, eB);
      h += x;
      if (icnt && x) atomicAdd(&icnt[sidx[kBc]], x);
    }
  }
  return h;
}

// ---- warp bin ------------------------------------------------------------------

// Advance + join for items [i0, i1) of one small pivot (u32 suffix ranges
// {b,e} in items[i].x/.y), executed by one warp against its private hash.
template <bool kPerVertex, typename Sink>
__device__ __forceinline__ uint32_t warp_join_small(const uint4* __restrict__ items, const uint32_t* __restrict__ item_e,
                                                    uint32_t i0, uint32_t i1, const uint32_t* __restrict__ col,
                                                    const uint32_t* __restrict__ src, const uint32_t* tab,
                                                    uint32_t mask, uint32_t shift, const Sink& sink,
                                                    uint32_t* item_cnt) {
  const unsigned lane = lane_id();
  const uint4* col4 = reinterpret_cast<const uint4*>(col);
  uint32_t hits = 0;
  for (uint32_t ib = i0; ib < i1; ib += 32) {
    const uint32_t my = ib + lane;
    uint32_t b = 0, e = 0, nch = 0;
    if (my < i1) {
      const uint2 it = __ldcs(reinterpret_cast<const uint2*>(items + my));
      b = it.x;
      e = it.y;
      nch = ((e + 3) >> 2) - (b >> 2);
    }
    const uint32_t pre = warp_inclusive_scan(nch);
    const uint32_t start = pre - nch;
    const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
    if (kPerVertex) {
      item_cnt[lane] = 0;
      __syncwarp();
    }
    for (uint32_t base = 0; base < total; base += 32) {
      const uint32_t k = item_of(base, nch, pre, start);
      const uint32_t bk = __shfl_sync(0xffffffffu, b, k), ek = __shfl_sync(0xffffffffu, e, k);
      const uint32_t sk = __shfl_sync(0xffffffffu, start, k);
      const uint32_t f = base + lane;
      if (f < total) {
        const uint32_t c = (bk >> 2) + (f - sk);
        const uint32_t x = probe_cold<kPerVertex>(__ldg(col4 + c), c, bk, ek, tab, mask, shift, sink);
        hits += x;
        if (kPerVertex && x) atomicAdd(&item_cnt[k], x);
      }
    }
    if (kPerVertex) {
      __syncwarp();
      const uint32_t c = item_cnt[lane];
      if (c) atomicAdd(&sink.t_rank[src[item_e[my]]], (unsigned long long)c);
      __syncwarp();
    }
  }
  return hits;
}

// Warp bin: each warp takes whole segments of small pivots (d+ <= 48) with a
// warp-private 128-slot hash table; the CTA shares the per-vertex top-rank
// counters (dynamic SMEM, pv only).
template <bool kPerVertex>
__global__ void __launch_bounds__(kJoinThreads) k_join_warp(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
    const uint4* __restrict__ items, const uint32_t* __restrict__ item_e, const uint4* __restrict__ segs,
    uint32_t nsegs, uint32_t rc, uint32_t ncnt, unsigned long long* __restrict__ t_rank,
    unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t top_cnt[];
  __shared__ uint32_t s_tab[kJoinWarps][kWarpTable];
  __shared__ uint32_t s_item[kJoinWarps][32];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* tab = s_tab[warp];
  for (uint32_t s = lane; s < kWarpTable; s += 32) tab[s] = kEmpty;
  if (kPerVertex) {
    for (uint32_t i = threadIdx.x; i < ncnt; i += kJoinThreads) top_cnt[i] = 0;
    __syncthreads();
  }
  __syncwarp();
  const uint32_t mask = kWarpTable - 1, shift = 32 - log2_pow2(kWarpTable);
  const PvSink<false> sink{top_cnt, rc, t_rank, g_pv_dbg};
  unsigned long long acc = 0;
  const uint32_t gw = blockIdx.x * kJoinWarps + warp, nw = gridDim.x * kJoinWarps;
  for (uint32_t si = gw; si < nsegs; si += nw) {
    const uint4 sg = segs[si];
    const uint32_t v = sg.x;
    const uint32_t nb = off[v], dv = off[v + 1] - nb;
    for (uint32_t j = lane; j < dv; j += 32) hash_insert(tab, mask, shift, col[nb + j]);
    __syncwarp();
    const uint32_t h =
        warp_join_small<kPerVertex>(items, item_e, sg.y, sg.z, col, src, tab, mask, shift, sink, s_item[warp]);
    __syncwarp();
    acc += h;
    if (kPerVertex) {
      const uint32_t hw = warp_sum(h);
      if (lane == 0 && hw) atomicAdd(&t_rank[v], (unsigned long long)hw);
    }
    for (uint32_t s = lane; s < kWarpTable; s += 32) tab[s] = kEmpty;
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
  if (kPerVertex) {
    __syncthreads();
    flush_top<false>(top_cnt, ncnt, rc, t_rank);
  }
}

// ---- CTA bin -------------------------------------------------------------------

// Per segment (pivot v, <= kCtaSegItems in-edge items):
//   1. stage N+(v): members >= h0 into the hot bitmap; the sorted prefix below
//      h0 (found in the same pass) into an open-addressing table -- in SMEM
//      when it fits, else in a per-CTA global slab.  Stage the items,
//      compacted into a hot list and a cold list with their chunk prefixes;
//   2. advance + join: each list's chunks are split evenly across the warps;
//      hot chunks = 8 16-bit ids probed in the bitmap, cold = 4 32-bit ids
//      probed in the hash;
//   3. clear the touched bitmap words / table slots, flush per-item counts.
// Segments come from a global queue, heaviest (top-rank pivots) first.
// Dynamic SMEM: [hot bitmap nbm words][cold hash kCtaSmemSlots][pv: ncnt counters].
template <bool kPerVertex>
__global__ void __launch_bounds__(kJoinThreads, 4) k_join_cta(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
    const uint16_t* __restrict__ colH, const uint4* __restrict__ items, const uint32_t* __restrict__ item_e,
    const uint4* __restrict__ segs, uint32_t nsegs, unsigned int* __restrict__ queue, uint32_t h0, uint32_t nbm,
    uint32_t stab_slots, uint32_t slab_cap, uint32_t* __restrict__ gslab, uint32_t rc, uint32_t ncnt,
    unsigned long long* __restrict__ t_rank, unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t dyn[];
  __shared__ uint32_t s_hb[kCtaSegItems], s_he[kCtaSegItems], s_hpre[kCtaSegItems + 1];
  __shared__ uint32_t s_cb[kCtaSegItems], s_ce[kCtaSegItems], s_cpre[kCtaSegItems + 1];
  __shared__ uint16_t s_hidx[kCtaSegItems], s_cidx[kCtaSegItems];
  __shared__ uint32_t s_icnt[kPerVertex ? kCtaSegItems : 1];
  __shared__ uint32_t s_seg, s_hits, s_cold, s_nl;
  __shared__ unsigned long long s_ctot;
  uint32_t* bm = dyn;
  uint32_t* stab = dyn + nbm;
  uint32_t* top_cnt = dyn + nbm + kCtaSmemSlots;
  uint32_t* gtab = gslab + (uint64_t)blockIdx.x * slab_cap;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < nbm; i += kJoinThreads) bm[i] = 0;
  for (uint32_t i = threadIdx.x; i < kCtaSmemSlots; i += kJoinThreads) stab[i] = kEmpty;
  for (uint32_t i = threadIdx.x; i < slab_cap; i += kJoinThreads) gtab[i] = kEmpty;
  if (kPerVertex) {
    for (uint32_t i = threadIdx.x; i < ncnt / 2; i += kJoinThreads) top_cnt[i] = 0;
    for (uint32_t i = threadIdx.x; i < kCtaSegItems; i += kJoinThreads) s_icnt[i] = 0;
  }
  const PvSink<true> sink{top_cnt, rc, t_rank, g_pv_dbg};
  unsigned long long acc = 0;
  uint32_t since_flush = 0;  // items since the last counter flush (bounds every 16-bit half)
  while (true) {
    if (threadIdx.x == 0) {
      s_seg = atomicAdd(queue, 1u);
      s_hits = 0;
      s_cold = 0;
    }
    __syncthreads();
    const uint32_t q = s_seg;
    if (q >= nsegs) break;
    const uint4 sg = segs[nsegs - 1 - q];  // heaviest (top ranks) first
    const uint32_t v = sg.x, i0 = sg.y, ni = sg.z - sg.y;
    if (kPerVertex) {
      // one segment adds at most ni to any counter: flush before a half could wrap
      if (since_flush + ni > 0xffffu) {
        flush_top<true>(top_cnt, ncnt, rc, t_rank);
        since_flush = 0;
        __syncthreads();
      }
      since_flush += ni;
    }
    const uint32_t nb = off[v], dv = off[v + 1] - nb;
    // (1a) hot members -> bitmap; s_cold = #members below h0 (sorted prefix)
    for (uint32_t j = threadIdx.x; j < dv; j += kJoinThreads) {
      const uint32_t x = col[nb + j];
      if (x >= h0) {
        atomicOr(&bm[(x - h0) >> 5], 1u << ((x - h0) & 31));
        if (j == 0 || col[nb + j - 1] < h0) s_cold = j;
      } else if (j + 1 == dv) {
        s_cold = dv;
      }
    }
    // (1b) stage items, compacted into hot / cold lists with chunk prefixes
    uint4 it[2];
    uint32_t nh[2], nc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t i = threadIdx.x * 2 + r;
      nh[r] = nc[r] = 0;
      if (i < ni) {
        it[r] = __ldcs(items + i0 + i);
        nh[r] = it[r].y > it[r].x ? ((it[r].y + 7) >> 3) - (it[r].x >> 3) : 0u;
        nc[r] = it[r].w > it[r].z ? ((it[r].w + 3) >> 2) - (it[r].z >> 2) : 0u;
      }
    }
    // list positions: hot count in the low 16 bits, cold count in the high 16
    const uint32_t lp = block_exclusive_scan(
        (uint32_t)((nh[0] > 0) + (nh[1] > 0)) | ((uint32_t)((nc[0] > 0) + (nc[1] > 0)) << 16), &s_nl);
    // chunk prefixes: hot in the low 32 bits, cold in the high 32
    const unsigned long long cp = block_exclusive_scan(
        (unsigned long long)(nh[0] + nh[1]) | ((unsigned long long)(nc[0] + nc[1]) << 32), &s_ctot);
    {
      uint32_t ph = lp & 0xffffu, pc = lp >> 16;
      uint32_t ch = (uint32_t)cp, cc = (uint32_t)(cp >> 32);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t i = threadIdx.x * 2 + r;
        if (nh[r]) {
          s_hb[ph] = it[r].x;
          s_he[ph] = it[r].y;
          s_hpre[ph] = ch;
          s_hidx[ph] = (uint16_t)i;
          ++ph;
          ch += nh[r];
        }
        if (nc[r]) {
          s_cb[pc] = it[r].z;
          s_ce[pc] = it[r].w;
          s_cpre[pc] = cc;
          s_cidx[pc] = (uint16_t)i;
          ++pc;
          cc += nc[r];
        }
      }
    }
    __syncthreads();
    const uint32_t nhot = s_nl & 0xffffu, ncold = s_nl >> 16;
    const uint32_t cold = s_cold;
    const uint32_t tchunks_h = (uint32_t)s_ctot, tchunks_c = (uint32_t)(s_ctot >> 32);
    if (threadIdx.x == 0) {
      s_hpre[nhot] = tchunks_h;
      s_cpre[ncold] = tchunks_c;
    }
    uint32_t ts = 0, tmask = 0, tshift = 31;  // no cold members: probe the always-empty stab[0]
    uint32_t* tab = stab;
    if (cold) {
      ts = table_size_for(cold);
      tmask = ts - 1;
      tshift = 32 - log2_pow2(ts);
      tab = ts <= stab_slots ? stab : gtab;
      for (uint32_t j = threadIdx.x; j < cold; j += kJoinThreads) hash_insert(tab, tmask, tshift, col[nb + j]);
      if (tab == gtab) __threadfence_block();
    }
    __syncthreads();
    // (2) advance + join: hot chunks, then cold chunks, evenly split
    uint32_t h = 0;
    uint32_t* icnt = kPerVertex ? s_icnt : nullptr;
    if (!(g_pv_dbg & 4)) {
      const uint32_t fb = (uint32_t)(((uint64_t)tchunks_h * warp) / kJoinWarps);
      const uint32_t fe = (uint32_t)(((uint64_t)tchunks_h * (warp + 1)) / kJoinWarps);
      h += warp_walk<8>(fb, fe, nhot, s_hpre, s_hb, s_he, s_hidx, icnt, colH,
                        [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e) {
                          return probe_hot<kPerVertex>(qq, c, b, e, bm, h0, sink);
                        });
    }
    if (ncold && !(g_pv_dbg & 4)) {
      const uint32_t fb = (uint32_t)(((uint64_t)tchunks_c * warp) / kJoinWarps);
      const uint32_t fe = (uint32_t)(((uint64_t)tchunks_c * (warp + 1)) / kJoinWarps);
      h += warp_walk<4>(fb, fe, ncold, s_cpre, s_cb, s_ce, s_cidx, icnt, col,
                        [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e) {
                          return probe_cold<kPerVertex>(qq, c, b, e, tab, tmask, tshift, sink);
                        });
    }
    acc += h;
    if (kPerVertex) {
      const uint32_t hw = warp_sum(h);
      if (lane == 0 && hw) atomicAdd(&s_hits, hw);
    }
    __syncthreads();
    // (3) clear + per-vertex flush
    for (uint32_t j = cold + threadIdx.x; j < dv; j += kJoinThreads) bm[(col[nb + j] - h0) >> 5] = 0;
    for (uint32_t j = threadIdx.x; j < ts; j += kJoinThreads) tab[j] = kEmpty;
    if (kPerVertex) {
      for (uint32_t i = threadIdx.x; i < ni; i += kJoinThreads) {
        const uint32_t c = s_icnt[i];
        if (c) {
          atomicAdd(&t_rank[src[item_e[i0 + i]]], (unsigned long long)c);
          s_icnt[i] = 0;
        }
      }
      if (threadIdx.x == 0 && s_hits) atomicAdd(&t_rank[v], (unsigned long long)s_hits);
    }
    if (ts && tab == gtab) __threadfence_block();
    __syncthreads();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
  if (kPerVertex) {
    __syncthreads();
    flush_top<true>(top_cnt, ncnt, rc, t_rank);
  }
}

__global__ void k_gather_pv(const unsigned long long* __restrict__ t_rank, const uint32_t* __restrict__ rank_of,
                            uint32_t n, uint64_t* __restrict__ out) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    out[v] = t_rank[rank_of[v]];
}

uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = getenv(name);
  return v ? (uint32_t)strtoul(v, nullptr, 10) : dflt;
}

unsigned grid_gs(uint64_t n, int device) {
  const uint64_t cap = (uint64_t)num_sms(device) * 16;
  uint64_t g = ceil_div64(n, 256);
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

struct Events {
  cudaEvent_t e[4];
  Events() {
    for (auto& x : e) TC_CUDA(cudaEventCreate(&x));
  }
  ~Events() {
    for (auto& x : e) cudaEventDestroy(x);
  }
  float ms(int a, int b) {
    float t = 0;
    cudaEventElapsedTime(&t, e[a], e[b]);
    return t;
  }
};

}  // namespace

const std::vector<uint64_t>& partition_bounds(tc_graph& g, uint32_t parts) {
  if (g.cached_parts != parts) {
    cudaStream_t s = g.stream;
    const uint64_t E = g.E;
    g.part_bounds.assign((size_t)parts + 1, 0);
    g.part_bounds[parts] = E;
    if (E && parts > 1) {
      DBuf<uint64_t> prefix(E, s), tot(1, s), bnd((uint64_t)parts + 1, s);
      scan_exclusive<uint64_t>(EdgeCost{g.off.get(), g.col.get(), g.src.get()}, prefix.get(), E, tot.get(), s);
      const uint64_t total_cost = read_scalar(tot.get(), s);
      k_part_bounds<<<ceil_div(parts + 1, 128), 128, 0, s>>>(prefix.get(), E, total_cost, parts, bnd.get());
      TC_LAUNCH();
      TC_CUDA(cudaMemcpyAsync(g.part_bounds.data(), bnd.get(), (parts + 1) * sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, s));
      TC_CUDA(cudaStreamSynchronize(s));
    }
    g.cached_parts = parts;
  }
  return g.part_bounds;
}

void count_triangles(tc_graph& g, const tc_count_opts& opts, uint64_t* d_total, uint64_t* d_pv,
                     tc_count_stats* stats) {
  cudaStream_t s = g.stream;
  const int dev = g.device;
  const uint32_t n = g.n;
  const uint64_t E = g.E;
  const uint32_t parts = opts.part_count ? opts.part_count : 1;
  const uint32_t part = opts.part_count ? opts.part_index : 0;
  const bool pv = d_pv != nullptr;
  Events ev;
  TC_CUDA(cudaEventRecord(ev.e[0], s));
  uint64_t kl = 0;  // kernels launched by this call

  DBuf<unsigned long long> acc(1, s);
  TC_CUDA(cudaMemsetAsync(acc.get(), 0, sizeof(unsigned long long), s));
  DBuf<unsigned long long> t_rank;
  if (pv) {
    t_rank.alloc(n ? n : 1, s);
    TC_CUDA(cudaMemsetAsync(t_rank.get(), 0, sizeof(unsigned long long) * (n ? n : 1), s));
  }

  // ---- work segments: the whole frontier, or this part's degree-weighted
  //      oriented-edge range (multi-GPU) ----
  const uint4* wsegs = g.fr_wsegs.get();
  const uint4* csegs = g.fr_csegs.get();
  uint64_t NSW = g.fr_nwsegs, NSC = g.fr_ncsegs;
  DBuf<uint4> pw, pc;
  if (parts > 1 && E) {
    if (g.cached_parts != parts) kl += 4;
    const std::vector<uint64_t>& b = partition_bounds(g, parts);
    part_segments(g, b[part], b[part + 1], pw, NSW, pc, NSC);
    kl += 6;
    wsegs = pw.get();
    csegs = pc.get();
  }
  TC_CUDA(cudaEventRecord(ev.e[1], s));

  // ---- advance + join ----
  const int sms = num_sms(dev);
  uint64_t launches = 0;
  // per-vertex SMEM counters for the top ranks [rc, n); TCB_TOP_COUNTERS /
  // TCB_SMEM_SLOTS shrink them so tests drive every path on small graphs
  const uint32_t top_cnt = env_u32("TCB_TOP_COUNTERS", kTopCounters);
  const uint32_t smem_slots = std::min(env_u32("TCB_SMEM_SLOTS", kCtaSmemSlots), kCtaSmemSlots);
  const uint32_t ncnt = pv ? ((n < top_cnt ? n : top_cnt) & ~1u) : 0;
  const uint32_t rc = pv ? n - ncnt : 0xffffffffu;
  {
    const uint32_t dbg = env_u32("TCB_PV_DBG", 0);
    TC_CUDA(cudaMemcpyToSymbolAsync(g_pv_dbg, &dbg, sizeof(dbg), 0, cudaMemcpyHostToDevice, s));
  }
  if (NSW) {
    // warp bin: plain 32-bit counters over half the window
    const uint32_t ncnt_w = ncnt / 2, rc_w = pv ? n - ncnt_w : 0xffffffffu;
    const size_t smem = (size_t)ncnt_w * sizeof(uint32_t);
    auto kern = pv ? k_join_warp<true> : k_join_warp<false>;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kJoinThreads, smem));
    const unsigned grid =
        (unsigned)std::min<uint64_t>(ceil_div64(NSW, kJoinWarps), (uint64_t)sms * std::max(occ, 1));
    kern<<<grid, kJoinThreads, smem, s>>>(g.off.get(), g.col.get(), g.src.get(), g.fr_items.get(), g.fr_e.get(),
                                         wsegs, (uint32_t)NSW, rc_w, ncnt_w, t_rank.get(), acc.get());
    TC_LAUNCH();
    ++launches;
  }
  if (NSC) {
    DBuf<unsigned int> queue(1, s);
    TC_CUDA(cudaMemsetAsync(queue.get(), 0, sizeof(unsigned int), s));
    const uint32_t nbm = (n - g.h0 + 31) / 32;
    // cold members spill to a per-CTA global slab only when a pivot has more
    // than smem_slots/2 members below h0
    const uint32_t cap = table_size_for(g.max_dplus);
    const uint32_t slab_cap = (cap > smem_slots) ? cap : 0;
    const size_t dsm = ((size_t)nbm + kCtaSmemSlots + ncnt / 2) * sizeof(uint32_t);
    auto kern = pv ? k_join_cta<true> : k_join_cta<false>;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    int occ = 0;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kJoinThreads, dsm));
    if (occ < 1) occ = 1;
    const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)sms * occ, NSC);
    DBuf<uint32_t> slab((uint64_t)grid * slab_cap + 1, s);
    kern<<<grid, kJoinThreads, dsm, s>>>(g.off.get(), g.col.get(), g.src.get(), g.colH.get(), g.fr_items.get(),
                                        g.fr_e.get(), csegs, (uint32_t)NSC, queue.get(), g.h0, nbm, smem_slots,
                                        slab_cap, slab.get(), rc, ncnt, t_rank.get(), acc.get());
    TC_LAUNCH();
    ++launches;
  }
  TC_CUDA(cudaEventRecord(ev.e[2], s));

  // ---- outputs ----
  TC_CUDA(cudaMemcpyAsync(d_total, acc.get(), sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  if (pv && n) {
    k_gather_pv<<<grid_gs(n, dev), 256, 0, s>>>(t_rank.get(), g.rank_of.get(), n, d_pv);
    TC_LAUNCH();
    ++kl;
  }
  TC_CUDA(cudaEventRecord(ev.e[3], s));
  if (stats) {
    TC_CUDA(cudaEventSynchronize(ev.e[3]));
    stats->frontier_ms = ev.ms(0, 1);
    stats->join_ms = ev.ms(1, 2);
    stats->reduce_ms = ev.ms(2, 3);
    stats->total_ms = ev.ms(0, 3);
    stats->items = g.fr_nitems;
    stats->wedges = g.fr_J;
    stats->segments = NSW + NSC;
    stats->join_launches = launches;
    stats->dag_W = (double)g.fr_W;
    stats->pivots = g.fr_pivots;
    stats->kernel_launches = kl + launches;
    stats->alg_bytes = 4.0 * (double)g.fr_W + 12.0 * (double)E + 8.0 * ((double)n + 1) + (pv ? 8.0 * n : 0.0);
    // bytes the implemented join must stream: hot ids 2 B, cold ids 4 B,
    // items 16 B, pivot lists 4 B per member (whole graph; a part does ~1/P)
    stats->probe_bytes = 2.0 * (double)g.fr_hot + 4.0 * (double)(g.fr_J - g.fr_hot) +
                         16.0 * (double)g.fr_nitems + 4.0 * (double)E;
  }
}

}  // namespace tcb
