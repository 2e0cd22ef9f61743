// count.cu -- the hot path: level-1 frontier, degree-binned advance and fused
// SMEM-hash join, warp-shuffle/atomic reduction (north_star (2)-(4)).
//
// Reference path replaced (matcher.cpp): count_triangles :301-303 -> match
// :249-299 -> filter_candidates :46-87 -> expand_level (level 1) :136-198 ->
// count_final_level :204-245, whose inner loop visits every x in N(u) for each
// row (u,w) and tests has_edge(w,x) by binary search (graph.cpp:23-31).
//
// Formulation on the (deg,id)-ordered DAG in rank space:
//   every triangle a<b<c (ranks) has oriented edges a->b, a->c, b->c and is
//   found exactly once with PIVOT v=b: for each in-edge u->v (u=a) the advance
//   expands the wedge candidates x = the suffix of N+(u) after v (x=c is in
//   it), and the join keeps x iff x in N+(v), probed in an SMEM hash of N+(v).
//   Candidate wedges J = sum_u C(d+(u),2) (4.2e10 at RMAT s24) instead of the
//   reference's sum_rows deg(u), and 4.4x fewer than the wedge-stream W.
//
// Frontier ("items"): one (b,e) pair per useful in-edge u->v, grouped by pivot
//   v: [b,e) = the suffix of N+(u) after v in col[].  Items whose suffix is
//   empty and pivots with d+(v)=0 never enter the frontier (they cannot close
//   a triangle) -- the GPU analogue of the 2-core filter + look-ahead pruning.
// Bins (by d+(v) = hash size):
//   warp bin  d+(v) <= kWarpMaxDeg: one warp per segment, warp-private table
//   CTA bin   larger: the CTA builds one table, its warps share it
// Within a warp the items are load-balanced at 16-byte chunk granularity:
//   lanes take consecutive int4 chunks of the concatenated suffixes (item found
//   by a ballot/redux start mask), so loads are coalesced, vectorised int4.
// Per-vertex counts (t[a],t[b],t[c] += 1 per triangle) are aggregated in SMEM:
//   t[c] per hash slot, t[a] per item, t[b] per segment; <= |E|+items+segments
//   global atomics instead of 3T.
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
constexpr uint32_t kWarpMaxDeg = 48;   // warp bin: d+(v) <= 48 -> 128-slot table
constexpr uint32_t kWarpTable = 128;
constexpr uint32_t kWarpSegItems = 64;  // items per warp segment
constexpr uint32_t kCtaSegItems = 512;  // items per CTA segment
constexpr uint32_t kTopBitmapBits = 1u << 17;  // membership bitmap window (16 KB)
constexpr uint32_t kTopCounters = 1u << 13;    // per-vertex SMEM counter window (32 KB)
constexpr uint32_t kCtaSmemSlots = 1024;     // below-window hash table in SMEM (4 KB)

__host__ __device__ __forceinline__ uint32_t table_size_for(uint32_t dplus) {
  // load factor <= 1/2, at least 32 slots
  uint32_t t = 32;
  while (t < 2 * dplus) t <<= 1;
  return t;
}

// ---- frontier construction -------------------------------------------------

struct FrontierSums {
  unsigned long long W;      // sum_{u->v} d+(v)
  unsigned long long J;      // sum of useful suffix lengths
  unsigned long long items;  // useful items
};

// Wedge work of oriented edge e = u->v as a pivot in-edge: the suffix of
// N+(u) after v, when v can close triangles (d+(v) > 0).
__device__ __forceinline__ uint32_t edge_work(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                                              const uint32_t* __restrict__ src, uint64_t e, uint32_t& v,
                                              uint32_t& end) {
  v = col[e];
  const uint32_t dv = off[v + 1] - off[v];
  end = off[src[e] + 1];
  return (dv > 0 && e + 1 < end) ? end - (uint32_t)(e + 1) : 0u;
}

__global__ void k_item_count(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                             const uint32_t* __restrict__ src, uint64_t e0, uint64_t e1,
                             uint32_t* __restrict__ cnt, FrontierSums* __restrict__ sums) {
  unsigned long long W = 0, J = 0, I = 0;
  for (uint64_t e = e0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v, end;
    const uint32_t w = edge_work(off, col, src, e, v, end);
    W += off[v + 1] - off[v];
    if (w) {
      atomicAdd(&cnt[v], 1u);
      J += w;
      ++I;
    }
  }
  W = warp_sum(W);
  J = warp_sum(J);
  I = warp_sum(I);
  if (lane_id() == 0) {
    atomicAdd(&sums->W, W);
    atomicAdd(&sums->J, J);
    atomicAdd(&sums->items, I);
  }
}

__global__ void k_item_scatter(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                               const uint32_t* __restrict__ src, uint64_t e0, uint64_t e1,
                               const uint32_t* __restrict__ in_off, uint32_t* __restrict__ fill,
                               uint2* __restrict__ items) {
  for (uint64_t e = e0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1;
       e += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v, end;
    if (edge_work(off, col, src, e, v, end)) {
      const uint32_t p = in_off[v] + atomicAdd(&fill[v], 1u);
      items[p] = make_uint2((uint32_t)e + 1, end);
    }
  }
}

// Multi-GPU partition: prefix of per-edge cost (wedge work + a per-item
// overhead) over the oriented edges, then P-1 binary searches.  Contiguous
// edge ranges = contiguous source ranges of the degree-ordered DAG: the
// north-star "degree-weighted ranges".
struct EdgeCost {
  const uint32_t* off;
  const uint32_t* col;
  const uint32_t* src;
  __device__ __forceinline__ uint64_t operator()(uint64_t e) const {
    uint32_t v, end;
    const uint32_t w = edge_work(off, col, src, e, v, end);
    return w ? (uint64_t)w + 8 : 0ull;
  }
};

__global__ void k_part_bounds(const uint64_t* __restrict__ prefix, uint64_t E, uint64_t total, uint32_t parts,
                              uint64_t* __restrict__ bounds) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  if (p == 0) { bounds[0] = 0; return; }
  if (p == parts) { bounds[parts] = E; return; }
  const uint64_t target = (uint64_t)((double)total * p / parts);
  uint64_t lo = 0, hi = E;  // first e with prefix[e] >= target
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (prefix[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[p] = lo;
}

struct SegCount {
  const uint32_t* off;
  const uint32_t* cnt;
  uint32_t lo, hi, per;  // d+ range [lo, hi], items per segment
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const {
    const uint32_t dv = off[v + 1] - off[v];
    const uint32_t c = cnt[v];
    return (c && dv >= lo && dv <= hi) ? (c + per - 1) / per : 0u;
  }
};

__global__ void k_seg_fill(const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                           const uint32_t* __restrict__ in_off, uint32_t n, uint32_t lo, uint32_t hi,
                           uint32_t per, const uint32_t* __restrict__ seg_off, uint2* __restrict__ segs,
                           unsigned long long* __restrict__ npivots) {
  unsigned long long np = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t dv = off[v + 1] - off[v];
    const uint32_t c = cnt[v];
    if (!c || dv < lo || dv > hi) continue;
    const uint32_t ns = (c + per - 1) / per;
    const uint32_t s0 = seg_off[v];
    for (uint32_t k = 0; k < ns; ++k) segs[s0 + k] = make_uint2((uint32_t)v, in_off[v] + k * per);
    ++np;
  }
  np = warp_sum(np);
  if (lane_id() == 0 && np) atomicAdd(npivots, np);
}

// ---- the fused advance + join ---------------------------------------------

// Multiplicative (Fibonacci) hashing: scatters runs of consecutive ranks, so
// linear-probe clusters stay short (identity hashing of the dense top-rank
// runs produced long, divergent probe chains -- profiles/README.md).
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
  uint32_t s = hslot(x, shift);
  while (atomicCAS(&tab[s], kEmpty, x) != kEmpty) s = (s + 1) & mask;
}

__host__ __device__ __forceinline__ uint32_t log2_pow2(uint32_t ts) {
  uint32_t l = 0;
  while ((1u << l) < ts) ++l;
  return l;
}

// Membership test for N+(v) (the closing edge v->x of wedge (u; v, x)):
// a bitmap over the top-rank window [r0, n) -- where ~all wedge endpoints of
// a power-law DAG land, and where neighbouring lanes probe neighbouring
// words -- plus an open-addressing hash for the members below r0.
struct PivotSet {
  const uint32_t* bm;
  const uint32_t* tab;
  uint32_t r0, mask, shift;
  __device__ __forceinline__ bool contains(uint32_t x) const {
    if (x >= r0) {
      const uint32_t d = x - r0;
      return (bm[d >> 5] >> (d & 31)) & 1u;
    }
    return hash_find(tab, mask, shift, x);
  }
};

// Per-vertex hits t[x]: SMEM counters for the top window [rc, n) (flushed
// once per CTA), global atomics below it.
struct PvSink {
  uint32_t* top;
  uint32_t rc;
  unsigned long long* t_rank;
  __device__ __forceinline__ void hit(uint32_t x) const {
    if (x >= rc) atomicAdd(&top[x - rc], 1u);
    else atomicAdd(&t_rank[x], 1ull);
  }
};

// Locate, for chunk window [w, w+32), the item each lane's chunk w+lane
// belongs to (items hold >= 1 chunk; start/pre are the lane's item's
// exclusive/inclusive chunk prefix).
__device__ __forceinline__ uint32_t item_of(uint32_t w, uint32_t nch, uint32_t pre, uint32_t start) {
  const unsigned lane = lane_id();
  const uint32_t kb = __popc(__ballot_sync(0xffffffffu, nch && pre <= w));
  const uint32_t bit = (nch && start > w && start < w + 32) ? (1u << (start - w)) : 0u;
  const uint32_t smask = __reduce_or_sync(0xffffffffu, bit);
  const uint32_t k = kb + __popc(smask & ((2u << lane) - 1u));
  return k < 32 ? k : 31;
}

template <bool kPerVertex>
__device__ __forceinline__ uint32_t probe_chunk(const uint4 q, uint32_t c, uint32_t bk, uint32_t ek,
                                                const PivotSet& set, const PvSink& sink) {
  const uint32_t xs[4] = {q.x, q.y, q.z, q.w};
  const uint32_t p0 = c << 2;
  uint32_t h = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t p = p0 + t;
    if (p >= bk && p < ek && set.contains(xs[t])) {
      ++h;
      if (kPerVertex) sink.hit(xs[t]);
    }
  }
  return h;
}

// Advance + join for items [i0, i1) of one pivot, executed by one warp.
// Advance: the items' suffixes are cut into 16-byte chunks and load-balanced
// across lanes (two chunks per lane per step, both int4 loads in flight before
// any probe).  Join: every wedge endpoint x in [b,e) is tested against N+(v).
// Returns the lane's hit count; per-vertex: t[x] via the sink, t[u] via
// per-item SMEM counters (one global atomic per item).
template <bool kPerVertex>
__device__ __forceinline__ uint32_t warp_join_items(const uint2* __restrict__ items, uint32_t i0, uint32_t i1,
                                                    const uint32_t* __restrict__ col,
                                                    const uint32_t* __restrict__ src, const PivotSet& set,
                                                    const PvSink& sink, uint32_t* item_cnt) {
  const unsigned lane = lane_id();
  const uint4* col4 = reinterpret_cast<const uint4*>(col);
  uint32_t hits = 0;
  for (uint32_t ib = i0; ib < i1; ib += 32) {
    const uint32_t my = ib + lane;
    uint32_t b = 0, e = 0, nch = 0;
    if (my < i1) {
      const uint2 it = items[my];
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
    for (uint32_t base = 0; base < total; base += 64) {
      const uint32_t k1 = item_of(base, nch, pre, start);
      const uint32_t k2 = item_of(base + 32, nch, pre, start);
      const uint32_t b1 = __shfl_sync(0xffffffffu, b, k1), e1 = __shfl_sync(0xffffffffu, e, k1);
      const uint32_t s1 = __shfl_sync(0xffffffffu, start, k1);
      const uint32_t b2 = __shfl_sync(0xffffffffu, b, k2), e2 = __shfl_sync(0xffffffffu, e, k2);
      const uint32_t s2 = __shfl_sync(0xffffffffu, start, k2);
      const uint32_t f1 = base + lane, f2 = base + 32 + lane;
      const uint32_t c1 = (b1 >> 2) + (f1 - s1), c2 = (b2 >> 2) + (f2 - s2);
      uint4 q1 = make_uint4(0, 0, 0, 0), q2 = make_uint4(0, 0, 0, 0);
      if (f1 < total) q1 = __ldg(col4 + c1);
      if (f2 < total) q2 = __ldg(col4 + c2);
      if (f1 < total) {
        const uint32_t h = probe_chunk<kPerVertex>(q1, c1, b1, e1, set, sink);
        hits += h;
        if (kPerVertex && h) atomicAdd(&item_cnt[k1], h);
      }
      if (f2 < total) {
        const uint32_t h = probe_chunk<kPerVertex>(q2, c2, b2, e2, set, sink);
        hits += h;
        if (kPerVertex && h) atomicAdd(&item_cnt[k2], h);
      }
    }
    if (kPerVertex) {
      __syncwarp();
      const uint32_t c = item_cnt[lane];
      if (c) atomicAdd(&sink.t_rank[src[b - 1]], (unsigned long long)c);
      __syncwarp();
    }
  }
  return hits;
}

// Warp bin: each warp takes whole segments of small pivots (d+ <= 48) with a
// warp-private 128-slot hash table; the CTA shares the per-vertex top-window
// counters (dynamic SMEM, pv only).
template <bool kPerVertex>
__global__ void __launch_bounds__(kJoinThreads) k_join_warp(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
    const uint2* __restrict__ items, const uint32_t* __restrict__ in_off, const uint2* __restrict__ segs,
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
  const PivotSet set{nullptr, tab, 0xffffffffu, mask, shift};
  const PvSink sink{top_cnt, rc, t_rank};
  unsigned long long acc = 0;
  const uint32_t gw = blockIdx.x * kJoinWarps + warp, nw = gridDim.x * kJoinWarps;
  for (uint32_t si = gw; si < nsegs; si += nw) {
    const uint2 sg = segs[si];
    const uint32_t v = sg.x, i0 = sg.y;
    const uint32_t i1 = min(i0 + kWarpSegItems, in_off[v + 1]);
    const uint32_t nb = off[v], dv = off[v + 1] - nb;
    for (uint32_t j = lane; j < dv; j += 32) hash_insert(tab, mask, shift, col[nb + j]);
    __syncwarp();
    const uint32_t h = warp_join_items<kPerVertex>(items, i0, i1, col, src, set, sink, s_item[warp]);
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
    for (uint32_t i = threadIdx.x; i < ncnt; i += kJoinThreads) {
      const uint32_t c = top_cnt[i];
      if (c) atomicAdd(&t_rank[rc + i], (unsigned long long)c);
    }
  }
}

// CTA bin.  Per segment (pivot v, <= kCtaSegItems in-edge items):
//   1. build N+(v): members >= r0 into the top-window bitmap; the sorted
//      prefix below r0 (hb members, found in the same pass) into an
//      open-addressing table -- in SMEM when it fits kCtaSmemSlots, else in a
//      per-CTA global slab;  stage the items (b, e, chunk prefix) in SMEM;
//   2. advance + join: the segment's 16-byte chunks are split evenly across
//      the warps (no warp waits on a long item of another), each warp walks
//      its chunk range window by window (item of each chunk from the SMEM
//      prefix via a ballot/redux start mask), two int4 loads in flight/lane;
//   3. clear the touched bitmap words / table slots, flush per-item counts.
// Segments come from a global queue, heaviest (top-rank pivots) first.
// Dynamic SMEM: [bitmap nbm words][hash kCtaSmemSlots][pv: top counters ncnt].
template <bool kPerVertex>
__global__ void __launch_bounds__(kJoinThreads, 2) k_join_cta(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
    const uint2* __restrict__ items, const uint32_t* __restrict__ in_off, const uint2* __restrict__ segs,
    uint32_t nsegs, unsigned int* __restrict__ queue, uint32_t r0, uint32_t nbm, uint32_t stab_slots,
    uint32_t slab_cap, uint32_t* __restrict__ gslab, uint32_t rc, uint32_t ncnt,
    unsigned long long* __restrict__ t_rank, unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t dyn[];
  __shared__ uint32_t s_b[kCtaSegItems], s_e[kCtaSegItems], s_pre[kCtaSegItems + 1];
  __shared__ uint32_t s_icnt[kPerVertex ? kCtaSegItems : 1];
  __shared__ uint32_t s_seg, s_hits, s_hb, s_tot;
  uint32_t* bm = dyn;
  uint32_t* stab = dyn + nbm;
  uint32_t* top_cnt = dyn + nbm + kCtaSmemSlots;
  uint32_t* gtab = gslab + (uint64_t)blockIdx.x * slab_cap;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint4* col4 = reinterpret_cast<const uint4*>(col);
  for (uint32_t i = threadIdx.x; i < nbm; i += kJoinThreads) bm[i] = 0;
  for (uint32_t i = threadIdx.x; i < kCtaSmemSlots; i += kJoinThreads) stab[i] = kEmpty;
  for (uint32_t i = threadIdx.x; i < slab_cap; i += kJoinThreads) gtab[i] = kEmpty;
  if (kPerVertex) {
    for (uint32_t i = threadIdx.x; i < ncnt; i += kJoinThreads) top_cnt[i] = 0;
    for (uint32_t i = threadIdx.x; i < kCtaSegItems; i += kJoinThreads) s_icnt[i] = 0;
  }
  const PvSink sink{top_cnt, rc, t_rank};
  unsigned long long acc = 0;
  while (true) {
    if (threadIdx.x == 0) {
      s_seg = atomicAdd(queue, 1u);
      s_hits = 0;
      s_hb = 0;
    }
    __syncthreads();
    const uint32_t q = s_seg;
    if (q >= nsegs) break;
    const uint2 sg = segs[nsegs - 1 - q];  // heaviest (top ranks) first
    const uint32_t v = sg.x, i0 = sg.y;
    const uint32_t ni = min(i0 + kCtaSegItems, in_off[v + 1]) - i0;
    const uint32_t nb = off[v], dv = off[v + 1] - nb;
    // (1) members >= r0 -> bitmap; hb = #members below r0 (sorted prefix)
    for (uint32_t j = threadIdx.x; j < dv; j += kJoinThreads) {
      const uint32_t x = col[nb + j];
      if (x >= r0) {
        atomicOr(&bm[(x - r0) >> 5], 1u << ((x - r0) & 31));
        if (j == 0 || col[nb + j - 1] < r0) s_hb = j;
      } else if (j + 1 == dv) {
        s_hb = dv;
      }
    }
    // stage the segment's items and their chunk prefix
    uint32_t nch[2], bb[2], ee[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t i = threadIdx.x * 2 + r;
      nch[r] = 0;
      if (i < ni) {
        const uint2 it = __ldcs(items + i0 + i);
        bb[r] = it.x;
        ee[r] = it.y;
        nch[r] = ((it.y + 3) >> 2) - (it.x >> 2);
      }
    }
    const uint32_t ex = block_exclusive_scan(nch[0] + nch[1], &s_tot);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t i = threadIdx.x * 2 + r;
      if (i < ni) {
        s_b[i] = bb[r];
        s_e[i] = ee[r];
        s_pre[i] = ex + (r ? nch[0] : 0);
      }
    }
    __syncthreads();
    const uint32_t hb = s_hb, C = s_tot;
    if (threadIdx.x == 0) s_pre[ni] = C;
    uint32_t ts = 0, tmask = 0, tshift = 31;  // no members below r0: probe the always-empty stab[0]
    uint32_t* tab = stab;
    if (hb) {
      ts = table_size_for(hb);
      tmask = ts - 1;
      tshift = 32 - log2_pow2(ts);
      tab = ts <= stab_slots ? stab : gtab;
      for (uint32_t j = threadIdx.x; j < hb; j += kJoinThreads) hash_insert(tab, tmask, tshift, col[nb + j]);
      if (tab == gtab) __threadfence_block();
    }
    __syncthreads();
    const PivotSet set{bm, tab, r0, tmask, tshift};
    // (2) advance + join over this warp's even share of the chunks
    const uint32_t fb = (uint32_t)(((uint64_t)C * warp) / kJoinWarps);
    const uint32_t fe = (uint32_t)(((uint64_t)C * (warp + 1)) / kJoinWarps);
    uint32_t h = 0;
    if (fb < fe) {
      uint32_t lo = 0, hi = ni;  // item containing chunk fb: last i with s_pre[i] <= fb
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (s_pre[mid] <= fb) lo = mid; else hi = mid;
      }
      uint32_t k0 = lo;
      for (uint32_t f = fb; f < fe; f += 64) {
        // window A = [f, f+32), window B = [f+32, f+64)
        uint32_t st = s_pre[min(k0 + 1 + lane, ni)];
        uint32_t bit = (st < f + 32 && k0 + 1 + lane < ni) ? (1u << (st - f)) : 0u;
        const uint32_t mA = __reduce_or_sync(0xffffffffu, bit);
        const uint32_t kA = k0 + __popc(mA & ((2u << lane) - 1u));
        const uint32_t k1 = k0 + __popc(__ballot_sync(0xffffffffu, k0 + 1 + lane < ni && st <= f + 32));
        st = s_pre[min(k1 + 1 + lane, ni)];
        bit = (st < f + 64 && k1 + 1 + lane < ni) ? (1u << (st - f - 32)) : 0u;
        const uint32_t mB = __reduce_or_sync(0xffffffffu, bit);
        const uint32_t kB = k1 + __popc(mB & ((2u << lane) - 1u));
        k0 = k1 + __popc(__ballot_sync(0xffffffffu, k1 + 1 + lane < ni && st <= f + 64));
        const uint32_t fA = f + lane, fB = f + 32 + lane;
        const bool vA = fA < fe, vB = fB < fe;
        const uint32_t kAc = vA ? kA : 0, kBc = vB ? kB : 0;
        const uint32_t bA = s_b[kAc], eA = s_e[kAc], cA = (bA >> 2) + (fA - s_pre[kAc]);
        const uint32_t bB = s_b[kBc], eB = s_e[kBc], cB = (bB >> 2) + (fB - s_pre[kBc]);
        uint4 qA = make_uint4(0, 0, 0, 0), qB = make_uint4(0, 0, 0, 0);
        if (vA) qA = __ldg(col4 + cA);
        if (vB) qB = __ldg(col4 + cB);
        if (vA) {
          const uint32_t x = probe_chunk<kPerVertex>(qA, cA, bA, eA, set, sink);
          h += x;
          if (kPerVertex && x) atomicAdd(&s_icnt[kAc], x);
        }
        if (vB) {
          const uint32_t x = probe_chunk<kPerVertex>(qB, cB, bB, eB, set, sink);
          h += x;
          if (kPerVertex && x) atomicAdd(&s_icnt[kBc], x);
        }
      }
    }
    acc += h;
    if (kPerVertex) {
      const uint32_t hw = warp_sum(h);
      if (lane == 0 && hw) atomicAdd(&s_hits, hw);
    }
    __syncthreads();
    // (3) clear + per-vertex flush
    for (uint32_t j = hb + threadIdx.x; j < dv; j += kJoinThreads) bm[(col[nb + j] - r0) >> 5] = 0;
    for (uint32_t j = threadIdx.x; j < ts; j += kJoinThreads) tab[j] = kEmpty;
    if (kPerVertex) {
      for (uint32_t i = threadIdx.x; i < ni; i += kJoinThreads) {
        const uint32_t c = s_icnt[i];
        if (c) {
          atomicAdd(&t_rank[src[s_b[i] - 1]], (unsigned long long)c);
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
    for (uint32_t i = threadIdx.x; i < ncnt; i += kJoinThreads) {
      const uint32_t c = top_cnt[i];
      if (c) atomicAdd(&t_rank[rc + i], (unsigned long long)c);
    }
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
  cudaEvent_t e[5];
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

  // ---- multi-GPU: this part's degree-weighted oriented-edge range ----
  uint64_t e0 = 0, e1 = E;
  if (parts > 1 && E) {
    if (g.cached_parts != parts) {
      DBuf<uint64_t> prefix(E, s), tot(1, s), bnd((uint64_t)parts + 1, s);
      kl += scan_exclusive<uint64_t>(EdgeCost{g.off.get(), g.col.get(), g.src.get()}, prefix.get(), E, tot.get(), s);
      const uint64_t total_cost = read_scalar(tot.get(), s);
      k_part_bounds<<<ceil_div(parts + 1, 128), 128, 0, s>>>(prefix.get(), E, total_cost, parts, bnd.get());
      TC_LAUNCH();
      ++kl;
      g.part_bounds.assign(parts + 1, 0);
      TC_CUDA(cudaMemcpyAsync(g.part_bounds.data(), bnd.get(), (parts + 1) * sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, s));
      TC_CUDA(cudaStreamSynchronize(s));
      g.cached_parts = parts;
    }
    e0 = g.part_bounds[part];
    e1 = g.part_bounds[part + 1];
  }

  // ---- level-1 frontier: useful in-edges grouped by pivot ----
  DBuf<uint32_t> cnt(n ? n : 1, s), in_off((uint64_t)n + 1, s);
  DBuf<FrontierSums> sums(1, s);
  TC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(uint32_t) * (n ? n : 1), s));
  TC_CUDA(cudaMemsetAsync(sums.get(), 0, sizeof(FrontierSums), s));
  if (e1 > e0) {
    k_item_count<<<grid_gs(e1 - e0, dev), 256, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), e0, e1, cnt.get(),
                                                       sums.get());
    TC_LAUNCH();
    ++kl;
  }
  kl += scan_exclusive<uint32_t>(LoadArray<uint32_t>{cnt.get()}, in_off.get(), n, in_off.get() + n, s);
  FrontierSums hs = read_scalar(sums.get(), s);
  const uint64_t NI = hs.items;
  DBuf<uint2> items(NI ? NI : 1, s);
  if (NI) {
    DBuf<uint32_t> fill(n, s);
    TC_CUDA(cudaMemsetAsync(fill.get(), 0, sizeof(uint32_t) * n, s));
    k_item_scatter<<<grid_gs(e1 - e0, dev), 256, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), e0, e1,
                                                         in_off.get(), fill.get(), items.get());
    TC_LAUNCH();
    ++kl;
  }
  // segments per bin
  DBuf<uint32_t> wseg_off(n ? n : 1, s), cseg_off(n ? n : 1, s), nseg(2, s);
  DBuf<unsigned long long> npiv(1, s);
  TC_CUDA(cudaMemsetAsync(npiv.get(), 0, sizeof(unsigned long long), s));
  uint32_t hn[2] = {0, 0};
  if (NI) {
    kl += scan_exclusive<uint32_t>(SegCount{g.off.get(), cnt.get(), 1, kWarpMaxDeg, kWarpSegItems}, wseg_off.get(),
                                   n, nseg.get(), s);
    kl += scan_exclusive<uint32_t>(SegCount{g.off.get(), cnt.get(), kWarpMaxDeg + 1, 0xffffffffu, kCtaSegItems},
                             cseg_off.get(), n, nseg.get() + 1, s);
    TC_CUDA(cudaMemcpyAsync(hn, nseg.get(), 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
  }
  uint32_t NSW = hn[0], NSC = hn[1];
  if (const char* dbg = getenv("TCB_DEBUG_BINS")) {  // diagnostics: 1 = warp bin only, 2 = CTA bin only
    const int m = atoi(dbg);
    if (!(m & 1)) NSW = 0;
    if (!(m & 2)) NSC = 0;
  }
  DBuf<uint2> wsegs(NSW ? NSW : 1, s), csegs(NSC ? NSC : 1, s);
  if (NSW) {
    k_seg_fill<<<grid_gs(n, dev), 256, 0, s>>>(g.off.get(), cnt.get(), in_off.get(), n, 1, kWarpMaxDeg,
                                               kWarpSegItems, wseg_off.get(), wsegs.get(), npiv.get());
    TC_LAUNCH();
    ++kl;
  }
  if (NSC) {
    k_seg_fill<<<grid_gs(n, dev), 256, 0, s>>>(g.off.get(), cnt.get(), in_off.get(), n, kWarpMaxDeg + 1,
                                               0xffffffffu, kCtaSegItems, cseg_off.get(), csegs.get(), npiv.get());
    TC_LAUNCH();
    ++kl;
  }
  TC_CUDA(cudaEventRecord(ev.e[1], s));

  // ---- advance + join ----
  const int sms = num_sms(dev);
  uint64_t launches = 0;
  // top-rank windows: membership bitmap [r0, n) and per-vertex counters [rc, n)
  // (TCB_TOP_BITMAP_BITS / TCB_TOP_COUNTERS / TCB_SMEM_MAX override the window
  // sizes so tests can drive every membership/counter path on small graphs)
  const uint32_t top_bits = env_u32("TCB_TOP_BITMAP_BITS", kTopBitmapBits) & ~31u;
  const uint32_t top_cnt = env_u32("TCB_TOP_COUNTERS", kTopCounters);
  const uint32_t smem_slots = env_u32("TCB_SMEM_SLOTS", kCtaSmemSlots);  // tests: force the global slab
  const uint32_t bm_bits = n < top_bits ? ((n + 31) & ~31u) : top_bits;
  const uint32_t r0 = n > bm_bits ? n - bm_bits : 0;
  const uint32_t nbm = bm_bits / 32;
  const uint32_t ncnt = pv ? (n < top_cnt ? n : top_cnt) : 0;
  const uint32_t rc = pv ? n - ncnt : 0xffffffffu;
  if (NSW) {
    const size_t smem = (size_t)ncnt * sizeof(uint32_t);
    auto kern = pv ? k_join_warp<true> : k_join_warp<false>;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kJoinThreads, smem));
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div64(NSW, kJoinWarps), (uint64_t)sms * std::max(occ, 1));
    kern<<<grid, kJoinThreads, smem, s>>>(g.off.get(), g.col.get(), g.src.get(), items.get(), in_off.get(),
                                         wsegs.get(), NSW, rc, ncnt, t_rank.get(), acc.get());
    TC_LAUNCH();
    ++launches;
  }
  if (NSC) {
    DBuf<unsigned int> queue(1, s);
    TC_CUDA(cudaMemsetAsync(queue.get(), 0, sizeof(unsigned int), s));
    // the below-window table spills to a per-CTA global slab only when a
    // pivot has more than kCtaSmemSlots/2 members below r0
    const uint32_t cap = table_size_for(g.max_dplus);
    const uint32_t slab_cap = (cap > smem_slots) ? cap : 0;
    const size_t dsm = ((size_t)nbm + kCtaSmemSlots + ncnt) * sizeof(uint32_t);
    auto kern = pv ? k_join_cta<true> : k_join_cta<false>;
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
    int occ = 0;
    TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kJoinThreads, dsm));
    if (occ < 1) occ = 1;
    const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)sms * occ, (uint64_t)NSC);
    DBuf<uint32_t> slab((uint64_t)grid * slab_cap + 1, s);
    kern<<<grid, kJoinThreads, dsm, s>>>(g.off.get(), g.col.get(), g.src.get(), items.get(), in_off.get(),
                                        csegs.get(), NSC, queue.get(), r0, nbm, std::min(smem_slots, kCtaSmemSlots),
                                        slab_cap, slab.get(), rc, ncnt,
                                        t_rank.get(), acc.get());
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
    stats->items = NI;
    stats->wedges = hs.J;
    stats->segments = (uint64_t)NSW + NSC;
    stats->join_launches = launches;
    stats->dag_W = (double)hs.W;
    stats->pivots = read_scalar(npiv.get(), s);
    stats->kernel_launches = kl + launches;
    stats->alg_bytes = 4.0 * (double)hs.W + 12.0 * (double)E + 8.0 * ((double)n + 1) + (pv ? 8.0 * n : 0.0);
    stats->probe_bytes = 4.0 * (double)hs.J + 8.0 * (double)NI + 4.0 * (double)E;
  }
}

}  // namespace tcb
