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
#include <cstdio>
#include <cstdlib>

#include "graph.cuh"
#include "prim.cuh"

namespace tcb {
namespace {

constexpr uint32_t kEmpty = 0xffffffffu;
constexpr int kJoinThreads = 256;
constexpr int kJoinWarps = kJoinThreads / 32;
#ifndef TCB_CTA_THREADS
#define TCB_CTA_THREADS 256
#endif
constexpr int kCtaThreads = TCB_CTA_THREADS;  // k_join_cta block (kCtaSegItems a multiple of it)
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr uint32_t kWarpTable = 128;         // warp-bin hash slots (d+ <= kWarpMaxDeg = 64)
constexpr uint32_t kTopCounters = 1u << 13;  // per-vertex SMEM counters (16-bit halves: 16 KB)
#ifndef TCB_CTA_SMEM_SLOTS
#define TCB_CTA_SMEM_SLOTS 1024
#endif
constexpr uint32_t kCtaSmemSlots = TCB_CTA_SMEM_SLOTS;  // cold-member hash table in SMEM (4 KB)
#ifndef TCB_HOT_WIN
#define TCB_HOT_WIN 2
#endif
#ifndef TCB_MIN_BLOCKS
#define TCB_MIN_BLOCKS 6  // CTA-bin residency target, both variants (A/B: profiles/README.md)
#endif
constexpr int kHotWin = TCB_HOT_WIN;              // hot chunk loads in flight per lane
constexpr int kCtaMinBlocks = TCB_MIN_BLOCKS;     // CTA-bin kernel residency target

__host__ __device__ __forceinline__ uint32_t table_size_for(uint32_t members) {
  // smallest power of two >= max(32, 2*members): load factor <= 1/2
  const uint32_t m2 = 2 * members;
  if (m2 <= 32) return 32;
#ifdef __CUDA_ARCH__
  return 1u << (32 - __clz(m2 - 1));
#else
  uint32_t t = 32;
  while (t < m2) t <<= 1;
  return t;
#endif
}

__host__ __device__ __forceinline__ uint32_t log2_pow2(uint32_t ts) {
  uint32_t l = 0;
  while ((1u << l) < ts) ++l;
  return l;
}

// ---- multi-GPU partition -------------------------------------------------------

// Work of pivot v (pivot-range parts): its candidate wedges J_v = sum over
// in-edges u->v of the suffix length |N+(u) after v|, plus a per-item and a
// per-segment overhead in candidate-probe units (item geometry / staging and
// the pivot row staged once per segment).  Accumulated edge-parallel (one
// coalesced pass over col; warp-aggregated per head), then an exclusive scan
// over the pivots and P-1 binary searches: part p = pivots [b[p], b[p+1]),
// contiguous rank ranges of ~equal work.  Every pivot's row is staged by one
// part only (no re-staging across parts), and the per-vertex row pass of a
// part reads only the items of its pivots (k_pv_rows PartRange).
#ifndef TCB_ITEM_COST
#define TCB_ITEM_COST 32
#endif
#ifndef TCB_SEG_COST
#define TCB_SEG_COST 4
#endif
#ifndef TCB_DENSE_COST
#define TCB_DENSE_COST 48  // one dense item (k_join_dense, ~50 warp instructions) in candidate-probe units
#endif
#ifndef TCB_COLD_COST
#define TCB_COLD_COST 6  // a cold (prefiltered hash) probe (8-part A/B on C4 and C5: profiles/)
#endif
#ifndef TCB_SMALL_COST
#define TCB_SMALL_COST 7  // multiplier of a small-bin pivot's probes (8-part A/B on C4 and C5)
#endif
#ifndef TCB_SLAB_COST
#define TCB_SLAB_COST 10  // a cold probe of a pivot whose table spills to the global slab
#endif
#ifndef TCB_WARP_COST
#define TCB_WARP_COST 12  // a warp-bin (hash) probe (8-part A/B: profiles/r02_ab_costs_env.log)
#endif
constexpr uint64_t kItemCost = TCB_ITEM_COST;
constexpr uint64_t kSegRowCost = TCB_SEG_COST;  // per member of N+(v), per segment

__global__ void k_pivot_wedges(const uint4* __restrict__ rowd, const uint32_t* __restrict__ col,
                               const uint32_t* __restrict__ src, uint64_t E, uint32_t r0, uint32_t dense_cost,
                               uint32_t cold_cost, uint32_t warp_cost, uint32_t small_cost, uint32_t slab_cost,
                               PivotClass pc,
                               unsigned long long* __restrict__ jv) {
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < E; base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = base + threadIdx.x;
    const bool ok = e < E;
    const uint32_t v = ok ? col[e] : 0xffffffffu;
    // cost of item e in candidate-probe units: its sparse suffix (bitmap
    // probes 1, cold hash probes cold_cost, warp-bin probes warp_cost) and
    // its dense core part, if any, as one k_join_dense item (dense_cost);
    // a warp's sum fits 32 bits
    uint32_t w = 0;
    if (ok) {
      const RowGeo r = load_row(rowd, r0, src[e]);
      const uint32_t a = (uint32_t)e + 1, se = r.end - r.cc(), ce = min(r.cold_end(), se);
      const uint32_t cold = ce > a ? ce - a : 0u;          // hash-probed candidates
      const uint32_t hot = se > max(a, ce) ? se - max(a, ce) : 0u;  // bitmap-probed
      uint32_t din = 0;
      const int cls = pc(v, din);
      // a pivot with more cold members than the SMEM table holds probes a
      // per-CTA global slab (k_join_cta): slab_cost per cold probe
      const RowGeo rv = load_row(rowd, r0, v);
      const uint32_t cc = (cls == 1 && 2 * (rv.d() - rv.h()) > kCtaSmemSlots) ? slab_cost : cold_cost;
      w = cls == 0 ? warp_cost * (cold + hot) : hot + cc * cold;
      if (cls == 2) w *= small_cost;  // one warp per pivot (k_join_small)
      if (r.didx != kNoDense && a < r.end) w += dense_cost;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, v);
    const uint32_t sum = __reduce_add_sync(peers, w);
    if (ok && (int)lane_id() == __ffs(peers) - 1 && sum) atomicAdd(&jv[v - r0], (unsigned long long)sum);
  }
}

struct PivotCost {  // pivots r0 + i (the isolated ranks [0, r0) have no work)
  const uint32_t* off;
  const uint32_t* inoff;
  const unsigned long long* jv;
  uint64_t item_cost, seg_cost;
  uint32_t r0;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    const uint64_t v = r0 + i;
    const uint64_t dv = off[v + 1] - off[v], din = inoff[v + 1] - inoff[v];
    if (!dv || !din) return 0;
    return jv[i] + item_cost * din + seg_cost * dv * ((din + kCtaSegItems - 1) / kCtaSegItems);
  }
};

__global__ void k_part_bounds(const uint64_t* __restrict__ prefix, uint32_t r0, uint32_t n, uint64_t total,
                              uint32_t parts, uint64_t* __restrict__ bounds) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p > parts) return;
  if (p == 0 || p == parts) {
    bounds[p] = p == 0 ? 0 : n;
    return;
  }
  const uint64_t target = (uint64_t)((double)total * p / parts);
  uint64_t lo = 0, hi = n - r0;  // first pivot r0 + i with prefix[i] >= target
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (prefix[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[p] = r0 + lo;
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

// A hot chunk's 8-bit hit mask (read once, by the row pass) is stored with
// the streaming (evict-first) hint so the 2.9 GB of mask bytes do not push
// the probed adjacency out of L2 (C4 CTA join 24.12 -> 24.08 ms).
#ifndef TCB_MASK_CS
#define TCB_MASK_CS 1
#endif
__device__ __forceinline__ void st_mask(uint8_t* p, uint32_t m) {
#if TCB_MASK_CS
  asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "r"(m) : "memory");
#else
  *p = (uint8_t)m;
#endif
}

// 8 hot ids (16-bit offsets from h0) per 16-byte chunk: bitmap probes (all
// 8 unpredicated: predicating the elements outside [b, e) measured slower,
// profiles/README.md).
__device__ __forceinline__ uint32_t hot_u16(const uint4& q, int i) {
  const uint32_t w = (i < 2) ? q.x : (i < 4) ? q.y : (i < 6) ? q.z : q.w;
  return (i & 1) ? (w >> 16) : (w & 0xffffu);
}

// Hit mask (bit i = element i of chunk c is in [b,e) and a member of N+(v)).
__device__ __forceinline__ uint32_t hot_hit_mask(const uint4& q, uint32_t c, uint32_t b, uint32_t e,
                                                 const uint32_t* bm) {
  const uint32_t p0 = c << 3;
  const uint32_t lo = b > p0 ? b - p0 : 0u;
  const uint32_t hi = e - p0 < 8u ? e - p0 : 8u;
  const uint32_t valid = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
  uint32_t hits = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t y = hot_u16(q, i);
    hits |= ((bm[y >> 5] >> (y & 31)) & 1u) << i;
  }
  return hits & valid;
}

// Cold-member prefilter of a pivot: one bit per 11-bit Fibonacci hash of
// each member below the hot window (2048 bits of SMEM).  Cold candidates
// close a triangle about once in 10^3 probes at RMAT s24, so a filter miss
// (one LDS + shift) replaces most linear-probe chains.
constexpr uint32_t kColdFilterWords = 64;
__device__ __forceinline__ uint32_t cfilt_bit(uint32_t x) { return (x * 0x9E3779B1u) >> 21; }
__device__ __forceinline__ bool cfilt_test(const uint32_t* cf, uint32_t x) {
  const uint32_t f = cfilt_bit(x);
  return (cf[f >> 5] >> (f & 31)) & 1u;
}

// 4 cold ids (32-bit) per chunk: hash probes (behind the prefilter cf when
// given).
template <bool kPerVertex, typename Sink>
__device__ __forceinline__ uint32_t probe_cold(const uint4& q, uint32_t c, uint32_t b, uint32_t e,
                                               const uint32_t* tab, uint32_t mask, uint32_t shift,
                                               const Sink& sink, const uint32_t* cf = nullptr) {
  const uint32_t xs[4] = {q.x, q.y, q.z, q.w};
  const uint32_t p0 = c << 2;
  uint32_t h = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint32_t p = p0 + t;
    if (p >= b && p < e && (cf == nullptr || cfilt_test(cf, xs[t])) && hash_find(tab, mask, shift, xs[t])) {
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

// A warp walks chunk range [fb, fe) of a segment list staged in SMEM (item i:
// chunk start pre[i] (pre[ni] = total), element range [sb[i], se[i]), original
// index sidx[i]), kWin windows of 32 chunks per step: every window's chunk is
// mapped to its item first, then all kWin int4 loads are issued, then probed
// (kWin loads in flight per lane).  fn(q, c, b, e, k) -> hits.
template <int kIdsPerChunk, int kWin, typename T, typename ChunkFn>
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
  for (uint32_t f = fb; f < fe; f += 32 * kWin) {
    uint32_t kk[kWin], bb[kWin], ee[kWin], cc[kWin];
    bool vv[kWin];
    uint4 qq[kWin];
#pragma unroll
    for (int w = 0; w < kWin; ++w) {
      const uint32_t fw = f + 32 * w;
      const uint32_t j = k0 + 1 + lane;  // items starting inside (fw, fw+32)
      const uint32_t st = pre[min(j, ni)];
      const uint32_t bit = (j < ni && st < fw + 32) ? (1u << (st - fw)) : 0u;
      const uint32_t m = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t k = k0 + __popc(m & ((2u << lane) - 1u));
      k0 += __popc(__ballot_sync(0xffffffffu, j < ni && st <= fw + 32));  // item holding fw+32
      const uint32_t fl = fw + lane;
      vv[w] = fl < fe;
      kk[w] = vv[w] ? k : 0;
      bb[w] = sb[kk[w]];
      ee[w] = se[kk[w]];
      cc[w] = (bb[w] >> kShift) + (fl - pre[kk[w]]);
    }
#pragma unroll
    for (int w = 0; w < kWin; ++w) qq[w] = vv[w] ? __ldg(base4 + cc[w]) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int w = 0; w < kWin; ++w) {
      if (vv[w]) {
        const uint32_t x = fn(qq[w], cc[w], bb[w], ee[w], kk[w]);
        h += x;
        if (icnt && x) atomicAdd(&icnt[sidx[kk[w]]], x);
      }
    }
  }
  return h;
}

// ---- item geometry (from the in-edge index) --------------------------------------

// Level-1 item = in-edge (e, u) of pivot v = col[e]: its wedge suffix is
// col[e+1 .. off[u+1]).  CTA/small bins take it from the row descriptor
// (graph.cuh RowGeo, one 32-byte sector) split into the sparse hot part
// (16-bit colH up to Ht) and the cold part (col): {hb, he, cb, ce} (empty
// ranges have he <= hb / ce <= cb).  mo = the item's first per-vertex mask
// byte (rowbase + RowMasks::P(k), k = e - beg, sparse hot part only).
// A dense row's core part is joined by k_join_dense.
// CTA bin, staging of the next segment's in-edge records one segment ahead:
// 0 = none (plain loads at staging), 1 = one bulk copy (TMA, cp.async.bulk +
// mbarrier) per segment, 2 = per-thread cp.async (LDGSTS) of the records each
// thread stages.  Measured at C4 (profiles/README.md): the total-only join
// gains ~1% with 2; in the per-vertex join the 4 KB record buffer lifts the
// CTA past the SMEM budget of 6 resident CTAs at the driver's 80% carveout
// and costs 24% (47.7 vs 38.5 ms), so the per-vertex instantiation stages
// with plain loads (kPrefetch below).
#ifndef TCB_PREFETCH
#define TCB_PREFETCH 2
#endif
// Per-vertex hits t[x] of the CTA / small bins: 1 = 8-bit hit masks per hot
// chunk folded row by row (k_pv_rows); 0 = per-hit increments of SMEM
// counters for the top ranks (16-bit halves, flushed every kTopFlushSegs
// segments) and global atomics below them -- no masks, no row pass.
#ifndef TCB_PV_MASKS
#define TCB_PV_MASKS 1
#endif
// CTA bin: L2 bulk prefetch of the next segment's suffixes (0 off, 1 hot,
// 2 hot + cold)
#ifndef TCB_L2PF
#define TCB_L2PF 0
#endif
constexpr uint32_t kTopFlushSegs = 120;  // <= 65535 / kCtaSegItems increments per counter between flushes
struct ItemGeo {
  const uint4* rowd;  // tc_graph::rowd, rows [r0, n)
  uint32_t r0;
  __device__ __forceinline__ uint4 hotcold(uint2 eu, uint64_t* mo) const {
    const uint32_t e = eu.x;
    const RowGeo r = load_row(rowd, r0, eu.y);
    if (e + 1 >= r.end) return make_uint4(0, 0, 0, 0);
    const uint32_t cold_end = r.cold_end();
    const uint4 it = (e + 1 >= cold_end) ? make_uint4(r.O + (e + 1 - cold_end), r.Ht, 0, 0)
                                         : make_uint4(r.O, r.Ht, e + 1, cold_end);
    if (mo != nullptr && it.y > it.x) *mo = r.rowbase + r.masks().P(e - r.beg);
    return it;
  }
};

// ---- warp bin ------------------------------------------------------------------

// Pivots with d+ <= 64 (warp-bin segments of <= 64 in-edge items).  A warp
// takes a group of kWarpGroup consecutive segments at once: every pivot gets
// its own 128-slot hash table (warp-private SMEM) and the group's items are
// packed into 32-lane batches -- a uniform-degree graph has ~8 items per
// pivot, so one segment per warp step would leave most lanes idle and pay
// the segment's dependent memory round trips four times as often.  Items are
// the u32 suffix ranges of col from their 32-byte records (a dense row's core
// members, its last cc, are k_join_dense's).  Per-vertex: the CTA bin's row
// pass reads hit masks for every item, so this bin zeroes its items' mask
// bytes (its hits go to per-hit counters instead); d+(v) = 0 pivots come here
// for that alone.
#ifndef TCB_WARP_GROUP
#define TCB_WARP_GROUP 4
#endif
constexpr int kWarpGroup = TCB_WARP_GROUP;
#ifndef TCB_LANE_ITEM_CHUNKS
#define TCB_LANE_ITEM_CHUNKS 4
#endif
// a batch whose items all span <= this many 4-id chunks is walked lane by lane
constexpr uint32_t kLaneItemChunks = TCB_LANE_ITEM_CHUNKS;

template <bool kPerVertex, typename Sink>
__device__ __forceinline__ uint32_t warp_join_group(const uint4* __restrict__ irec, const uint32_t (&gi0)[kWarpGroup],
                                                    const uint32_t (&gpre)[kWarpGroup + 1], uint32_t probe_mask,
                                                    const uint32_t* __restrict__ col, const uint32_t* tabs,
                                                    uint32_t mask, uint32_t shift, const Sink& sink,
                                                    uint8_t* __restrict__ masks, uint32_t* item_cnt,
                                                    uint32_t (&hseg)[kWarpGroup]) {
  const unsigned lane = lane_id();
  const uint4* col4 = reinterpret_cast<const uint4*>(col);
  uint32_t hits = 0;
  const uint32_t nitems = gpre[kWarpGroup];
  for (uint32_t ib = 0; ib < nitems; ib += 32) {
    const uint32_t p = ib + lane;
    uint32_t b = 0, e = 0, nch = 0, u = 0, tj = 0;
#pragma unroll
    for (int j = 1; j < kWarpGroup; ++j) tj += p >= gpre[j] ? 1u : 0u;  // the item's segment
    if (p < nitems) {
      const uint32_t my = gi0[tj] + (p - gpre[tj]);
      // the item record: its suffix in col is [e+1, e+1 + cold + sparse hot)
      // (the cold members are followed by the hot ones in col)
      const uint4 g4 = ld_stream(irec + 2 * (uint64_t)my), ax = ld_stream(irec + 2 * (uint64_t)my + 1);
      u = ax.y;
      b = ax.x + 1;
      const uint32_t hot = g4.y > g4.x ? g4.y - g4.x : 0u;
      e = b + (g4.w > g4.z ? g4.w - g4.z : 0u) + hot;
      nch = (b < e && ((probe_mask >> tj) & 1u)) ? ((e + 3) >> 2) - (b >> 2) : 0u;
      if (kPerVertex && TCB_PV_MASKS && hot && masks) {
        // the row pass reads every item's sparse hot mask bytes: zero this
        // item's (its hits are counted here, per hit)
        uint8_t* z = masks + (ax.z | ((uint64_t)ax.w << 32));
        const uint32_t nb = ((g4.y + 7) >> 3) - (g4.x >> 3);
        for (uint32_t t = 0; t < nb; ++t) z[t] = 0;
      }
    }
    const uint32_t ne = __ballot_sync(0xffffffffu, nch > 0);
    if (!ne) continue;
    if (__reduce_max_sync(0xffffffffu, nch) <= kLaneItemChunks) {
      // short items (a uniform-degree graph's): every lane walks its own
      // item's few chunks -- no chunk -> item mapping, no shuffles
      uint32_t hl = 0;
      for (uint32_t c = b >> 2, ce = c + nch; c < ce; ++c) hl += probe_cold<kPerVertex>(__ldg(col4 + c), c, b, e,
                                                                                 tabs + tj * kWarpTable, mask, shift,
                                                                                 sink);
      hits += hl;
      if (kPerVertex) {
#pragma unroll
        for (int j = 0; j < kWarpGroup; ++j) hseg[j] += tj == (uint32_t)j ? hl : 0u;
        if (hl) atomicAdd(&sink.t_rank[u], (unsigned long long)hl);
      }
      continue;
    }
    // compact the non-empty items to the low lanes (item_of needs nch >= 1);
    // lane L takes the item of the (L+1)-th non-empty lane
    uint32_t owner_u;
    {
      const uint32_t from = lane < (uint32_t)__popc(ne) ? __fns(ne, 0, lane + 1) : lane;
      b = __shfl_sync(0xffffffffu, b, from);
      e = __shfl_sync(0xffffffffu, e, from);
      nch = __shfl_sync(0xffffffffu, nch, from);
      tj = __shfl_sync(0xffffffffu, tj, from);
      owner_u = __shfl_sync(0xffffffffu, u, from);
      if (lane >= (uint32_t)__popc(ne)) nch = 0;
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
      const uint32_t sk = __shfl_sync(0xffffffffu, start, k), tk = __shfl_sync(0xffffffffu, tj, k);
      const uint32_t f = base + lane;
      if (f < total) {
        const uint32_t c = (bk >> 2) + (f - sk);
        const uint32_t x =
            probe_cold<kPerVertex>(__ldg(col4 + c), c, bk, ek, tabs + tk * kWarpTable, mask, shift, sink);
        hits += x;
        if (kPerVertex) {
#pragma unroll
          for (int j = 0; j < kWarpGroup; ++j) hseg[j] += tk == (uint32_t)j ? x : 0u;
          if (x) atomicAdd(&item_cnt[k], x);
        }
      }
    }
    if (kPerVertex) {
      __syncwarp();
      const uint32_t c = item_cnt[lane];
      if (c) atomicAdd(&sink.t_rank[owner_u], (unsigned long long)c);
      __syncwarp();
    }
  }
  return hits;
}

// Warp bin kernel: groups of kWarpGroup segments per warp step, the CTA
// shares the per-vertex top-rank counters (dynamic SMEM, pv only).  The
// segment count is read on the device.
// 5 CTAs per SM (51 registers): warp bin 1.64 -> 1.52 ms at C4 per-vertex
// (a small spill), C2 0.698 -> 0.675 ms
#ifndef TCB_WARP_MINB
#define TCB_WARP_MINB 5
#endif
template <bool kPerVertex>
__global__ void __launch_bounds__(kJoinThreads, TCB_WARP_MINB) k_join_warp(
    const uint32_t* __restrict__ off, const uint4* __restrict__ rowd, uint32_t r0, const uint32_t* __restrict__ col,
    const uint4* __restrict__ irec, const uint4* __restrict__ segs, const uint32_t* __restrict__ nsegs_p,
    const uint32_t* __restrict__ inoff, uint32_t v_lo, uint32_t v_hi,
    uint32_t gsz, uint32_t rc, uint32_t ncnt, uint8_t* __restrict__ masks,
    unsigned long long* __restrict__ t_rank, unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t top_cnt[];
  __shared__ uint32_t s_tab[kJoinWarps][kWarpGroup * kWarpTable];
  __shared__ uint32_t s_item[kJoinWarps][32];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  // direct mode (inoff != null, no count plan): segment j is pivot v_lo + j
  // with all its in-edge items -- every pivot of the graph fits one segment
  const uint32_t nsegs = inoff ? v_hi - v_lo : *nsegs_p;
  uint32_t* tabs = s_tab[warp];
  for (uint32_t s = lane; s < kWarpGroup * kWarpTable; s += 32) tabs[s] = kEmpty;
  if (kPerVertex) {
    for (uint32_t i = threadIdx.x; i < ncnt; i += kJoinThreads) top_cnt[i] = 0;
    __syncthreads();
  }
  __syncwarp();
  const uint32_t mask = kWarpTable - 1, shift = 32 - log2_pow2(kWarpTable);
  const PvSink<false> sink{top_cnt, rc, t_rank, g_pv_dbg};
  unsigned long long acc = 0;
  const uint32_t gw = blockIdx.x * kJoinWarps + warp, nw = gridDim.x * kJoinWarps;
  // gsz (<= kWarpGroup) segments per warp step: kWarpGroup when there are
  // enough segments to keep every resident warp busy, else 1
  for (uint64_t g0 = (uint64_t)gw * gsz; g0 < nsegs; g0 += (uint64_t)nw * gsz) {
    // lane j < gsz: segment g0 + j's descriptor and pivot row
    uint4 sgl = make_uint4(0, 0, 0, 0);
    uint32_t nbl = 0, dvl = 0;
    if (lane < gsz && g0 + lane < nsegs) {
      if (inoff) {
        const uint32_t v = v_lo + (uint32_t)(g0 + lane);
        sgl = make_uint4(v, inoff[v], inoff[v + 1], 0);
      } else {
        sgl = segs[g0 + lane];
      }
      nbl = off[sgl.x];
      dvl = off[sgl.x + 1] - nbl;
    }
    uint32_t gv[kWarpGroup], gi0[kWarpGroup], gpre[kWarpGroup + 1], gnb[kWarpGroup], mpre[kWarpGroup + 1];
    uint32_t probe_mask = 0;
    gpre[0] = mpre[0] = 0;
#pragma unroll
    for (int j = 0; j < kWarpGroup; ++j) {
      gv[j] = __shfl_sync(0xffffffffu, sgl.x, j);
      gi0[j] = __shfl_sync(0xffffffffu, sgl.y, j);
      const uint32_t ni = __shfl_sync(0xffffffffu, sgl.z, j) - gi0[j];
      gnb[j] = __shfl_sync(0xffffffffu, nbl, j);
      const uint32_t dv = __shfl_sync(0xffffffffu, dvl, j);
      gpre[j + 1] = gpre[j] + ni;
      mpre[j + 1] = mpre[j] + dv;
      probe_mask |= (dv > 0 ? 1u : 0u) << j;
    }
    // the group's pivot members, flattened over the lanes, into their tables
    for (uint32_t q = lane; q < mpre[kWarpGroup]; q += 32) {
      uint32_t j = 0;
#pragma unroll
      for (int t = 1; t < kWarpGroup; ++t) j += q >= mpre[t] ? 1u : 0u;
      hash_insert(tabs + j * kWarpTable, mask, shift, col[gnb[j] + (q - mpre[j])]);
    }
    __syncwarp();
    uint32_t hseg[kWarpGroup];
#pragma unroll
    for (int j = 0; j < kWarpGroup; ++j) hseg[j] = 0;
    const uint32_t h = warp_join_group<kPerVertex>(irec, gi0, gpre, probe_mask, col, tabs, mask, shift, sink, masks,
                                                   s_item[warp], hseg);
    __syncwarp();
    acc += h;
    if (kPerVertex) {
#pragma unroll
      for (int j = 0; j < kWarpGroup; ++j) {
        const uint32_t hw = warp_sum(hseg[j]);
        if (lane == 0 && hw) atomicAdd(&t_rank[gv[j]], (unsigned long long)hw);
      }
    }
#pragma unroll
    for (int j = 0; j < kWarpGroup; ++j)
      if ((probe_mask >> j) & 1u)
        for (uint32_t s = lane; s < kWarpTable; s += 32) tabs[j * kWarpTable + s] = kEmpty;
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
  if (kPerVertex) {
    __syncthreads();
    flush_top<false>(top_cnt, ncnt, rc, t_rank);
  }
}

// ---- dense core join ------------------------------------------------------------
// The core part of every dense item (graph.cuh tc_graph::dine): the item's
// row keeps its members among the top ranks [cb, n) as a bitmap of cw words,
// and so does the pivot (its own bitmap when its row is dense, else built
// from its few core members), so the join is a word-parallel AND + popcount
// -- no per-candidate probes.  One warp per segment (<= kDenseSeg items of
// one pivot); lane j holds pivot words j + 32k (P[k]; every member ranks
// above v, so no suffix bound is needed) and loads the same words of each
// item's row (coalesced, 128 B per k; lanes whose pivot word is zero skip
// the load), 4 items in flight.
// Per-vertex: t[u] += the item's hits, t[v] += the segment's; t[x] for the
// hit bits through per-lane bit-sliced counters: the 4 items' hit words are
// added into kPlanes bit planes per word by carry-save adders (c0..c(P-1),
// count = sum c_p 2^p; ~6 ops per item-word instead of an atomic per hit)
// and folded into the CTA's SMEM counters every (2^kPlanes - 4) items.
constexpr int kDenseThreads = 256;
constexpr int kDenseWarps = kDenseThreads / 32;
// The kernel is latency-bound on the row-word loads.  Per-vertex: held to 64
// registers (4 CTAs/SM), 8 items (16 row words) in flight per step with a
// three-level carry-save tree, 10 bit planes, and the planes folded into the
// SMEM counters by a bit-matrix transpose (C4 dense 5.27 -> 4.85 ms; other
// plane counts, the per-bit fold, Harley-Seal trees and the uncapped kernel
// measured slower: profiles/README.md).  Total-only: 4 items per step at
// 8 CTAs/SM (32 registers).
#ifndef TCB_DENSE_MINB
#define TCB_DENSE_MINB 4
#endif
#ifndef TCB_DENSE_PLANES
#define TCB_DENSE_PLANES 10
#endif
constexpr int kPlanes = TCB_DENSE_PLANES;  // bit planes per counter: a fold every 2^kPlanes - 4 items
#ifndef TCB_DENSE_GROUP
#define TCB_DENSE_GROUP 8
#endif
static_assert(TCB_DENSE_GROUP == 4 || TCB_DENSE_GROUP == 8, "dense group of 4 or 8 items");

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (a & c) | (b & c); }

template <bool kPV, int kCW>
__global__ void __launch_bounds__(kDenseThreads, kPV ? TCB_DENSE_MINB : 8) k_join_dense(
    const uint4* __restrict__ dseg, const uint32_t* __restrict__ dsoff, uint32_t v_lo, uint32_t v_hi,
    unsigned int* __restrict__ queue, const uint32_t* __restrict__ dine, const uint32_t* __restrict__ drow,
    const uint32_t* __restrict__ cbits, uint32_t cw, uint32_t cb, uint32_t cbh, uint32_t core_min,
    const uint4* __restrict__ rowd, uint32_t r0, const uint16_t* __restrict__ colH,
    unsigned long long* __restrict__ t_rank, unsigned long long* __restrict__ total) {
  // kCW core words per lane: 2 for the default 2048-rank core (or smaller),
  // 3 for a 3072-rank core (TCB_CORE_BITS=3072 at graph build); items per
  // step (row loads in flight): 8 per-vertex at 2 words per lane, else 4
  constexpr int kDG = kPV && kCW == 2 ? TCB_DENSE_GROUP : 4;
  __shared__ uint32_t s_p[kDenseWarps][32 * kCW];              // pivot core words (non-dense pivots)
  __shared__ uint32_t s_cnt[kPV ? 32 * 32 * kCW : 1];          // t[x] of core ranks, this CTA
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  if (kPV) {
    for (uint32_t i = threadIdx.x; i < 32 * 32 * kCW; i += kDenseThreads) s_cnt[i] = 0;
    __syncthreads();
  }
  for (uint32_t i = lane; i < 32 * kCW; i += 32) s_p[warp][i] = 0;
  __syncwarp();
  const uint32_t sb = dsoff[v_lo], se = dsoff[v_hi];  // this part's segments (pivots [v_lo, v_hi))
  uint32_t c[kPV ? kPlanes : 1][kCW];
#pragma unroll
  for (int p = 0; p < (kPV ? kPlanes : 1); ++p)
#pragma unroll
    for (int k = 0; k < kCW; ++k) c[p][k] = 0;
  uint32_t since = 0;  // items added to the planes since the last fold
  auto fold = [&]() {
    // bit-matrix transpose of the planes (16 x 32 as two 16 x 16 blocks, four
    // swap stages): word i then holds bit i's count in its low half and bit
    // i + 16's in its high half
    static_assert(kPlanes <= 16, "transpose fold holds at most 16 planes");
#pragma unroll
    for (int k = 0; k < kCW; ++k) {
      const uint32_t j = lane + 32 * k;
      if (j >= cw) continue;
      uint32_t A[16];
#pragma unroll
      for (int p = 0; p < 16; ++p) A[p] = p < (kPV ? kPlanes : 1) ? c[p < (kPV ? kPlanes : 1) ? p : 0][k] : 0u;
#pragma unroll
      for (int st = 0; st < 4; ++st) {
        const int sh = 8 >> st;
        const uint32_t m = st == 0 ? 0x00FF00FFu : st == 1 ? 0x0F0F0F0Fu : st == 2 ? 0x33333333u : 0x55555555u;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          if (r & sh) continue;
          const uint32_t t = ((A[r] >> sh) ^ A[r + sh]) & m;
          A[r + sh] ^= t;
          A[r] ^= t << sh;
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (A[i] & 0xffffu) atomicAdd(&s_cnt[32 * j + i], A[i] & 0xffffu);
        if (A[i] >> 16) atomicAdd(&s_cnt[32 * j + 16 + i], A[i] >> 16);
      }
#pragma unroll
      for (int p = 0; p < (kPV ? kPlanes : 1); ++p) c[p][k] = 0;
    }
    since = 0;
  };
  unsigned long long acc = 0;
  while (true) {
    uint32_t q = 0;
    if (lane == 0) q = atomicAdd(queue, 1u);
    q = sb + __shfl_sync(0xffffffffu, q, 0);
    if (q >= se) break;
    const uint4 sg = dseg[q];
    const uint32_t v = sg.x;
    // pivot core words
    uint32_t P[kCW];
    {
      const RowGeo rv = load_row(rowd, r0, v);
      if (rv.didx != kNoDense) {
#pragma unroll
        for (int k = 0; k < kCW; ++k) {
          const uint32_t j = lane + 32 * k;
          P[k] = j < cw ? __ldg(cbits + (uint64_t)rv.didx * cw + j) : 0u;
        }
      } else {
        // fewer than core_min core members: the last entries of its hot row
        const uint32_t h = rv.h();
        for (uint32_t l = lane; l < core_min && l < h; l += 32) {
          const uint32_t y = colH[rv.Hf - 1 - l];
          if (y >= cbh) atomicOr(&s_p[warp][(y - cbh) >> 5], 1u << ((y - cbh) & 31));
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kCW; ++k) {
          P[k] = s_p[warp][lane + 32 * k];
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kCW; ++k) s_p[warp][lane + 32 * k] = 0;
        __syncwarp();
      }
    }
    uint32_t hseg = 0;
    const uint32_t* cl = cbits + lane;  // this lane's words: + didx * cw + 32 k
    for (uint32_t base = sg.y; base < sg.z; base += 32) {
      // 32 items per round: lane l loads item l's dense index (coalesced) and,
      // per-vertex, its row rank; lane l also owns item l's t[u] update
      const uint32_t cnt = min(32u, sg.z - base);
      const uint32_t myd = lane < cnt ? __ldg(dine + base + lane) : kNoDense;
      const uint32_t myu = (kPV && lane < cnt) ? __ldg(drow + myd) : 0u;
      uint32_t mysum = 0;
      for (uint32_t a0 = 0; a0 < cnt; a0 += kDG) {
        uint32_t m[kDG][kCW];
#pragma unroll
        for (int a = 0; a < kDG; ++a) {
          const uint32_t d = __shfl_sync(0xffffffffu, myd, (a0 + a) & 31);
          const uint32_t* row = cl + d * cw;  // d * cw < 2^32 (ndense * core_words words)
#pragma unroll
          for (int k = 0; k < kCW; ++k) m[a][k] = (a0 + a < cnt && P[k]) ? __ldg(row + 32 * k) & P[k] : 0u;
        }
#pragma unroll
        for (int a = 0; a < kDG; ++a) {
          uint32_t hi = 0;
#pragma unroll
          for (int k = 0; k < kCW; ++k) hi += __popc(m[a][k]);
          hseg += hi;
          if (kPV) {
            const uint32_t sum = __reduce_add_sync(0xffffffffu, hi);
            mysum = lane == a0 + a ? sum : mysum;
          }
        }
        if (kPV) {
#pragma unroll
          for (int k = 0; k < kCW; ++k) {
            // carry-save: c0 + m0 + m1 + m2 + m3 + 2 c1 -> c0 + 2 c1 + 4 k4
            const uint32_t k1 = maj3(c[0][k], m[0][k], m[1][k]);
            c[0][k] ^= m[0][k] ^ m[1][k];
            const uint32_t k2 = maj3(c[0][k], m[2][k], m[3][k]);
            c[0][k] ^= m[2][k] ^ m[3][k];
            uint32_t k4 = maj3(c[kPV ? 1 : 0][k], k1, k2);
            c[kPV ? 1 : 0][k] ^= k1 ^ k2;
            int p0 = 2;
            if constexpr (kDG == 8) {  // m4..m7: c0 + 2 c1 + 4 c2 + 8 k8
              const uint32_t k1b = maj3(c[0][k], m[4 % kDG][k], m[5 % kDG][k]);
              c[0][k] ^= m[4 % kDG][k] ^ m[5 % kDG][k];
              const uint32_t k2b = maj3(c[0][k], m[6 % kDG][k], m[7 % kDG][k]);
              c[0][k] ^= m[6 % kDG][k] ^ m[7 % kDG][k];
              const uint32_t t2b = maj3(c[kPV ? 1 : 0][k], k1b, k2b);
              c[kPV ? 1 : 0][k] ^= k1b ^ k2b;
              const uint32_t k8 = maj3(c[kPV ? 2 : 0][k], k4, t2b);
              c[kPV ? 2 : 0][k] ^= k4 ^ t2b;
              k4 = k8;
              p0 = 3;
            }
#pragma unroll
            for (int p = 2; p < (kPV ? kPlanes : 1); ++p) {
              if (p < p0) continue;
              const uint32_t t = c[p][k] & k4;
              c[p][k] ^= k4;
              k4 = t;
            }
          }
          since += kDG;
          if (since > (1u << kPlanes) - 1 - kDG) fold();
        }
      }
      if (kPV && mysum) atomicAdd(&t_rank[myu], (unsigned long long)mysum);
    }
    acc += hseg;
    if (kPV) {
      const uint32_t hv = warp_sum(hseg);
      if (lane == 0 && hv) atomicAdd(&t_rank[v], (unsigned long long)hv);
    }
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
  if (kPV) {
    if (since) fold();
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 32 * cw; i += kDenseThreads)
      if (s_cnt[i]) atomicAdd(&t_rank[cb + i], (unsigned long long)s_cnt[i]);
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
// Dynamic SMEM: [hot bitmap nbm words][cold hash kCtaSmemSlots].
template <bool kPerVertex>
__global__ void __launch_bounds__(kCtaThreads, kCtaMinBlocks) k_join_cta(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint4* __restrict__ rowd, uint32_t r0,
    const uint16_t* __restrict__ colH, const uint4* __restrict__ irec,
    const uint4* __restrict__ segs, const uint32_t* __restrict__ nsegs_p, unsigned int* __restrict__ queue,
    uint32_t h0, uint32_t nbm, uint32_t stab_slots, uint32_t slab_cap, uint32_t* __restrict__ gslab,
    uint8_t* __restrict__ masks, uint32_t rc, uint32_t ncnt, unsigned long long* __restrict__ t_rank,
    unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t dyn[];
  constexpr bool kMasks = kPerVertex && TCB_PV_MASKS;
  constexpr bool kHits = kPerVertex && !TCB_PV_MASKS;
  constexpr int kPF = kPerVertex ? 0 : TCB_PREFETCH;  // staging prefetch (see TCB_PREFETCH)
  __shared__ unsigned long long s_hmo[kMasks ? kCtaSegItems : 1];  // hot items' mask offsets
  __shared__ uint16_t s_hidx[kHits ? kCtaSegItems : 1];  // hot item -> segment index (t[u] counts)
  __shared__ uint32_t s_hb[kCtaSegItems], s_he[kCtaSegItems], s_hpre[kCtaSegItems + 1];
  __shared__ uint32_t s_cb[kCtaSegItems], s_ce[kCtaSegItems], s_cpre[kCtaSegItems + 1];
  __shared__ uint16_t s_cidx[kPerVertex ? kCtaSegItems : 1];  // cold item -> segment index (t[u] counts)
  __shared__ uint32_t s_icnt[kPerVertex ? kCtaSegItems : 1];
  __shared__ uint32_t s_cf[kColdFilterWords];  // cold-member prefilter
  __shared__ uint32_t s_hits, s_cold, s_nl;
  __shared__ uint32_t s_wl[kCtaWarps];
  __shared__ unsigned long long s_wc[kCtaWarps];
  __shared__ uint32_t s_desc[6];  // current segment: v, i0, ni, off[v], d+(v), queue index
  __shared__ unsigned long long s_ctot;
  // the segment's in-edge records {e, u}, bulk-copied (TMA) one segment ahead
  __shared__ __align__(16) uint4 s_ine[kPF ? kCtaSegItems : 1];  // the segment's item geometry records
  __shared__ __align__(8) unsigned long long s_mbar;
  __shared__ uint4 s_sgn;  // the next segment, held by thread 0
  uint32_t* bm = dyn;
  uint32_t* stab = dyn + nbm;
  uint32_t* top = stab + kCtaSmemSlots;  // kHits: ncnt 16-bit counters for ranks [rc, rc + ncnt)
  uint32_t* gtab = gslab + (uint64_t)blockIdx.x * slab_cap;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t nsegs = *nsegs_p;
  for (uint32_t i = threadIdx.x; i < nbm; i += kCtaThreads) bm[i] = 0;
  for (uint32_t i = threadIdx.x; i < kCtaSmemSlots; i += kCtaThreads) stab[i] = kEmpty;
  for (uint32_t i = threadIdx.x; i < slab_cap; i += kCtaThreads) gtab[i] = kEmpty;
  for (uint32_t i = threadIdx.x; i < kColdFilterWords; i += kCtaThreads) s_cf[i] = 0;
  if (kPerVertex)
    for (uint32_t i = threadIdx.x; i < kCtaSegItems; i += kCtaThreads) s_icnt[i] = 0;
  if (kHits)
    for (uint32_t i = threadIdx.x; i < ncnt / 2; i += kCtaThreads) top[i] = 0;
  // cold hits (x < h0) go straight to global atomics; hot hits leave as masks
  // (kMasks) or go to the top counters / global atomics (kHits)
  const PvSink<true> sink{nullptr, 0xffffffffu, t_rank, g_pv_dbg};
  const PvSink<true> hsink{top, rc, t_rank, g_pv_dbg};
  uint32_t segs_since_flush = 0;
  unsigned long long acc = 0;
  // Segments are pipelined one ahead by thread 0: the next segment is taken
  // from the queue at the top of the current one, and once the current
  // segment's in-edge records have been read (after the staging scans) the
  // next segment's slice of the in-edge index is bulk-copied into s_ine by the
  // TMA unit, landing while this segment is walked.  A segment therefore
  // starts on SMEM descriptors and records instead of a chain of global loads.
  auto load_desc = [&](uint32_t q, const uint4& sg) {
    if (q < nsegs) {
      s_desc[0] = sg.x;
      s_desc[1] = sg.y;
      s_desc[2] = sg.z - sg.y;
      s_desc[3] = off[sg.x];
      s_desc[4] = off[sg.x + 1] - s_desc[3];
    }
    s_desc[5] = q;
  };
  // the segment's item geometry (the first 16 bytes of records [i0, i1)) -> s_ine
  // (records are 32 bytes, the staging takes their first 16: a per-thread
  // cp.async gather, no contiguous bulk copy)
  static_assert(kPF != 1, "TCB_PREFETCH=1 (bulk copy of the segment's records) needs contiguous 16-byte records");
  auto issue_ine = [&](const uint4&) {};
  uint32_t phase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&s_mbar, 1);
    const uint32_t q = atomicAdd(queue, 1u);
    if (q < nsegs) {
      s_sgn = segs[nsegs - 1 - q];  // heaviest (top ranks) first
      if constexpr (kPF == 1) issue_ine(s_sgn);
    }
    load_desc(q, s_sgn);
  }
  if constexpr (kPF == 2) {
    __syncthreads();
    if (s_desc[5] < nsegs) {
#pragma unroll
      for (int r = 0; r < kCtaSegItems / kCtaThreads; ++r) {
        const uint32_t i = threadIdx.x * (kCtaSegItems / kCtaThreads) + r;
        if (i < s_desc[2]) cp_async16(&s_ine[i], irec + 2 * ((uint64_t)s_desc[1] + i));
      }
    }
    cp_async_commit();
  }
  while (true) {
    if (threadIdx.x == 0) {
      s_hits = 0;
      s_cold = 0;
    }
    __syncthreads();
    if (s_desc[5] >= nsegs) break;
    const uint32_t v = s_desc[0], i0 = s_desc[1], ni = s_desc[2];
    const uint32_t nb = s_desc[3], dv = s_desc[4];
    uint32_t qnext = 0;
    if (threadIdx.x == 0) {
      qnext = atomicAdd(queue, 1u);
      if (qnext < nsegs) s_sgn = segs[nsegs - 1 - qnext];
    }
    // (1a) hot members -> bitmap; s_cold = #members below h0 (sorted prefix)
    for (uint32_t j = threadIdx.x; j < dv; j += kCtaThreads) {
      const uint32_t x = col[nb + j];
      if (x >= h0) {
        atomicOr(&bm[(x - h0) >> 5], 1u << ((x - h0) & 31));
        if (j == 0 || col[nb + j - 1] < h0) s_cold = j;
      } else if (j + 1 == dv) {
        s_cold = dv;
      }
    }
    // (1b) stage items, compacted into hot / cold lists with chunk prefixes
    constexpr int kIPT = kCtaSegItems / kCtaThreads;  // items per thread
    static_assert(kCtaSegItems % kCtaThreads == 0, "segment items must be a multiple of the CTA size");
    uint4 it[kIPT];
    uint64_t mo[kIPT];
    uint32_t nh[kIPT], nc[kIPT];
    if constexpr (kPF == 1) {
      mbar_wait(&s_mbar, phase);  // this segment's in-edge records have landed
      phase ^= 1u;
    } else if constexpr (kPF == 2) {
      cp_async_wait_all();  // this thread's in-edge records (it copied them itself) have landed
    }
#pragma unroll
    for (int r = 0; r < kIPT; ++r) {
      const uint32_t i = threadIdx.x * kIPT + r;
      nh[r] = nc[r] = 0;
      it[r] = make_uint4(0, 0, 0, 0);
      mo[r] = 0;
      if (i < ni) {
        it[r] = kPF ? s_ine[i] : irec[2 * (uint64_t)(i0 + i)];
        if (kMasks && it[r].y > it[r].x) {
          const uint4 ax = irec[2 * (uint64_t)(i0 + i) + 1];
          mo[r] = ax.z | ((uint64_t)ax.w << 32);
        }
        nh[r] = it[r].y > it[r].x ? ((it[r].y + 7) >> 3) - (it[r].x >> 3) : 0u;
        nc[r] = it[r].w > it[r].z ? ((it[r].w + 3) >> 2) - (it[r].z >> 2) : 0u;
      }
    }
    // one block scan of the pair (list positions: hot count in the low 16
    // bits, cold in the high 16; chunk prefixes: hot in the low 32 bits, cold
    // in the high 32), two barriers
    uint32_t lp = 0;
    unsigned long long cp = 0;
#pragma unroll
    for (int r = 0; r < kIPT; ++r) {
      lp += (uint32_t)(nh[r] > 0) | ((uint32_t)(nc[r] > 0) << 16);
      cp += (unsigned long long)nh[r] | ((unsigned long long)nc[r] << 32);
    }
    {
      const uint32_t il = warp_inclusive_scan(lp);
      const unsigned long long ic = warp_inclusive_scan(cp);
      if (lane == 31) {
        s_wl[warp] = il;
        s_wc[warp] = ic;
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t xl = lane < kCtaWarps ? s_wl[lane] : 0u;
        const unsigned long long xc = lane < kCtaWarps ? s_wc[lane] : 0ull;
        const uint32_t yl = warp_inclusive_scan(xl);
        const unsigned long long yc = warp_inclusive_scan(xc);
        if (lane < kCtaWarps) {
          s_wl[lane] = yl - xl;
          s_wc[lane] = yc - xc;
        }
        if (lane == kCtaWarps - 1) {
          s_nl = yl;
          s_ctot = yc;
        }
      }
      __syncthreads();
      // every thread is past its s_ine reads: start the next segment's copy
      if constexpr (kPF == 1) {
        if (threadIdx.x == 0 && qnext < nsegs) {
          fence_proxy_async_smem();
          issue_ine(s_sgn);
        }
      } else if constexpr (kPF == 2) {
        // each thread prefetches the next segment's records it will stage
        // (LDGSTS into its own s_ine slots; s_sgn is stale when the queue is
        // drained, and then never consumed)
        const uint4 nx = s_sgn;
#pragma unroll
        for (int r = 0; r < kIPT; ++r) {
          const uint32_t i = threadIdx.x * kIPT + r;
          if (i < nx.z - nx.y) cp_async16(&s_ine[i], irec + 2 * ((uint64_t)nx.y + i));
        }
        cp_async_commit();
      }
      lp = il - lp + s_wl[warp];
      cp = ic - cp + s_wc[warp];
      // s_wl/s_wc are rewritten only after the staging barrier below
    }
    {
      uint32_t ph = lp & 0xffffu, pc = lp >> 16;
      uint32_t ch = (uint32_t)cp, cc = (uint32_t)(cp >> 32);
#pragma unroll
      for (int r = 0; r < kIPT; ++r) {
        const uint32_t i = threadIdx.x * kIPT + r;
        if (nh[r]) {
          s_hb[ph] = it[r].x;
          s_he[ph] = it[r].y;
          s_hpre[ph] = ch;
          if (kMasks) s_hmo[ph] = mo[r];
          if (kHits) s_hidx[ph] = (uint16_t)i;
          ++ph;
          ch += nh[r];
        }
        if (nc[r]) {
          s_cb[pc] = it[r].z;
          s_ce[pc] = it[r].w;
          s_cpre[pc] = cc;
          if (kPerVertex) s_cidx[pc] = (uint16_t)i;
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
      tshift = __clz(ts) + 1;  // 32 - log2(ts), ts a power of two
      tab = ts <= stab_slots ? stab : gtab;
      for (uint32_t j = threadIdx.x; j < cold; j += kCtaThreads) {
        const uint32_t x = col[nb + j];
        hash_insert(tab, tmask, tshift, x);
        const uint32_t f = cfilt_bit(x);
        atomicOr(&s_cf[f >> 5], 1u << (f & 31));
      }
      if (tab == gtab) __threadfence_block();
    }
    __syncthreads();
    // (2) advance + join: hot chunks, then cold chunks, evenly split
    uint32_t h = 0;
    uint32_t* icnt = kPerVertex ? s_icnt : nullptr;
    if (!(g_pv_dbg & 4)) {
      const uint32_t fb = (uint32_t)(((uint64_t)tchunks_h * warp) / kCtaWarps);
      const uint32_t fe = (uint32_t)(((uint64_t)tchunks_h * (warp + 1)) / kCtaWarps);
      // per-vertex: the hot chunk's 8-bit hit mask goes to HBM (one byte store,
      // coalesced across the lanes of an item); k_pv_rows turns the masks into
      // t[u] and t[x] row by row, with no per-hit atomics
      h += warp_walk<8, kHotWin>(fb, fe, nhot, s_hpre, s_hb, s_he, kHits ? s_hidx : nullptr,
                                 kHits ? icnt : nullptr, colH,
                                 [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e, uint32_t k) {
                                   const uint32_t m = hot_hit_mask(qq, c, b, e, bm);
                                   if (kMasks) st_mask(masks + s_hmo[k] + (c - (b >> 3)), m);
                                   if (kHits && m) {
#pragma unroll
                                     for (int j = 0; j < 8; ++j)
                                       if ((m >> j) & 1u) hsink.hit(h0 + hot_u16(qq, j));
                                   }
                                   return (uint32_t)__popc(m);
                                 });
    }
    if (ncold && cold && !(g_pv_dbg & 4)) {  // a pivot with no cold members: no cold candidate can hit
      const uint32_t fb = (uint32_t)(((uint64_t)tchunks_c * warp) / kCtaWarps);
      const uint32_t fe = (uint32_t)(((uint64_t)tchunks_c * (warp + 1)) / kCtaWarps);
      if (tab == stab)  // SMEM table (LDS probes); the global slab only for huge pivots
        h += warp_walk<4, 2>(fb, fe, ncold, s_cpre, s_cb, s_ce, s_cidx, icnt, col,
                             [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e, uint32_t) {
                               return probe_cold<kPerVertex>(qq, c, b, e, stab, tmask, tshift, sink, s_cf);
                             });
      else
        h += warp_walk<4, 2>(fb, fe, ncold, s_cpre, s_cb, s_ce, s_cidx, icnt, col,
                             [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e, uint32_t) {
                               return probe_cold<kPerVertex>(qq, c, b, e, gtab, tmask, tshift, sink, s_cf);
                             });
    }
#if TCB_L2PF
    // TMA bulk prefetch into L2 of the next segment's item suffixes (hot part
    // in colH; with TCB_L2PF=2 also the cold part in col): they stream in
    // under this segment's barrier tail and the next segment's staging, so
    // its walk's chunk loads hit L2.  (s_sgn is stale once the queue is
    // drained: the prefetch is then merely useless.)
    {
      const uint4 nx = s_sgn;
#pragma unroll
      for (int r = 0; r < kIPT; ++r) {
        const uint32_t i = threadIdx.x * kIPT + r;
        if (i < nx.z - nx.y) {
          const uint4 g4 = irec[2 * (uint64_t)(nx.y + i)];
          if (g4.y > g4.x) prefetch_range_l2(colH + g4.x, 2ull * (g4.y - g4.x));
          if (TCB_L2PF >= 2 && g4.w > g4.z) prefetch_range_l2(col + g4.z, 4ull * (g4.w - g4.z));
        }
      }
    }
#endif
    acc += h;
    if (kPerVertex) {
      const uint32_t hw = warp_sum(h);
      if (lane == 0 && hw) atomicAdd(&s_hits, hw);
    }
    __syncthreads();
    // (3) clear + per-vertex flush
    // clear the bitmap: whole words by 16-byte stores when the pivot has many
    // hot members (no global re-read), else the touched words
    if (dv - cold > nbm / 8) {
      uint4* bm4 = reinterpret_cast<uint4*>(bm);
      for (uint32_t i = threadIdx.x; i < nbm / 4; i += kCtaThreads) bm4[i] = make_uint4(0, 0, 0, 0);
      for (uint32_t i = (nbm & ~3u) + threadIdx.x; i < nbm; i += kCtaThreads) bm[i] = 0;
    } else {
      for (uint32_t j = cold + threadIdx.x; j < dv; j += kCtaThreads) bm[(col[nb + j] - h0) >> 5] = 0;
    }
    for (uint32_t j = threadIdx.x; j < ts; j += kCtaThreads) tab[j] = kEmpty;
    if (cold)
      for (uint32_t j = threadIdx.x; j < kColdFilterWords; j += kCtaThreads) s_cf[j] = 0;
    if (kPerVertex) {
      for (uint32_t i = threadIdx.x; i < ni; i += kCtaThreads) {
        const uint32_t c = s_icnt[i];
        if (c) {
          atomicAdd(&t_rank[irec[2 * (uint64_t)(i0 + i) + 1].y], (unsigned long long)c);
          s_icnt[i] = 0;
        }
      }
      if (threadIdx.x == 0 && s_hits) atomicAdd(&t_rank[v], (unsigned long long)s_hits);
    }
    if (ts && tab == gtab) __threadfence_block();
    __syncthreads();  // everyone is done with s_desc of this segment
    if (threadIdx.x == 0) load_desc(qnext, s_sgn);
    if (kHits && ++segs_since_flush == kTopFlushSegs) {  // before any 16-bit half could wrap
      flush_top<true>(top, ncnt, rc, t_rank);
      segs_since_flush = 0;
    }
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
  if (kHits) {
    __syncthreads();
    flush_top<true>(top, ncnt, rc, t_rank);
  }
}

// ---- small CTA-bin pivots: one warp each -------------------------------------
// Pivots with d+ > kWarpMaxDeg but at most kSmallItems in-edge items and
// kSmallCold members below the hot window (frontier.cu PivotClass 2).  The
// same staging and walks as k_join_cta, at warp granularity: a warp-private
// hot bitmap and 256-slot cold hash, warp scans instead of block scans, and
// no block barriers -- these pivots are 60% of the CTA-bin segments at RMAT
// s24 but carry 2% of the wedges, so the CTA path's per-segment barriers and
// latency chain dominated them.
// two warps per CTA: the per-warp SMEM (hot bitmap + tables, ~12 KB) bounds
// residency, and 2-warp CTAs pack 18 warps per SM instead of 16 (C4 small bin
// 1.05 -> 0.97 ms, C3 0.57 -> 0.52 ms; 1 warp: 0.99 / 0.53)
#ifndef TCB_SMALL_THREADS
#define TCB_SMALL_THREADS 64
#endif
constexpr int kSmallThreads = TCB_SMALL_THREADS;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr uint32_t kSmallTable = 2 * kSmallCold;
constexpr int kSmallR = kSmallItems / 32;  // items per lane
// small bin: the next pivot's descriptor loaded one pivot ahead (C4 small
// bin 1.021 -> 1.000 ms total-only, 1.069 -> 1.039 ms per-vertex)
#ifndef TCB_SMALL_PIPE
#define TCB_SMALL_PIPE 1
#endif

struct SmallWarpSmem {
  uint32_t* bm;
  uint32_t* tab;
  uint32_t* cf;  // cold-member prefilter
  uint32_t *hb, *he, *hpre, *cb, *ce, *cpre, *icnt;
  uint16_t *hidx, *cidx;
  unsigned long long* hmo;
  __host__ __device__ static uint32_t bytes(uint32_t nbm) {
    const uint32_t nb4 = (nbm + 3) & ~3u;
    // hmo u64[64] | bm[nb4] | tab[256] | hb, he, cb, ce, icnt [64 each] | hpre, cpre [65] | hidx, cidx u16[64]
    return kSmallItems * 8 + (nb4 + kSmallTable) * 4 + (kSmallItems * 5 + (kSmallItems + 1) * 2) * 4 +
           kSmallItems * 2 * 2 + kColdFilterWords * 4 + 16;
  }
  __device__ SmallWarpSmem(uint8_t* base, uint32_t nbm) {
    const uint32_t nb4 = (nbm + 3) & ~3u;
    hmo = reinterpret_cast<unsigned long long*>(base);
    bm = reinterpret_cast<uint32_t*>(base + kSmallItems * 8);
    tab = bm + nb4;
    hb = tab + kSmallTable;
    he = hb + kSmallItems;
    cb = he + kSmallItems;
    ce = cb + kSmallItems;
    icnt = ce + kSmallItems;
    hpre = icnt + kSmallItems;
    cpre = hpre + kSmallItems + 1;
    cf = cpre + kSmallItems + 1;
    hidx = reinterpret_cast<uint16_t*>(cf + kColdFilterWords);
    cidx = hidx + kSmallItems;
  }
};

template <bool kPerVertex>
__global__ void __launch_bounds__(kSmallThreads) k_join_small(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint4* __restrict__ rowd, uint32_t r0,
    const uint16_t* __restrict__ colH, const uint4* __restrict__ irec,
    const uint4* __restrict__ segs, const uint32_t* __restrict__ nsegs_p, unsigned int* __restrict__ queue,
    uint32_t h0, uint32_t nbm, uint8_t* __restrict__ masks, uint32_t rc, uint32_t ncnt,
    unsigned long long* __restrict__ t_rank, unsigned long long* __restrict__ total) {
  extern __shared__ __align__(16) uint8_t dsm_small[];
  constexpr bool kMasks = kPerVertex && TCB_PV_MASKS;
  constexpr bool kHits = kPerVertex && !TCB_PV_MASKS;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t nsegs = *nsegs_p;
  const ItemGeo geo{rowd, r0};
  const uint32_t wbytes = (SmallWarpSmem::bytes(nbm) + 15) & ~15u;
  SmallWarpSmem w(dsm_small + warp * wbytes, nbm);
  // kHits: CTA-shared 32-bit counters for ranks [rc, rc + ncnt), after the warps' regions
  uint32_t* top = reinterpret_cast<uint32_t*>(dsm_small + kSmallWarps * wbytes);
  if (kHits) {
    for (uint32_t i = threadIdx.x; i < ncnt; i += kSmallThreads) top[i] = 0;
    __syncthreads();
  }
  const PvSink<false> hsink{top, rc, t_rank, 0};
  for (uint32_t i = lane; i < nbm; i += 32) w.bm[i] = 0;
  for (uint32_t i = lane; i < kSmallTable; i += 32) w.tab[i] = kEmpty;
  for (uint32_t i = lane; i < kSmallItems; i += 32) w.icnt[i] = 0;
  for (uint32_t i = lane; i < kColdFilterWords; i += 32) w.cf[i] = 0;
  __syncwarp();
  const uint32_t tmask = kSmallTable - 1, tshift = __clz(kSmallTable) + 1;  // 32 - log2(kSmallTable)
  const PvSink<true> sink{nullptr, 0xffffffffu, t_rank, 0};
  unsigned long long acc = 0;
#if TCB_SMALL_PIPE
  // the next pivot's queue slot, descriptor and row bounds are loaded under
  // the current pivot's work (its dependent global round trips leave the
  // per-pivot chain), and its records and row are prefetched into L2
  uint32_t qc = 0;
  if (lane == 0) qc = atomicAdd(queue, 1u);
  qc = __shfl_sync(0xffffffffu, qc, 0);
  uint4 sgc = qc < nsegs ? segs[qc] : make_uint4(0, 0, 0, 0);
  uint32_t nbc = 0, dvc = 0;
  if (qc < nsegs) {
    nbc = off[sgc.x];
    dvc = off[sgc.x + 1] - nbc;
  }
  while (qc < nsegs) {
    const uint4 sg = sgc;
    const uint32_t nb = nbc, dv = dvc;
    uint32_t qn = 0;
    if (lane == 0) qn = atomicAdd(queue, 1u);
    qn = __shfl_sync(0xffffffffu, qn, 0);
    const uint4 sgn = qn < nsegs ? segs[qn] : make_uint4(0, 0, 0, 0);
#else
  while (true) {
    uint32_t q = 0;
    if (lane == 0) q = atomicAdd(queue, 1u);
    q = __shfl_sync(0xffffffffu, q, 0);
    if (q >= nsegs) break;
    const uint4 sg = segs[q];
    const uint32_t nb = off[sg.x], dv = off[sg.x + 1] - nb;
#endif
    const uint32_t v = sg.x, i0 = sg.y, ni = sg.z - sg.y;
    // (1) members: hot -> bitmap, count the sorted cold prefix
    uint32_t cold = 0;
    for (uint32_t j0 = 0; j0 < dv; j0 += 32) {
      const uint32_t j = j0 + lane;
      const uint32_t x = j < dv ? col[nb + j] : 0xffffffffu;
      if (j < dv && x >= h0) atomicOr(&w.bm[(x - h0) >> 5], 1u << ((x - h0) & 31));
      cold += __popc(__ballot_sync(0xffffffffu, j < dv && x < h0));
    }
#if TCB_SMALL_PIPE
    if (qn < nsegs) {
      nbc = off[sgn.x];
      dvc = off[sgn.x + 1] - nbc;
      if (lane < sgn.z - sgn.y) prefetch_l2(irec + 2 * ((uint64_t)sgn.y + lane));
    }
#endif
    for (uint32_t j = lane; j < cold; j += 32) {
      const uint32_t x = col[nb + j];
      hash_insert(w.tab, tmask, tshift, x);
      const uint32_t f = cfilt_bit(x);
      atomicOr(&w.cf[f >> 5], 1u << (f & 31));
    }
    // (2) items (<= kSmallItems, kSmallR per lane) -> hot / cold lists with chunk prefixes
    uint4 it[kSmallR];
    uint64_t mo[kSmallR];
    uint32_t nh[kSmallR], nc[kSmallR];
#pragma unroll
    for (int r = 0; r < kSmallR; ++r) {
      const uint32_t i = lane + 32 * r;
      nh[r] = nc[r] = 0;
      it[r] = make_uint4(0, 0, 0, 0);
      mo[r] = 0;
      if (i < ni) {
        it[r] = ld_stream(irec + 2 * (uint64_t)(i0 + i));
        if (kPerVertex && it[r].y > it[r].x) {
          const uint4 ax = ld_stream(irec + 2 * (uint64_t)(i0 + i) + 1);
          mo[r] = ax.z | ((uint64_t)ax.w << 32);
        }
        nh[r] = it[r].y > it[r].x ? ((it[r].y + 7) >> 3) - (it[r].x >> 3) : 0u;
        nc[r] = it[r].w > it[r].z ? ((it[r].w + 3) >> 2) - (it[r].z >> 2) : 0u;
      }
    }
    uint32_t ph = 0, pc = 0, ch = 0, cc = 0, nhot = 0, ncold = 0, th = 0, tcc = 0;
#pragma unroll
    for (int r = 0; r < kSmallR; ++r) {  // item lane + 32r: positions after all of round r-1
      const uint32_t hf = nh[r] > 0, cf = nc[r] > 0;
      const uint32_t iph = warp_inclusive_scan(hf), ipc = warp_inclusive_scan(cf);
      const uint32_t ich = warp_inclusive_scan(nh[r]), icc = warp_inclusive_scan(nc[r]);
      const uint32_t i = lane + 32 * r;
      ph = nhot + iph - hf;
      pc = ncold + ipc - cf;
      ch = th + ich - nh[r];
      cc = tcc + icc - nc[r];
      if (hf) {
        w.hb[ph] = it[r].x;
        w.he[ph] = it[r].y;
        w.hpre[ph] = ch;
        w.hidx[ph] = (uint16_t)i;
        if (kMasks) w.hmo[ph] = mo[r];
      }
      if (cf) {
        w.cb[pc] = it[r].z;
        w.ce[pc] = it[r].w;
        w.cpre[pc] = cc;
        w.cidx[pc] = (uint16_t)i;
      }
      nhot += __shfl_sync(0xffffffffu, iph, 31);
      ncold += __shfl_sync(0xffffffffu, ipc, 31);
      th += __shfl_sync(0xffffffffu, ich, 31);
      tcc += __shfl_sync(0xffffffffu, icc, 31);
    }
    if (lane == 0) {
      w.hpre[nhot] = th;
      w.cpre[ncold] = tcc;
    }
    __syncwarp();
    // (3) advance + join
    uint32_t h = warp_walk<8, kHotWin>(0, th, nhot, w.hpre, w.hb, w.he, w.hidx, kHits ? w.icnt : nullptr, colH,
                                       [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e, uint32_t k) {
                                         const uint32_t m = hot_hit_mask(qq, c, b, e, w.bm);
                                         if (kMasks) st_mask(masks + w.hmo[k] + (c - (b >> 3)), m);
                                         if (kHits && m) {
#pragma unroll
                                           for (int j = 0; j < 8; ++j)
                                             if ((m >> j) & 1u) hsink.hit(h0 + hot_u16(qq, j));
                                         }
                                         return (uint32_t)__popc(m);
                                       });
    if (ncold && cold)  // a pivot with no cold members: no cold candidate can hit
      h += warp_walk<4, 2>(0, tcc, ncold, w.cpre, w.cb, w.ce, w.cidx, kPerVertex ? w.icnt : nullptr, col,
                           [&](const uint4& qq, uint32_t c, uint32_t b, uint32_t e, uint32_t) {
                             return probe_cold<kPerVertex>(qq, c, b, e, w.tab, tmask, tshift, sink, w.cf);
                           });
    acc += h;
    __syncwarp();
    if (kPerVertex) {
      const uint32_t hw = warp_sum(h);
      if (lane == 0 && hw) atomicAdd(&t_rank[v], (unsigned long long)hw);
      for (uint32_t i = lane; i < ni; i += 32) {
        const uint32_t c = w.icnt[i];
        if (c) {
          atomicAdd(&t_rank[irec[2 * (uint64_t)(i0 + i) + 1].y], (unsigned long long)c);
          w.icnt[i] = 0;
        }
      }
    }
    // (4) clear the touched bitmap words and table slots
    for (uint32_t j = cold + lane; j < dv; j += 32) w.bm[(col[nb + j] - h0) >> 5] = 0;
    if (cold) {
      for (uint32_t i = lane; i < kSmallTable; i += 32) w.tab[i] = kEmpty;
      for (uint32_t i = lane; i < kColdFilterWords; i += 32) w.cf[i] = 0;
    }
    __syncwarp();
#if TCB_SMALL_PIPE
    qc = qn;
    sgc = sgn;
#endif
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
  if (kHits) {
    __syncthreads();
    flush_top<false>(top, ncnt, rc, t_rank);
  }
}

// Per-vertex counts from the CTA bin's hot hit masks.
// Mask byte (item k, chunk c) has bit j set iff element 8c+j of colH -- an
// oriented edge u->x -- closed a triangle (u, v_k, x).  For each hot position
// p of row u, B[p] = sum over u's items of that bit = the triangles whose
// low->top edge is u->x_p; then t[x_p] += B[p] and t[u] += sum_p B[p].
// The row's mask block has the closed-form layout of graph.cuh RowMasks
// (item k's bytes at rowbase + P(k), chunks cs_k..c_hi-1), so the pass needs
// no per-item metadata.  Lanes own consecutive chunks of the row (groups of
// 32; narrow rows with C <= 16 chunks split the warp into sub-groups of
// w = pow2 >= C lanes that take different items), the warp walks the items
// that reach the group (one item's bytes are coalesced across the lanes),
// kRowU items in flight, and each byte is spread into 4+4 byte-lane counters
// by a multiply (b*0x00204081 & 0x01010101).  Warp-bin items' bytes are zero
// (memset): their hits are counted in k_join_warp.
//   k_pv_rows        one warp per light row, 32 rows per queue grab (top rank
//                    down); rows with more than row_heavy_threshold item-steps are
//                    appended to a list instead
//   k_pv_rows_heavy  one CTA per listed row, its 8 warps splitting each
//                    group's items, partial counters reduced in SMEM
constexpr int kRowWarps = 8;
#ifndef TCB_ROWU_LIGHT
#define TCB_ROWU_LIGHT 8
#endif
constexpr int kRowULight = TCB_ROWU_LIGHT;  // light rows: a warp each, many warps per SM
constexpr int kRowUHeavy = 16;  // heavy rows: latency-bound on the byte loads (A/B: profiles/README.md)
#ifndef TCB_TINY_ITEMS
#define TCB_TINY_ITEMS 64
#endif
constexpr uint32_t kTinyItems = TCB_TINY_ITEMS;  // rows of few items and chunks folded lane by lane (<= 255)
// ... of at most kTC mask chunks: 4 for a whole count, 8 for a split part
// (whose rows hold fewer items each).  Measured at C4 (profiles/README.md):
// rows 5.8 -> 5.0 ms whole, 8-part maximum 7.73 -> 6.82 ms.
// Rows with more item-steps than the threshold go to the CTA-per-row kernel.
// With many rows the warp-per-row kernel balances rows of up to 2048 steps
// and runs them faster (C4 whole count: 128 -> 2048 takes the row pass from
// 11.5 to 9.9 ms; 4096 overloads single warps); a multi-GPU part holding few,
// long rows (the top ranks) needs the CTA kernel sooner.  Threshold =
// rows / 8192 clamped to [kRowHeavyMin, kRowHeavyMax].
#ifndef TCB_ROW_HEAVY
#define TCB_ROW_HEAVY 2048
#endif
constexpr uint32_t kRowHeavyMax = TCB_ROW_HEAVY;
constexpr uint32_t kRowHeavyMin = 128;
__host__ __device__ __forceinline__ uint32_t row_heavy_threshold(uint64_t rows) {
  const uint64_t t = rows / 8192;
  return (uint32_t)(t < kRowHeavyMin ? kRowHeavyMin : t > kRowHeavyMax ? kRowHeavyMax : t);
}

struct RowLanes {
  uint32_t w, G, sub;  // lanes per sub-group, sub-groups, this lane's sub-group
  __device__ __forceinline__ RowLanes(uint32_t C, unsigned lane) {
    if (C > 16) {
      w = 32;
    } else {
      const uint32_t lg = 32 - __clz(C - 1);
      w = C > 1 ? 1u << lg : 1u;
    }
    G = 32 / w;
    sub = lane / w;
  }
};

// Row geometry relative to the row's first chunk c_lo (32-bit): item k's
// first chunk is csr_k = (o7 + max(k+1-c0, 0)) >> 3, it owns C - csr_k mask
// bytes, P(k) = bytes of the items before it.
struct RowRel {
  uint32_t o7, c0, C, nk;
  __device__ __forceinline__ explicit RowRel(const RowMasks& rm)
      : o7((uint32_t)(rm.O & 7)), c0(rm.c0), C((uint32_t)(rm.c_hi - rm.c_lo)), nk(rm.d - 1) {}
  __device__ __forceinline__ uint32_t csr(uint32_t k) const {
    const int sk = max((int)(k + 1 - c0), 0);
    return (o7 + (uint32_t)sk) >> 3;
  }
  __device__ static __forceinline__ uint32_t F(uint32_t x) {  // sum_{t < x} floor(t/8)
    const uint32_t q = x >> 3, r = x & 7;
    return 4 * q * (q ? q - 1 : 0) + r * q;
  }
  __device__ __forceinline__ uint32_t P(uint32_t k) const {
    if (k <= c0) return k * C;
    const uint32_t S = k - c0;
    return c0 * C + S * C - (F(o7 + S + 1) - F(o7 + 1));
  }
  // items reaching relative chunk group [g, g+span): all k < c0, and k >= c0
  // while csr_k <= the group's last chunk
  __device__ __forceinline__ uint32_t reaching(uint32_t g, uint32_t span) const {
    const uint32_t last = min(g + span, C) - 1;
    const uint32_t kk = 8 * last + 7 - o7 + c0;  // first k with csr_k > last
    return min(kk, nk);
  }
};

// byte b -> its 8 bits spread over 8 byte lanes (x: bits 0-3, y: bits 4-7)
__device__ __forceinline__ void init_spread(uint2* s_spread) {
  for (uint32_t b = threadIdx.x; b < 256; b += blockDim.x)
    s_spread[b] = make_uint2(((b & 0xfu) * 0x00204081u) & 0x01010101u, ((b >> 4) * 0x00204081u) & 0x01010101u);
}

// cnt[j] += bit j of byte (k, cr) over items k = ka + sub + G*i in [ka, kb);
// kRowU mask-byte loads in flight per lane.
template <int kRowU>
__device__ __forceinline__ void row_accumulate(const RowRel& rr, const uint8_t* __restrict__ rowm, uint32_t cr,
                                               bool cvalid, const RowLanes& rl, uint32_t ka, uint32_t kb,
                                               const uint2* s_spread, uint32_t (&cnt)[8]) {
  uint32_t acc_lo = 0, acc_hi = 0, nacc = 0;
  auto fold = [&]() {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cnt[j] += (acc_lo >> (8 * j)) & 0xffu;
      cnt[4 + j] += (acc_hi >> (8 * j)) & 0xffu;
    }
    acc_lo = acc_hi = nacc = 0;
  };
  auto add = [&](uint32_t b) {
    const uint2 sp = s_spread[b];
    acc_lo += sp.x;
    acc_hi += sp.y;
  };
  if (rl.G == 1) {
    // items before c0 start at the row's first chunk: P(k) = k*C
    const uint32_t kbA = min(kb, rr.c0);
    uint32_t P = ka * rr.C + cr;
    for (uint32_t k0 = ka; k0 < kbA; k0 += kRowU) {
      uint32_t bits[kRowU];
#pragma unroll
      for (int t = 0; t < kRowU; ++t) {
        bits[t] = (k0 + t < kbA && cvalid) ? rowm[P] : 0u;
        P += rr.C;
      }
      if (nacc + kRowU > 255) fold();
#pragma unroll
      for (int t = 0; t < kRowU; ++t) add(bits[t]);
      nacc += kRowU;
    }
    // items k >= c0: the first chunk cs_k = (o7 + k + 1 - c0) >> 3 steps every
    // 8 items, so within an aligned block of 8 items the byte addresses are
    // an arithmetic sequence (stride C - cs) under one predicate
    const uint32_t kaB = max(ka, rr.c0);
    uint32_t PB = rr.P(kaB);
    uint32_t k0 = kaB;
    for (; k0 < kb && ((rr.o7 + k0 + 1 - rr.c0) & 7); ++k0) {  // head up to a block boundary
      const uint32_t cs = (rr.o7 + (k0 + 1 - rr.c0)) >> 3;
      const uint32_t b = (cvalid && cr >= cs) ? rowm[PB + cr - cs] : 0u;
      PB += rr.C - cs;
      if (nacc + 1 > 255) fold();
      add(b);
      ++nacc;
    }
    for (; k0 < kb; k0 += 8) {
      const uint32_t cs = (rr.o7 + (k0 + 1 - rr.c0)) >> 3;  // same for k0..k0+7
      const uint32_t stride = rr.C - cs;
      const bool ok = cvalid && cr >= cs;
      const uint32_t a0 = PB + cr - cs;
      uint32_t bits[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) bits[t] = (ok && k0 + t < kb) ? rowm[a0 + t * stride] : 0u;
      PB += 8 * stride;
      if (nacc + 8 > 255) fold();
#pragma unroll
      for (int t = 0; t < 8; ++t) add(bits[t]);
      nacc += 8;
    }
  } else {
    // sub-group `sub` takes a contiguous run of the items; item k's first
    // chunk cs and its block offset P advance incrementally (P(k+1) = P(k) +
    // C - cs_k), so no closed-form offset per item
    const uint32_t per = (kb - ka + rl.G - 1) / rl.G;
    const uint32_t k_lo = min(kb, ka + rl.sub * per), k_hi = min(kb, k_lo + per);
    uint32_t P = k_lo < k_hi ? rr.P(k_lo) : 0u;
    for (uint32_t k0 = k_lo; k0 < k_hi; k0 += kRowU) {
      uint32_t bits[kRowU];
#pragma unroll
      for (int t = 0; t < kRowU; ++t) {
        const uint32_t k = k0 + t;
        const uint32_t cs = rr.csr(k);
        bits[t] = (k < k_hi && cvalid && cr >= cs) ? rowm[P + cr - cs] : 0u;
        P += rr.C - cs;
      }
      if (nacc + kRowU > 255) fold();
#pragma unroll
      for (int t = 0; t < kRowU; ++t) add(bits[t]);
      nacc += kRowU;
    }
  }
  fold();
}

// t[x_p] += cnt for position j of chunk c (global); returns the count added.
// t[x_p] += cnt for position j of the row's relative chunk cr (p = 8*cr + j
// relative to the row's first chunk; the row's hot ids sit at [o7, o7 + h)).
__device__ __forceinline__ uint32_t row_emit1(const RowRel& rr, uint32_t h, const uint4& q, uint32_t cr, int j,
                                              uint32_t cnt, uint32_t h0, uint32_t rc, uint32_t* top,
                                              unsigned long long* __restrict__ t_rank) {
  const uint32_t p = 8 * cr + j;
  if (!cnt || p < rr.o7 || p >= rr.o7 + h) return 0;
  const uint32_t x = h0 + hot_u16(q, j);
  if (x >= rc) atomicAdd(&top[x - rc], cnt);
  else atomicAdd(&t_rank[x], (unsigned long long)cnt);
  return cnt;
}

__device__ __forceinline__ void flush_top_rows(const uint32_t* top, uint32_t ncnt, uint32_t rc,
                                               unsigned long long* __restrict__ t_rank) {
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x)
    if (top[i]) atomicAdd(&t_rank[rc + i], (unsigned long long)top[i]);
}

// Items of row u whose pivot lies in the part's rank range [v_lo, v_hi): a
// contiguous range [k_lo, k_hi) of N+(u) (rows are sorted); the whole row
// when the count is not split.
struct PartRange {
  const uint32_t* col;
  uint32_t v_lo, v_hi;
  bool split;
  uint32_t r0;  // rows [r0, n) (rowbase[u - r0])
  __device__ static __forceinline__ uint32_t lb(const uint32_t* a, uint32_t b, uint32_t e, uint32_t key) {
    while (b < e) {
      const uint32_t m = b + ((e - b) >> 1);  // edge indices: b + e may pass 2^32
      if (a[m] < key) b = m + 1; else e = m;
    }
    return b;
  }
  const uint2* krange;  // split counts: cached {k_lo, k_hi} per row (k_part_krange), else null
  __device__ __forceinline__ void items(uint32_t u, uint32_t beg, uint32_t d, uint32_t& k_lo, uint32_t& k_hi) const {
    k_lo = 0;
    k_hi = d ? d - 1 : 0;  // item d-1 has an empty suffix (no mask bytes)
    if (!split || d == 0) return;
    if (krange) {
      const uint2 kr = krange[u - r0];
      k_lo = kr.x;
      k_hi = min(k_hi, kr.y);
      return;
    }
    if (v_lo) k_lo = lb(col, beg, beg + d, v_lo) - beg;
    if (v_hi != 0xffffffffu) k_hi = min(k_hi, lb(col, beg + k_lo, beg + d, v_hi) - beg);
  }
};

// The item range of every row for one part (graph + split property, cached
// on the handle by count_triangles): rows scanned once per (P, part) instead
// of two binary searches per row in every count's row pass.
__global__ void k_part_krange(PartRange pr, const uint32_t* __restrict__ off, uint32_t n, uint2* __restrict__ out) {
  for (uint64_t u = pr.r0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t beg = off[u], d = off[u + 1] - beg;
    uint32_t k_lo = 0, k_hi = 0;
    if (d) {
      k_hi = d - 1;
      if (pr.v_lo) k_lo = PartRange::lb(pr.col, beg, beg + d, pr.v_lo) - beg;
      if (pr.v_hi != 0xffffffffu) k_hi = min(k_hi, PartRange::lb(pr.col, beg + k_lo, beg + d, pr.v_hi) - beg);
    }
    out[u - pr.r0] = make_uint2(k_lo, k_hi);
  }
}

// Tiny row (<= kC mask chunks, <= kTinyItems items in the part): one lane
// folds it alone, no warp-serial row step.  Item k owns the row's relative
// chunks csr_k .. C-1 at P(k) (RowRel); every chunk counter takes <=
// kTinyItems byte adds, so the byte lanes cannot overflow.
template <int kC>
__device__ __forceinline__ void tiny_row(const RowMasks& rm, const uint8_t* __restrict__ rowm, uint32_t kl,
                                         uint32_t kh, const uint2* s_spread, const uint4* __restrict__ colH4,
                                         uint32_t h0, uint32_t rc, uint32_t* top,
                                         unsigned long long* __restrict__ t_rank, uint32_t ul) {
  const RowRel rr(rm);
  uint32_t lo[kC], hi[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) lo[c] = hi[c] = 0;
  uint32_t P = rr.P(kl);
  for (uint32_t k = kl; k < kh; ++k) {
    const uint32_t cs = kC == 1 ? 0u : rr.csr(k);
#pragma unroll
    for (int c = 0; c < kC; ++c) {
      if ((uint32_t)c >= cs && (uint32_t)c < rr.C) {
        const uint2 sp = s_spread[rowm[P + c - cs]];
        lo[c] += sp.x;
        hi[c] += sp.y;
      }
    }
    P += rr.C - cs;
  }
  uint32_t tot = 0;
#pragma unroll
  for (int c = 0; c < kC; ++c) {
    if ((uint32_t)c >= rr.C || !(lo[c] | hi[c])) continue;
    const uint4 q = colH4[rm.c_lo + c];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t cj = ((j < 4 ? lo[c] : hi[c]) >> (8 * (j & 3))) & 0xffu;
      const uint32_t p = 8 * c + j;
      if (cj && p >= rr.o7 && p < rr.o7 + rm.h) {
        const uint32_t x = h0 + hot_u16(q, j);
        if (x >= rc) atomicAdd(&top[x - rc], cj);
        else atomicAdd(&t_rank[x], (unsigned long long)cj);
        tot += cj;
      }
    }
  }
  if (tot) atomicAdd(&t_rank[ul], (unsigned long long)tot);
}

// Held to 64 registers for 4 CTAs per SM: the row pass is latency bound on
// the mask-byte loads and their table lookups (C4 whole count 5.16 -> 4.62 ms;
// 8-part sum 46.4 -> 45.5 ms).
template <int kTC>
__global__ void __launch_bounds__(kRowWarps * 32, 4) k_pv_rows(
    const uint4* __restrict__ rowd, const uint16_t* __restrict__ colH, const uint8_t* __restrict__ masks, uint32_t n,
    PartRange pr,
    uint32_t h0, uint32_t rc, uint32_t ncnt, unsigned long long* __restrict__ queue, uint32_t* __restrict__ heavy,
    unsigned int* __restrict__ nheavy, uint32_t heavy_thr, uint32_t row_first,
    unsigned long long* __restrict__ t_rank) {
  extern __shared__ uint32_t top[];  // 32-bit counters for ranks [rc, rc+ncnt)
  __shared__ uint2 s_spread[256];
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x) top[i] = 0;
  init_spread(s_spread);
  __syncthreads();
  const unsigned lane = lane_id();
  const uint32_t nrows = n - pr.r0;
  const uint4* colH4 = reinterpret_cast<const uint4*>(colH);
  while (true) {
    unsigned long long rb64 = 0;  // 64-bit queue: row counts may approach 2^32
    if (lane == 0) rb64 = atomicAdd(queue, 32ull) + row_first;
    rb64 = __shfl_sync(0xffffffffu, rb64, 0);
    if (rb64 >= nrows) break;
    const uint32_t rb = (uint32_t)rb64;  // from the part's first row with items (u < v_hi)
    const uint32_t i = rb + lane;
    uint32_t ul = 0, dl = 0, Ol = 0, hl = 0, kl = 0, kh = 0;
    uint64_t rbl = 0;
    bool work = false;
    if (i < nrows) {
      ul = n - 1 - i;
      const RowGeo r = load_row(rowd, pr.r0, ul);
      // the sparse hot part only (a dense row's core members are counted in
      // the joins' dense step)
      dl = r.d() - r.cc();
      Ol = r.O;
      hl = r.Ht - r.O;
      rbl = r.rowbase;
      work = hl > 0 && dl >= 2;
      if (work) pr.items(ul, r.beg, r.d(), kl, kh);
      kh = min(kh, dl - 1);
      work = work && kh > kl;
      if (work) {
        const RowMasks rm(dl, Ol, hl);
        const uint32_t C = (uint32_t)(rm.c_hi - rm.c_lo);
        if (C <= kTC && kh - kl <= kTinyItems) {
          tiny_row<kTC>(rm, masks + rbl, kl, kh, s_spread, colH4, h0, rc, top, t_rank, ul);
          work = false;
        } else {
          const uint32_t steps = C > 16 ? (dl - 1) * ((C + 31) / 32) : (dl - 1) / (32 / RowLanes(C, 0).w);
          if (steps > heavy_thr) {
            heavy[atomicAdd(nheavy, 1u)] = ul;
            work = false;
          }
        }
      }
    }
    uint32_t rows = __ballot_sync(0xffffffffu, work);
    while (rows) {
      const int rj = __ffs(rows) - 1;
      rows &= rows - 1;
      const uint32_t u = __shfl_sync(0xffffffffu, ul, rj);
      const uint32_t ka = __shfl_sync(0xffffffffu, kl, rj), kb = __shfl_sync(0xffffffffu, kh, rj);
      const RowMasks rm(__shfl_sync(0xffffffffu, dl, rj), __shfl_sync(0xffffffffu, Ol, rj),
                        __shfl_sync(0xffffffffu, hl, rj));
      const RowRel rr(rm);
      const uint8_t* rowm = masks + __shfl_sync(0xffffffffu, rbl, rj);
      const RowLanes rl(rr.C, lane);
      uint32_t row_total = 0;
      for (uint32_t g = 0; g < rr.C; g += rl.w) {
        const uint32_t cr = g + (lane & (rl.w - 1));
        const bool cvalid = cr < rr.C;
        uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const uint32_t reach = min(rr.reaching(g, rl.w), kb);
        row_accumulate<kRowULight>(rr, rowm, cr, cvalid, rl, min(ka, reach), reach, s_spread, cnt);
        if (rl.G > 1) {  // sum the sub-groups: counts < 2^16 here, two per word
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) pk[j] = cnt[2 * j] | (cnt[2 * j + 1] << 16);
#pragma unroll
          for (int j = 0; j < 4; ++j)
            for (uint32_t o = rl.w; o < 32; o <<= 1) pk[j] += __shfl_xor_sync(0xffffffffu, pk[j], o);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            cnt[2 * j] = pk[j] & 0xffffu;
            cnt[2 * j + 1] = pk[j] >> 16;
          }
        }
        if (rl.sub == 0 && cvalid) {
          const uint64_t c = rm.c_lo + cr;
          const uint4 q = colH4[c];
#pragma unroll
          for (int j = 0; j < 8; ++j) row_total += row_emit1(rr, rm.h, q, cr, j, cnt[j], h0, rc, top, t_rank);
        }
      }
      row_total = warp_sum(row_total);
      if (lane == 0 && row_total) atomicAdd(&t_rank[u], (unsigned long long)row_total);
    }
  }
  __syncthreads();
  flush_top_rows(top, ncnt, rc, t_rank);
}

// 4 CTAs per SM (64 registers): heavy rows 1.18 -> 0.67 ms at C4
#ifndef TCB_HEAVY_MINB
#define TCB_HEAVY_MINB 4
#endif
__global__ void __launch_bounds__(kRowWarps * 32, TCB_HEAVY_MINB) k_pv_rows_heavy(
    const uint4* __restrict__ rowd, const uint16_t* __restrict__ colH, const uint8_t* __restrict__ masks,
    PartRange pr, uint32_t h0,
    uint32_t rc, uint32_t ncnt, unsigned int* __restrict__ queue, const uint32_t* __restrict__ heavy,
    const unsigned int* __restrict__ nheavy, unsigned long long* __restrict__ t_rank) {
  extern __shared__ uint32_t top[];
  __shared__ uint32_t red[kRowWarps][8][32];
  __shared__ uint2 s_spread[256];
  __shared__ uint32_t s_row;
  for (uint32_t i = threadIdx.x; i < ncnt; i += blockDim.x) top[i] = 0;
  init_spread(s_spread);
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint4* colH4 = reinterpret_cast<const uint4*>(colH);
  const uint32_t nh = *nheavy;
  uint32_t my_total = 0;  // this warp's share of the current row's t[u]
  while (true) {
    __syncthreads();
    if (threadIdx.x == 0) s_row = atomicAdd(queue, 1u);
    __syncthreads();
    const uint32_t r = s_row;
    if (r >= nh) break;
    const uint32_t u = heavy[r];
    const RowGeo rg = load_row(rowd, pr.r0, u);
    uint32_t k_lo = 0, k_hi = 0;
    pr.items(u, rg.beg, rg.d(), k_lo, k_hi);
    const RowMasks rm = rg.masks();
    k_hi = min(k_hi, rm.d - 1);
    const RowRel rr(rm);
    const uint8_t* rowm = masks + rg.rowbase;
    const RowLanes rl(rr.C, lane);
    my_total = 0;
    for (uint32_t g = 0; g < rr.C; g += rl.w) {
      const uint32_t cr = g + (lane & (rl.w - 1));
      const bool cvalid = cr < rr.C;
      const uint32_t K = min(rr.reaching(g, rl.w), k_hi);
      const uint32_t K0 = min(k_lo, K);
      // this warp's slice of the items
      const uint32_t per = (K - K0 + kRowWarps - 1) / kRowWarps;
      const uint32_t ka = min(K, K0 + warp * per), kb = min(K, ka + per);
      uint32_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      row_accumulate<kRowUHeavy>(rr, rowm, cr, cvalid, rl, ka, kb, s_spread, cnt);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        for (uint32_t o = rl.w; o < 32; o <<= 1) cnt[j] += __shfl_xor_sync(0xffffffffu, cnt[j], o);
        red[warp][j][lane] = cnt[j];
      }
      __syncthreads();
      // warp w emits position j = w of every chunk of the group
      {
        uint32_t t = 0;
#pragma unroll
        for (int w2 = 0; w2 < kRowWarps; ++w2) t += red[w2][warp][lane];
        if (rl.sub == 0 && cvalid && t) {
          const uint64_t c = rm.c_lo + cr;
          my_total += row_emit1(rr, rm.h, colH4[c], cr, (int)warp, t, h0, rc, top, t_rank);
        }
      }
      __syncthreads();
    }
    my_total = warp_sum(my_total);
    if (lane == 0 && my_total) atomicAdd(&t_rank[u], (unsigned long long)my_total);
  }
  __syncthreads();
  flush_top_rows(top, ncnt, rc, t_rank);
}

__global__ void k_gather_pv(const unsigned long long* __restrict__ t_rank, const uint32_t* __restrict__ rank_of,
                            uint32_t n, uint64_t* __restrict__ out) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    out[v] = t_rank[rank_of[v]];
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
  // 0 start, 1 plan done, 2 join done, 3 outputs done; around the join
  // kernels: 4-5 warp, 5-6 small, 7-8 dense (lo stream), 10-11 cta (hi
  // stream), 12-9 rows
  cudaEvent_t e[13] = {};
  bool on = false;
  explicit Events(bool enable) : on(enable) {  // only a timed call (stats) creates them
    if (on)
      for (auto& x : e) TC_CUDA(cudaEventCreate(&x));
  }
  ~Events() {
    if (on)
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
  if (g.part_bounds_P == parts && g.part_bounds.size() == (size_t)parts + 1) return g.part_bounds;
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  g.part_bounds.assign((size_t)parts + 1, 0);
  g.part_bounds[parts] = n;
  if (g.E && parts > 1) {
    const uint32_t nr = n - g.r0;
    DBuf<unsigned long long> jv(nr, s);
    DBuf<uint64_t> prefix(nr, s), tot(1, s), bnd((uint64_t)parts + 1, s);
    TC_CUDA(cudaMemsetAsync(jv.get(), 0, sizeof(unsigned long long) * nr, s));
    k_pivot_wedges<<<grid_gs(g.E, g.device), 256, 0, s>>>(g.rowd.get(), g.col.get(), g.src.get(), g.E, g.r0,
                                                          env_u32("TCB_DENSE_COST", TCB_DENSE_COST),
                                                          env_u32("TCB_COLD_COST", TCB_COLD_COST),
                                                          env_u32("TCB_WARP_COST", TCB_WARP_COST),
                                                          env_u32("TCB_SMALL_COST", TCB_SMALL_COST),
                                                          env_u32("TCB_SLAB_COST", TCB_SLAB_COST),
                                                          PivotClass{g.off.get(), g.offH.get(), g.inoff.get(), false},
                                                          jv.get());
    TC_LAUNCH();
    const uint64_t item_cost = env_u32("TCB_ITEM_COST", (uint32_t)kItemCost);  // cost-model knobs
    const uint64_t seg_cost = env_u32("TCB_SEG_COST", (uint32_t)kSegRowCost);
    scan_exclusive<uint64_t>(PivotCost{g.off.get(), g.inoff.get(), jv.get(), item_cost, seg_cost, g.r0},
                             prefix.get(), nr, tot.get(), s);
    const uint64_t total_cost = read_scalar(tot.get(), s);
    k_part_bounds<<<ceil_div(parts + 1, 128), 128, 0, s>>>(prefix.get(), g.r0, n, total_cost, parts, bnd.get());
    TC_LAUNCH();
    TC_CUDA(cudaMemcpyAsync(g.part_bounds.data(), bnd.get(), (parts + 1) * sizeof(uint64_t),
                            cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
  }
  g.part_bounds_P = parts;
  return g.part_bounds;
}

namespace {
template <typename K>
int occupancy(K kern, int threads, size_t smem) {
  TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // TCB_CARVEOUT (percent of the unified L1/shared array as shared memory):
  // a tuning knob; by default the driver picks the carveout
  if (const char* c = getenv("TCB_CARVEOUT"))
    TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(c)));
  int occ = 0;
  TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
  if (getenv("TCB_PHASES")) fprintf(stderr, "[tcb] occupancy %d blocks/SM (smem %zu + static)\n", occ, smem);
  return occ < 1 ? 1 : occ;
}
}  // namespace

void count_triangles(tc_graph& g, const tc_count_opts& opts, uint64_t* d_total, uint64_t* d_pv,
                     tc_count_stats* stats) {
  cudaStream_t s = g.stream;
  const int dev = g.device;
  const uint32_t n = g.n;
  const uint32_t parts = opts.part_count ? opts.part_count : 1;
  const uint32_t part = opts.part_count ? opts.part_index : 0;
  const bool pv = d_pv != nullptr;
  const bool timing = stats != nullptr;
  Events ev(timing);
  if (timing) TC_CUDA(cudaEventRecord(ev.e[0], s));
  uint64_t kl = 0;  // kernels launched by this call
  PhaseLog pl(s);

  unsigned long long* acc = g.scratch[kSlotAcc].get<unsigned long long>(2, s);  // [0] total, [1] row queue
  TC_CUDA(cudaMemsetAsync(acc, 0, sizeof(unsigned long long), s));
  unsigned long long* t_rank = nullptr;
  if (pv) {
    t_rank = g.scratch[kSlotTRank].get<unsigned long long>(n ? n : 1, s);
    TC_CUDA(cudaMemsetAsync(t_rank, 0, sizeof(unsigned long long) * (n ? n : 1), s));
  }

  // ---- level-1 frontier plan of the whole graph, or of this part's
  //      degree-weighted pivot rank range (multi-GPU) ----
  uint32_t v_lo = 0, v_hi = n;
  if (parts > 1 && g.E) {
    const std::vector<uint64_t>& b = partition_bounds(g, parts);  // cached per P
    v_lo = (uint32_t)b[part];
    v_hi = (uint32_t)b[part + 1];
  }
  const bool split = v_lo != 0 || v_hi != n;
  Plan plan;
  constexpr bool kUseMasks = TCB_PV_MASKS;
  // Uniform-degree graphs (every pivot's row and in-edge list fit one
  // warp-bin segment, e.g. Erdos-Renyi): no plan, no CTA/small bins, no hit
  // masks -- the warp join takes the pivots directly (TCB_DIRECT=0: off).
  const bool direct = g.max_dplus <= kWarpMaxDeg && g.max_din <= kWarpSegItems && env_u32("TCB_DIRECT", 1) != 0;
  const bool want_sums = stats != nullptr && opts.work_counters != 0;
  if (!direct || want_sums) kl += build_plan(g, v_lo, v_hi, pv, pv && kUseMasks && !direct, want_sums, plan);
  if (direct) plan.cap[1] = plan.cap[2] = 0;
  uint8_t* masks = direct ? nullptr : plan.masks;
  pl.mark("plan");
  if (timing) TC_CUDA(cudaEventRecord(ev.e[1], s));

  // ---- advance + join ----
  const int sms = num_sms(dev);
  uint64_t launches = 0;
  // per-vertex SMEM counters for the top ranks [rc, n); TCB_TOP_COUNTERS /
  // TCB_SMEM_SLOTS shrink them so tests drive every path on small graphs
  const uint32_t top_cnt = env_u32("TCB_TOP_COUNTERS", kTopCounters);
  const uint32_t smem_slots = std::min(env_u32("TCB_SMEM_SLOTS", kCtaSmemSlots), kCtaSmemSlots);
  const uint32_t ncnt = pv ? ((n < top_cnt ? n : top_cnt) & ~1u) : 0;
  {
    // diagnostics knob (TCB_PV_DBG); set synchronously and only when it
    // changes, so a count stays free of host-memory copies (CUDA-graph
    // capturable: bench.py replays whole counts as one graph)
    static uint32_t dbg_set = 0;
    const uint32_t dbg = env_u32("TCB_PV_DBG", 0);
    if (dbg != dbg_set) {
      TC_CUDA(cudaStreamSynchronize(s));
      TC_CUDA(cudaMemcpyToSymbol(g_pv_dbg, &dbg, sizeof(dbg)));
      dbg_set = dbg;
    }
  }
  const uint32_t nbm = (n - g.h0 + 31) / 32;
  unsigned int* queues = g.scratch[kSlotCounters].get<unsigned int>(16, s) + 4;  // [0..3] = plan.nseg
  TC_CUDA(cudaMemsetAsync(queues, 0, 8 * sizeof(unsigned int), s));
  // Fork: the dominant CTA join on a high-priority stream, the warp / small /
  // dense joins (independent of it: disjoint items, atomic outputs) on a
  // low-priority one -- their blocks fill the SMs the CTA join's tail frees.
  // Join back before the row pass.  (TCB_CONCURRENT=0: one stream.)
  const bool fork = env_u32("TCB_CONCURRENT", 0) != 0;  // measured: no gain (profiles/README.md)
  // the CTA join's launch shape and global-slab scratch (taken before the fork)
  const uint32_t ncnt_hits0 = (pv && !kUseMasks) ? std::min<uint32_t>(ncnt, env_u32("TCB_HIT_COUNTERS", 4096)) & ~1u : 0;
  const uint32_t rc_hits0 = ncnt_hits0 ? n - ncnt_hits0 : 0xffffffffu;
  const uint32_t slab_cap = (table_size_for(g.max_dplus) > smem_slots) ? table_size_for(g.max_dplus) : 0;
  const size_t cta_dsm = ((size_t)nbm + kCtaSmemSlots + ncnt_hits0 / 2) * sizeof(uint32_t);
  auto cta_kern = pv ? k_join_cta<true> : k_join_cta<false>;
  const unsigned cta_grid =
      plan.cap[1] ? (unsigned)std::min<uint64_t>((uint64_t)sms * occupancy(cta_kern, kCtaThreads, cta_dsm), plan.cap[1])
                  : 0u;
  uint32_t* slab = plan.cap[1] ? g.scratch[kSlotSlab].get<uint32_t>((uint64_t)cta_grid * slab_cap + 1, s) : nullptr;
  cudaStream_t sh = s, sl = s;
  if (fork) {
    if (!g.hi_stream) {
      int least = 0, greatest = 0;
      TC_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      TC_CUDA(cudaStreamCreateWithPriority(&g.hi_stream, cudaStreamNonBlocking, greatest));
      TC_CUDA(cudaStreamCreateWithPriority(&g.lo_stream, cudaStreamNonBlocking, least));
      for (cudaEvent_t* e : {&g.fork_ev, &g.join_hi, &g.join_lo})
        TC_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    sh = g.hi_stream;
    sl = g.lo_stream;
    TC_CUDA(cudaEventRecord(g.fork_ev, s));
    TC_CUDA(cudaStreamWaitEvent(sh, g.fork_ev, 0));
    TC_CUDA(cudaStreamWaitEvent(sl, g.fork_ev, 0));
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[10], sh));
  if (plan.cap[1]) {
    // cold members spill to a per-CTA global slab only when a pivot has more
    // than smem_slots/2 members below h0
    cta_kern<<<cta_grid, kCtaThreads, cta_dsm, sh>>>(
        g.off.get(), g.col.get(), g.rowd.get(), g.r0, g.colH.get(), g.irec.get(), plan.csegs, plan.nseg + 1,
        queues + 1, g.h0, nbm, smem_slots, slab_cap, slab, masks, rc_hits0, ncnt_hits0, t_rank, acc);
    TC_LAUNCH();
    ++launches;
    pl.mark("join_cta");
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[11], sh));
  if (timing) TC_CUDA(cudaEventRecord(ev.e[4], sl));
  if (plan.cap[0] || direct) {
    // warp bin: plain 32-bit counters over half the window
    const uint32_t ncnt_w = ncnt / 2, rc_w = pv ? n - ncnt_w : 0xffffffffu;
    const size_t smem = (size_t)ncnt_w * sizeof(uint32_t);
    auto kern = pv ? k_join_warp<true> : k_join_warp<false>;
    const int occ = occupancy(kern, kJoinThreads, smem);
    const uint64_t resident_warps = (uint64_t)sms * occ * kJoinWarps;
    const uint64_t nseg_w = direct ? (uint64_t)(v_hi - v_lo) : plan.cap[0];
    const uint32_t gsz = nseg_w >= (uint64_t)kWarpGroup * resident_warps ? kWarpGroup : 1u;
    const unsigned grid =
        (unsigned)std::min<uint64_t>(ceil_div64(ceil_div64(nseg_w, gsz), kJoinWarps), (uint64_t)sms * occ);
    kern<<<grid ? grid : 1, kJoinThreads, smem, sl>>>(g.off.get(), g.rowd.get(), g.r0, g.col.get(), g.irec.get(),
                                                     plan.wsegs, plan.nseg + 0, direct ? g.inoff.get() : nullptr,
                                                     v_lo, v_hi, gsz, rc_w, ncnt_w, masks, t_rank, acc);
    TC_LAUNCH();
    ++launches;
    pl.mark("join_warp");
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[5], sl));
  // per-hit top counters of the CTA / small bins (no-mask per-vertex mode)
  const uint32_t ncnt_hits = (pv && !kUseMasks) ? std::min<uint32_t>(ncnt, env_u32("TCB_HIT_COUNTERS", 4096)) & ~1u : 0;
  const uint32_t rc_hits = ncnt_hits ? n - ncnt_hits : 0xffffffffu;
  if (plan.cap[2]) {
    const uint32_t ncnt_s = ncnt_hits / 2;  // 32-bit counters: half the window
    const size_t ssm = (size_t)kSmallWarps * ((SmallWarpSmem::bytes(nbm) + 15) & ~15u) + (size_t)ncnt_s * 4;
    auto kern = pv ? k_join_small<true> : k_join_small<false>;
    const int occ = occupancy(kern, kSmallThreads, ssm);
    const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)sms * occ, ceil_div64(plan.cap[2], kSmallWarps));
    kern<<<grid, kSmallThreads, ssm, sl>>>(g.off.get(), g.col.get(), g.rowd.get(), g.r0, g.colH.get(), g.irec.get(),
                                         plan.ssegs, plan.nseg + 2, queues + 0, g.h0, nbm, masks,
                                         ncnt_s ? n - ncnt_s : 0xffffffffu, ncnt_s, t_rank, acc);
    TC_LAUNCH();
    ++launches;
    pl.mark("join_small");
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[6], sl));
  if (timing) TC_CUDA(cudaEventRecord(ev.e[7], sl));
  if (g.ndine) {
    // dense core parts: word-parallel intersections (k_join_dense)
    const bool cw3 = g.core_words > 32u * 2u;  // core words per lane: 3 (3072-rank core), else <= 2
    auto kern = pv ? (cw3 ? k_join_dense<true, 3> : k_join_dense<true, 2>)
                   : (cw3 ? k_join_dense<false, 3> : k_join_dense<false, 2>);
    const int occ = occupancy(kern, kDenseThreads, 0);
    kern<<<(unsigned)(sms * occ), kDenseThreads, 0, sl>>>(
        g.dseg.get(), g.dsoff.get(), v_lo, v_hi, queues + 4, g.dine.get(), g.drow.get(), g.cbits.get(), g.core_words,
        g.cb, g.cb - g.h0, g.core_min, g.rowd.get(), g.r0, g.colH.get(), t_rank, acc);
    TC_LAUNCH();
    ++launches;
    pl.mark("join_dense");
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[8], sl));
  if (fork) {  // join
    TC_CUDA(cudaEventRecord(g.join_hi, sh));
    TC_CUDA(cudaEventRecord(g.join_lo, sl));
    TC_CUDA(cudaStreamWaitEvent(s, g.join_hi, 0));
    TC_CUDA(cudaStreamWaitEvent(s, g.join_lo, 0));
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[12], s));
  if (pv && kUseMasks && n && g.mask_total && !direct) {
    // hot hit masks -> t[u], t[x] (row-major, no per-hit atomics); a split
    // count folds only the items of its own pivots
    unsigned int* rq = queues + 2;  // heavy queue, heavy count
    unsigned long long* lq = g.scratch[kSlotAcc].get<unsigned long long>(2, s) + 1;
    TC_CUDA(cudaMemsetAsync(lq, 0, sizeof(unsigned long long), s));
    uint32_t* heavy = g.scratch[kSlotHeavy].get<uint32_t>(n, s);
    const uint32_t rcnt = n < top_cnt ? n : top_cnt;
    const size_t rsm = (size_t)rcnt * sizeof(uint32_t);
    auto rows_kern = split ? k_pv_rows<8> : k_pv_rows<4>;
    const int rocc = occupancy(rows_kern, kRowWarps * 32, rsm);
    const int hocc = occupancy(k_pv_rows_heavy, kRowWarps * 32, rsm);
    // items u -> v of pivots [v_lo, v_hi) have u < v_hi: rows [v_hi, n) skip
    // (the light pass walks rows top-down from queue position n - v_hi)
    PartRange pr{g.col.get(), v_lo, v_hi == n ? 0xffffffffu : v_hi, split, g.r0, nullptr};
    if (split && n > g.r0) {
      // per-row item ranges of this part, cached per (P, part) on the handle
      if (g.part_kr_P != parts || g.part_kr.size() != parts) {
        g.part_kr.clear();
        g.part_kr.resize(parts);
        g.part_kr_P = parts;
      }
      DBuf<uint2>& kr = g.part_kr[part];
      if (!kr.get()) {
        kr.alloc(n - g.r0, s);
        k_part_krange<<<grid_gs(n - g.r0, dev), 256, 0, s>>>(pr, g.off.get(), n, kr.get());
        TC_LAUNCH();
      }
      pr.krange = kr.get();
    }
    rows_kern<<<(unsigned)(sms * rocc), kRowWarps * 32, rsm, s>>>(
        g.rowd.get(), g.colH.get(), masks, n, pr, g.h0, n - rcnt, rcnt, lq, heavy, rq + 1, row_heavy_threshold(n),
        n - v_hi, t_rank);
    TC_LAUNCH();
    ++launches;
    pl.mark("pv_rows_light");
    k_pv_rows_heavy<<<(unsigned)(sms * hocc), kRowWarps * 32, rsm, s>>>(
        g.rowd.get(), g.colH.get(), masks, pr, g.h0, n - rcnt, rcnt, rq, heavy, rq + 1, t_rank);
    TC_LAUNCH();
    ++launches;
    pl.mark("pv_rows");
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[9], s));
  if (timing) TC_CUDA(cudaEventRecord(ev.e[2], s));

  // ---- outputs ----
  TC_CUDA(cudaMemcpyAsync(d_total, acc, sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  if (pv && n) {
    k_gather_pv<<<grid_gs(n, dev), 256, 0, s>>>(t_rank, g.rank_of.get(), n, d_pv);
    TC_LAUNCH();
    ++kl;
  }
  if (timing) TC_CUDA(cudaEventRecord(ev.e[3], s));
  if (stats) {
    TC_CUDA(cudaEventSynchronize(ev.e[3]));
    read_plan_sums(plan, s);
    stats->frontier_ms = ev.ms(0, 1);
    stats->join_ms = ev.ms(1, 2);
    stats->reduce_ms = ev.ms(2, 3);
    stats->total_ms = ev.ms(0, 3);
    stats->join_launches = launches;
    stats->kernel_launches = kl + launches;
    stats->part_first_vertex = v_lo;
    stats->part_last_vertex = v_hi;
    stats->warp_ms = ev.ms(4, 5);
    stats->small_ms = ev.ms(5, 6);
    stats->cta_ms = ev.ms(10, 11);
    stats->dense_ms = ev.ms(7, 8);
    stats->rows_ms = ev.ms(12, 9);
    if (opts.work_counters) {
      stats->items = plan.items;
      stats->wedges = plan.J;
      stats->pivots = plan.pivots;
      stats->dag_W = (double)plan.W;
      // this part's share of SURVEY 8d's B_alg (vertex terms on part 0): the
      // parts' values sum to the whole graph's.  |E+| is counted per in-edge
      // of the part's pivots.
      uint32_t in_lo = 0, in_hi = 0;
      TC_CUDA(cudaMemcpy(&in_lo, g.inoff.get() + v_lo, sizeof(uint32_t), cudaMemcpyDeviceToHost));
      TC_CUDA(cudaMemcpy(&in_hi, g.inoff.get() + v_hi, sizeof(uint32_t), cudaMemcpyDeviceToHost));
      const double Ep = (double)(in_hi - in_lo);
      stats->alg_bytes = 4.0 * (double)plan.W + 12.0 * Ep +
                         (part == 0 ? 8.0 * ((double)n + 1) + (pv ? 8.0 * n : 0.0) : 0.0);
      // bytes the implemented join streams per count: hot ids 2 B, cold ids
      // 4 B, the in-edge record 8 B + its row geometry 16 B per item, the
      // pivot rows 4 B per member per segment; per-vertex: the hit masks
      // written and read back (1 B per hot chunk, twice) and the u64 counters
      stats->probe_bytes = 2.0 * (double)plan.hot + 4.0 * (double)(plan.J - plan.hot) + 24.0 * Ep +
                           4.0 * Ep + (pv ? 2.0 * (double)g.mask_total + 16.0 * n : 0.0);
      stats->cta_bytes = plan.cta_bytes;
      stats->dense_bytes = plan.dense_bytes;
    }
  }
}

}  // namespace tcb
