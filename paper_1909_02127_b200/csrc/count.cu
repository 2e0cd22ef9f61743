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

__device__ __forceinline__ uint32_t hash_slot(uint32_t x, uint32_t mask) { return x & mask; }

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

__global__ void k_item_count(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                             const uint32_t* __restrict__ src, uint64_t E, uint32_t* __restrict__ cnt,
                             FrontierSums* __restrict__ sums) {
  unsigned long long W = 0, J = 0, I = 0;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = col[e];
    const uint32_t dv = off[v + 1] - off[v];
    const uint32_t end = off[src[e] + 1];
    W += dv;
    if (dv > 0 && e + 1 < end) {
      atomicAdd(&cnt[v], 1u);
      J += end - (e + 1);
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
                               const uint32_t* __restrict__ src, uint64_t E, const uint32_t* __restrict__ in_off,
                               uint32_t* __restrict__ fill, uint2* __restrict__ items) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = col[e];
    const uint32_t dv = off[v + 1] - off[v];
    const uint32_t end = off[src[e] + 1];
    if (dv > 0 && e + 1 < end) {
      const uint32_t p = in_off[v] + atomicAdd(&fill[v], 1u);
      items[p] = make_uint2((uint32_t)e + 1, end);
    }
  }
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

// Probe x in an open-addressing table (linear probing).  Returns the slot or
// kEmpty.
__device__ __forceinline__ uint32_t probe(const uint32_t* tab, uint32_t mask, uint32_t x) {
  uint32_t s = hash_slot(x, mask);
  while (true) {
    const uint32_t k = tab[s];
    if (k == x) return s;
    if (k == kEmpty) return kEmpty;
    s = (s + 1) & mask;
  }
}

__device__ __forceinline__ void insert(uint32_t* tab, uint32_t mask, uint32_t x) {
  uint32_t s = hash_slot(x, mask);
  while (atomicCAS(&tab[s], kEmpty, x) != kEmpty) s = (s + 1) & mask;
}

// One warp processes items [i0, i1) of pivot v against the table `tab`.
// Advance: items -> 16-byte chunks of their suffixes, load-balanced across
// lanes; join: each element x in the item's [b,e) is probed.  Returns the
// lane's hit count; per-vertex updates go to slot counters (t[c]), per-item
// counters (t[a]).
template <bool kPerVertex>
__device__ __forceinline__ uint32_t warp_join_items(const uint2* __restrict__ items, uint32_t i0, uint32_t i1,
                                                    const uint32_t* __restrict__ col,
                                                    const uint32_t* __restrict__ src, const uint32_t* tab,
                                                    uint32_t* slot_cnt, uint32_t mask, uint32_t xmax,
                                                    uint32_t* item_cnt /* 32 per warp, smem */,
                                                    unsigned long long* __restrict__ t_rank) {
  const unsigned lane = lane_id();
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
    const uint32_t pre = warp_inclusive_scan(nch);  // inclusive chunk prefix
    const uint32_t start = pre - nch;
    const uint32_t total = __shfl_sync(0xffffffffu, pre, 31);
    if (kPerVertex) {
      item_cnt[lane] = 0;
      __syncwarp();
    }
    for (uint32_t base = 0; base < total; base += 32) {
      const uint32_t f = base + lane;
      // item containing chunk `base`: count of items ending at or before it
      const uint32_t kb = __popc(__ballot_sync(0xffffffffu, nch && pre <= base));
      const uint32_t bit = (nch && start > base && start < base + 32) ? (1u << (start - base)) : 0u;
      const uint32_t smask = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t k = kb + __popc(smask & ((2u << lane) - 1u));
      const uint32_t kk = k < 32 ? k : 31;
      const uint32_t bk = __shfl_sync(0xffffffffu, b, kk);
      const uint32_t ek = __shfl_sync(0xffffffffu, e, kk);
      const uint32_t sk = __shfl_sync(0xffffffffu, start, kk);
      if (f < total) {
        const uint32_t c = (bk >> 2) + (f - sk);
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(col) + c);
        const uint32_t p0 = c << 2;
        uint32_t h = 0;
        const uint32_t xs[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t p = p0 + t;
          const uint32_t x = xs[t];
          if (p >= bk && p < ek && x <= xmax) {
            const uint32_t s = probe(tab, mask, x);
            if (s != kEmpty) {
              ++h;
              if (kPerVertex) atomicAdd(&slot_cnt[s], 1u);
            }
          }
        }
        hits += h;
        if (kPerVertex && h) atomicAdd(&item_cnt[k], h);
      }
    }
    if (kPerVertex) {
      __syncwarp();
      const uint32_t c = item_cnt[lane];
      if (c) atomicAdd(&t_rank[src[b - 1]], (unsigned long long)c);
      __syncwarp();
    }
  }
  return hits;
}

// Warp bin: each warp takes whole segments of small pivots (d+ <= 48) with a
// warp-private 128-slot table.
template <bool kPerVertex>
__global__ void __launch_bounds__(kJoinThreads) k_join_warp(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
    const uint2* __restrict__ items, const uint32_t* __restrict__ in_off, const uint2* __restrict__ segs,
    uint32_t nsegs, uint32_t seg_lo, uint32_t seg_stride, unsigned long long* __restrict__ t_rank,
    unsigned long long* __restrict__ total) {
  __shared__ uint32_t s_tab[kJoinWarps][kWarpTable];
  __shared__ uint32_t s_cnt[kJoinWarps][kPerVertex ? kWarpTable : 1];
  __shared__ uint32_t s_item[kJoinWarps][32];
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t* tab = s_tab[warp];
  uint32_t* scnt = s_cnt[warp];
  for (uint32_t s = lane; s < kWarpTable; s += 32) {
    tab[s] = kEmpty;
    if (kPerVertex) scnt[s] = 0;
  }
  __syncwarp();
  unsigned long long acc = 0;
  const uint32_t gw = blockIdx.x * kJoinWarps + warp, nw = gridDim.x * kJoinWarps;
  for (uint32_t si = seg_lo + gw * seg_stride; si < nsegs; si += nw * seg_stride) {
    const uint2 sg = segs[si];
    const uint32_t v = sg.x, i0 = sg.y;
    const uint32_t i1 = min(i0 + kWarpSegItems, in_off[v + 1]);
    const uint32_t nb = off[v], dv = off[v + 1] - nb;
    const uint32_t mask = kWarpTable - 1;
    uint32_t xmax = 0;
    for (uint32_t j = lane; j < dv; j += 32) {
      const uint32_t x = col[nb + j];
      insert(tab, mask, x);
      xmax = max(xmax, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    __syncwarp();
    const uint32_t h = warp_join_items<kPerVertex>(items, i0, i1, col, src, tab, scnt, mask, xmax,
                                                   s_item[warp], t_rank);
    __syncwarp();
    const uint32_t hw = warp_sum(h);
    acc += h;
    if (kPerVertex) {
      for (uint32_t s = lane; s < kWarpTable; s += 32) {
        const uint32_t c = scnt[s];
        if (c) {
          atomicAdd(&t_rank[tab[s]], (unsigned long long)c);
          scnt[s] = 0;
        }
        tab[s] = kEmpty;
      }
      if (lane == 0 && hw) atomicAdd(&t_rank[v], (unsigned long long)hw);
    } else {
      for (uint32_t s = lane; s < kWarpTable; s += 32) tab[s] = kEmpty;
    }
    __syncwarp();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
}

// CTA bin: the CTA builds the table of N+(v) once per segment (table in SMEM,
// or in a per-CTA global slab when d+(v) is too large for SMEM), its warps
// share it.  Segments are taken from a global queue, heaviest (top-rank
// pivots) first.
template <bool kPerVertex, bool kGlobalTable>
__global__ void __launch_bounds__(kJoinThreads, 2) k_join_cta(
    const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, const uint32_t* __restrict__ src,
    const uint2* __restrict__ items, const uint32_t* __restrict__ in_off, const uint2* __restrict__ segs,
    uint32_t nsegs, uint32_t seg_lo, uint32_t seg_stride, unsigned int* __restrict__ queue,
    uint32_t table_cap, uint32_t* __restrict__ gslab, unsigned long long* __restrict__ t_rank,
    unsigned long long* __restrict__ total) {
  extern __shared__ uint32_t dyn[];
  __shared__ uint32_t s_item[kJoinWarps][32];
  __shared__ uint32_t s_seg, s_xmax, s_hits;
  uint32_t* tab = kGlobalTable ? gslab + (uint64_t)blockIdx.x * table_cap * (kPerVertex ? 2 : 1) : dyn;
  uint32_t* scnt = tab + table_cap;
  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  for (uint32_t s = threadIdx.x; s < table_cap; s += kJoinThreads) {
    tab[s] = kEmpty;
    if (kPerVertex) scnt[s] = 0;
  }
  unsigned long long acc = 0;
  while (true) {
    if (threadIdx.x == 0) {
      s_seg = atomicAdd(queue, 1u);
      s_xmax = 0;
      s_hits = 0;
    }
    __syncthreads();
    const uint32_t q = s_seg;
    const uint64_t sidx64 = (uint64_t)seg_lo + (uint64_t)q * seg_stride;
    if (sidx64 >= nsegs) break;
    const uint32_t si = nsegs - 1 - (uint32_t)sidx64;  // heaviest (top ranks) first
    const uint2 sg = segs[si];
    const uint32_t v = sg.x, i0 = sg.y;
    const uint32_t i1 = min(i0 + kCtaSegItems, in_off[v + 1]);
    const uint32_t nb = off[v], dv = off[v + 1] - nb;
    const uint32_t ts = table_size_for(dv);
    const uint32_t mask = ts - 1;
    uint32_t xmax = 0;
    for (uint32_t j = threadIdx.x; j < dv; j += kJoinThreads) {
      const uint32_t x = col[nb + j];
      insert(tab, mask, x);
      xmax = max(xmax, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xmax = max(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    if (lane == 0) atomicMax(&s_xmax, xmax);
    if (kGlobalTable) __threadfence_block();
    __syncthreads();
    xmax = s_xmax;
    // warps take 32-item batches of the segment
    uint32_t h = 0;
    for (uint32_t ib = i0 + warp * 32; ib < i1; ib += kJoinWarps * 32)
      h += warp_join_items<kPerVertex>(items, ib, min(ib + 32, i1), col, src, tab, scnt, mask, xmax,
                                       s_item[warp], t_rank);
    acc += h;
    if (kPerVertex) {
      const uint32_t hw = warp_sum(h);
      if (lane == 0 && hw) atomicAdd(&s_hits, hw);
    }
    if (kGlobalTable) __threadfence_block();
    __syncthreads();
    if (kPerVertex) {
      for (uint32_t s = threadIdx.x; s < ts; s += kJoinThreads) {
        const uint32_t c = scnt[s];
        if (c) {
          atomicAdd(&t_rank[tab[s]], (unsigned long long)c);
          scnt[s] = 0;
        }
        tab[s] = kEmpty;
      }
      if (threadIdx.x == 0 && s_hits) atomicAdd(&t_rank[v], (unsigned long long)s_hits);
    } else {
      for (uint32_t s = threadIdx.x; s < ts; s += kJoinThreads) tab[s] = kEmpty;
    }
    if (kGlobalTable) __threadfence_block();
    __syncthreads();
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc) atomicAdd(total, acc);
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

  // ---- level-1 frontier: useful in-edges grouped by pivot ----
  DBuf<uint32_t> cnt(n ? n : 1, s), in_off((uint64_t)n + 1, s);
  DBuf<FrontierSums> sums(1, s);
  TC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(uint32_t) * (n ? n : 1), s));
  TC_CUDA(cudaMemsetAsync(sums.get(), 0, sizeof(FrontierSums), s));
  if (E) {
    k_item_count<<<grid_gs(E, dev), 256, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), E, cnt.get(), sums.get());
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
    k_item_scatter<<<grid_gs(E, dev), 256, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), E, in_off.get(),
                                                   fill.get(), items.get());
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
  const uint32_t NSW = hn[0], NSC = hn[1];
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
  if (NSW) {
    // part p of P takes segments p, p+P, ... (interleaved -> balanced)
    const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div64(ceil_div64(NSW, parts), kJoinWarps),
                                                       (uint64_t)sms * 8);
    if (pv)
      k_join_warp<true><<<grid, kJoinThreads, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), items.get(),
                                                      in_off.get(), wsegs.get(), NSW, part, parts,
                                                      t_rank.get(), acc.get());
    else
      k_join_warp<false><<<grid, kJoinThreads, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), items.get(),
                                                       in_off.get(), wsegs.get(), NSW, part, parts,
                                                       t_rank.get(), acc.get());
    TC_LAUNCH();
    ++launches;
  }
  if (NSC) {
    const uint32_t cap = table_size_for(g.max_dplus);
    const size_t smem = (size_t)cap * sizeof(uint32_t) * (pv ? 2 : 1);
    DBuf<unsigned int> queue(1, s);
    TC_CUDA(cudaMemsetAsync(queue.get(), 0, sizeof(unsigned int), s));
    const size_t kSmemMax = 160 * 1024;
    if (smem <= kSmemMax) {
      auto kern = pv ? k_join_cta<true, false> : k_join_cta<false, false>;
      TC_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int occ = 0;
      TC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kJoinThreads, smem));
      if (occ < 1) occ = 1;
      const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)sms * occ, ceil_div64(NSC, parts));
      kern<<<grid, kJoinThreads, smem, s>>>(g.off.get(), g.col.get(), g.src.get(), items.get(), in_off.get(),
                                           csegs.get(), NSC, part, parts, queue.get(), cap, nullptr,
                                           t_rank.get(), acc.get());
      TC_LAUNCH();
    } else {
      auto kern = pv ? k_join_cta<true, true> : k_join_cta<false, true>;
      const unsigned grid = (unsigned)std::min<uint64_t>((uint64_t)sms * 4, ceil_div64(NSC, parts));
      DBuf<uint32_t> slab((uint64_t)grid * cap * (pv ? 2 : 1), s);
      kern<<<grid, kJoinThreads, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), items.get(), in_off.get(),
                                        csegs.get(), NSC, part, parts, queue.get(), cap, slab.get(),
                                        t_rank.get(), acc.get());
      TC_LAUNCH();
    }
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
