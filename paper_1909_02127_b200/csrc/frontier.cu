// frontier.cu -- the level-1 frontier index: useful in-edges grouped by pivot.
//
// The reference materialises level-1 rows (u, w) with expand_level
// (matcher.cpp:136-198: advance over N(u), accept w > u, 2-core membership,
// look-ahead) before its final level.  Here the level-1 frontier is a
// graph-static index over the (deg,id)-oriented DAG: for every oriented edge
// e = u->v that can close a triangle as a pivot in-edge (d+(v) > 0 and a
// non-empty suffix of N+(u) after v) one item, grouped by pivot v and sorted
// by e (a stable order, so multi-GPU edge ranges select the same items on
// every rank).  Built once per graph, right after the oriented CSR:
//   keys (v << be | e) of useful edges -> radix sort -> item geometry ->
//   per-pivot offsets -> per-bin work segments.
#include <cuda_runtime.h>

#include <algorithm>

#include "graph.cuh"
#include "prim.cuh"

namespace tcb {
namespace {

constexpr int kT = 256;

unsigned grid_gs(uint64_t n, int device) {
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

struct Sums {
  unsigned long long W, J, hot, items_c;
};

// Useful in-edge?  Writes the sort key, or the all-ones sentinel.
__global__ void k_fr_keys(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ src, uint64_t E, int be, uint64_t sentinel,
                          uint64_t* __restrict__ keys, unsigned long long* __restrict__ W) {
  unsigned long long w = 0;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = col[e];
    const uint32_t dv = off[v + 1] - off[v];
    w += dv;
    const bool useful = dv > 0 && e + 1 < off[src[e] + 1];
    keys[e] = useful ? (((uint64_t)v << be) | e) : sentinel;
  }
  w = warp_sum(w);
  if (lane_id() == 0 && w) atomicAdd(W, w);
}

struct NotSentinel {
  const uint64_t* k;
  uint64_t sentinel;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return k[i] != sentinel ? 1u : 0u; }
};

// sorted keys -> item geometry, edge ids, per-pivot counts
__global__ void k_fr_items(const uint64_t* __restrict__ keys, uint64_t NI, int be, const uint32_t* __restrict__ off,
                           const uint32_t* __restrict__ src, const uint32_t* __restrict__ offH, uint32_t h0,
                           uint4* __restrict__ items, uint32_t* __restrict__ item_e, uint32_t* __restrict__ cnt,
                           uint32_t* __restrict__ item_of_e, Sums* __restrict__ sums) {
  const uint64_t emask = (1ull << be) - 1;
  unsigned long long J = 0, H = 0, IC = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < NI; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool valid = i < NI;
    uint32_t v = 0xffffffffu;
    if (valid) {
      const uint64_t key = keys[i];
      v = (uint32_t)(key >> be);
      const uint32_t e = (uint32_t)(key & emask);
      const uint32_t dv = off[v + 1] - off[v];
      const uint32_t u = src[e];
      const uint32_t end = off[u + 1];
      J += end - (e + 1);
      uint4 it;
      if (dv <= kWarpMaxDeg) {
        it = make_uint4(e + 1, end, 0, 0);
      } else {
        const uint32_t ohb = offH[u], ohe = offH[u + 1];
        const uint32_t cold_end = end - (ohe - ohb);
        if (v >= h0) {  // v itself is hot: the whole suffix is hot
          it = make_uint4(ohb + (e - cold_end) + 1, ohe, 0, 0);
        } else {
          it = make_uint4(ohb, ohe, e + 1, cold_end);
        }
        H += it.y - it.x;
        ++IC;
        item_of_e[e] = (uint32_t)i;
      }
      items[i] = it;
      item_e[i] = e;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, v);
    if (valid && lane_id() == (unsigned)(__ffs(peers) - 1)) atomicAdd(&cnt[v], (uint32_t)__popc(peers));
  }
  J = warp_sum(J);
  H = warp_sum(H);
  IC = warp_sum(IC);
  if (lane_id() == 0) {
    atomicAdd(&sums->J, J);
    atomicAdd(&sums->hot, H);
    atomicAdd(&sums->items_c, IC);
  }
}

// Per-vertex hit masks (count.cu): one byte per hot chunk of every CTA-bin item.
// Mask bytes of oriented edge e's CTA-bin item (0 if none / warp bin).  The
// scan runs in edge order, so each row's masks are contiguous: the per-vertex
// row pass (count.cu k_pv_rows) streams them instead of gathering per item.
struct MaskBytes {
  const uint4* items;
  const uint32_t* item_of_e;
  const uint32_t* off;
  const uint32_t* col;
  __device__ __forceinline__ uint64_t operator()(uint64_t e) const {
    const uint32_t i = item_of_e[e];
    if (i == 0xffffffffu) return 0;
    const uint32_t v = col[e];
    if (off[v + 1] - off[v] <= kWarpMaxDeg) return 0;
    const uint4 it = items[i];
    return it.y > it.x ? (uint64_t)(((it.y + 7) >> 3) - (it.x >> 3)) : 0ull;
  }
};

// Per-pivot item range of a part: [lo, hi) within [in[v], in[v+1]).
struct PartRange {
  const uint32_t* in;
  const uint32_t* item_e;
  uint64_t e0, e1;
  __device__ __forceinline__ uint2 operator()(uint32_t v) const {
    uint32_t a = in[v], b = in[v + 1];
    if (e0 == 0 && e1 == ~0ull) return make_uint2(a, b);
    uint32_t lo = a, hi = b;  // first item with e >= e0
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      if (item_e[m] < e0) lo = m + 1; else hi = m;
    }
    const uint32_t r0 = lo;
    hi = b;  // first item with e >= e1
    while (lo < hi) {
      const uint32_t m = (lo + hi) >> 1;
      if (item_e[m] < e1) lo = m + 1; else hi = m;
    }
    return make_uint2(r0, lo);
  }
};

struct SegCountBin {
  const uint32_t* off;
  PartRange pr;
  bool warp_bin;
  uint32_t per;
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const {
    const uint32_t dv = off[v + 1] - off[v];
    if (dv == 0 || (dv <= kWarpMaxDeg) != warp_bin) return 0;
    const uint2 r = pr((uint32_t)v);
    return (r.y - r.x + per - 1) / per;
  }
};

__global__ void k_fr_segs(const uint32_t* __restrict__ off, PartRange pr, uint32_t n, bool warp_bin, uint32_t per,
                          const uint32_t* __restrict__ seg_off, uint4* __restrict__ segs,
                          unsigned long long* __restrict__ npivots) {
  unsigned long long np = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t dv = off[v + 1] - off[v];
    if (dv == 0 || (dv <= kWarpMaxDeg) != warp_bin) continue;
    const uint2 r = pr((uint32_t)v);
    if (r.y <= r.x) continue;
    uint32_t s = seg_off[v];
    for (uint32_t i = r.x; i < r.y; i += per) segs[s++] = make_uint4((uint32_t)v, i, min(i + per, r.y), 0);
    ++np;
  }
  np = warp_sum(np);
  if (lane_id() == 0 && np) atomicAdd(npivots, np);
}

void make_segments(tc_graph& g, const PartRange& pr, DBuf<uint4>& wsegs, uint64_t& nw, DBuf<uint4>& csegs,
                   uint64_t& nc, uint64_t* npivots) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const uint32_t nn = n ? n : 1;
  DBuf<uint32_t> woff(nn, s), coff(nn, s), tot(2, s);
  DBuf<unsigned long long> np(1, s);
  TC_CUDA(cudaMemsetAsync(np.get(), 0, sizeof(unsigned long long), s));
  scan_exclusive<uint32_t>(SegCountBin{g.off.get(), pr, true, kWarpSegItems}, woff.get(), n, tot.get(), s);
  scan_exclusive<uint32_t>(SegCountBin{g.off.get(), pr, false, kCtaSegItems}, coff.get(), n, tot.get() + 1, s);
  uint32_t h[2] = {0, 0};
  TC_CUDA(cudaMemcpyAsync(h, tot.get(), 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  nw = n ? h[0] : 0;
  nc = n ? h[1] : 0;
  wsegs.alloc(nw ? nw : 1, s);
  csegs.alloc(nc ? nc : 1, s);
  if (nw) {
    k_fr_segs<<<grid_gs(n, g.device), kT, 0, s>>>(g.off.get(), pr, n, true, kWarpSegItems, woff.get(), wsegs.get(),
                                                   np.get());
    TC_LAUNCH();
  }
  if (nc) {
    k_fr_segs<<<grid_gs(n, g.device), kT, 0, s>>>(g.off.get(), pr, n, false, kCtaSegItems, coff.get(),
                                                   csegs.get(), np.get());
    TC_LAUNCH();
  }
  if (npivots) *npivots = read_scalar(np.get(), s);
}

}  // namespace

void build_frontier(tc_graph& g) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const uint64_t E = g.E;
  const int dev = g.device;
  cudaEvent_t t0, t1;
  TC_CUDA(cudaEventCreate(&t0));
  TC_CUDA(cudaEventCreate(&t1));
  TC_CUDA(cudaEventRecord(t0, s));
  const int bv = bits_for(n ? n - 1 : 0) ? bits_for(n ? n - 1 : 0) : 1;
  const int be = bits_for(E ? E - 1 : 0) ? bits_for(E ? E - 1 : 0) : 1;
  if (bv + be > 64) fail(TC_ERANGE, "frontier key exceeds 64 bits");
  const uint64_t sentinel = (bv + be >= 64) ? ~0ull : ((1ull << (bv + be)) - 1);
  DBuf<Sums> sums(1, s);
  TC_CUDA(cudaMemsetAsync(sums.get(), 0, sizeof(Sums), s));
  g.fr_in.alloc((uint64_t)n + 1, s);
  uint64_t NI = 0;
  if (E) {
    DBuf<uint64_t> k1(E, s), k2(E, s);
    k_fr_keys<<<grid_gs(E, dev), kT, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), E, be, sentinel, k1.get(),
                                             &sums.get()->W);
    TC_LAUNCH();
    DBuf<uint32_t> pos(1, s);
    // count useful (sentinels sort to the end)
    {
      DBuf<uint32_t> tmp(E, s);
      scan_exclusive<uint32_t>(NotSentinel{k1.get(), sentinel}, tmp.get(), E, pos.get(), s);
      NI = read_scalar(pos.get(), s);
    }
    uint64_t* sorted = radix_sort_u64(k1.get(), k2.get(), E, 0, bv + be, s);
    g.fr_items.alloc(NI ? NI : 1, s);
    g.fr_e.alloc(NI ? NI : 1, s);
    DBuf<uint32_t> item_of_e(E, s);  // CTA-bin item of edge e (~0 if none); build-time only
    TC_CUDA(cudaMemsetAsync(item_of_e.get(), 0xff, E * sizeof(uint32_t), s));
    DBuf<uint32_t> cnt(n ? n : 1, s);
    TC_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(uint32_t) * (n ? n : 1), s));
    if (NI) {
      k_fr_items<<<grid_gs(NI, dev), kT, 0, s>>>(sorted, NI, be, g.off.get(), g.src.get(), g.offH.get(), g.h0,
                                                 g.fr_items.get(), g.fr_e.get(), cnt.get(), item_of_e.get(),
                                                 sums.get());
      TC_LAUNCH();
    }
    scan_exclusive<uint32_t>(LoadArray<uint32_t>{cnt.get()}, g.fr_in.get(), n, g.fr_in.get() + n, s);
    // per-vertex hit-mask layout: one byte per hot chunk of every CTA-bin
    // item, in edge order (fr_moff[e], E+1 entries)
    g.fr_moff.alloc(E + 1, s);
    scan_exclusive<uint64_t>(MaskBytes{g.fr_items.get(), item_of_e.get(), g.off.get(), g.col.get()},
                             g.fr_moff.get(), E, g.fr_moff.get() + E, s);
    g.fr_mask_bytes = read_scalar(g.fr_moff.get() + E, s);
  } else {
    g.fr_items.alloc(1, s);
    g.fr_e.alloc(1, s);
    g.fr_moff.alloc(1, s);
    TC_CUDA(cudaMemsetAsync(g.fr_in.get(), 0, sizeof(uint32_t) * ((uint64_t)n + 1), s));
  }
  g.fr_nitems = NI;
  const Sums hs = read_scalar(sums.get(), s);
  g.fr_W = hs.W;
  g.fr_J = hs.J;
  g.fr_hot = hs.hot;
  g.fr_nitems_c = hs.items_c;
  make_segments(g, PartRange{g.fr_in.get(), g.fr_e.get(), 0, ~0ull}, g.fr_wsegs, g.fr_nwsegs, g.fr_csegs,
                g.fr_ncsegs, &g.fr_pivots);
  TC_CUDA(cudaEventRecord(t1, s));
  TC_CUDA(cudaEventSynchronize(t1));
  float ms = 0;
  cudaEventElapsedTime(&ms, t0, t1);
  g.frontier_ms = ms;
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
}

void part_segments(tc_graph& g, uint64_t e0, uint64_t e1, DBuf<uint4>& wsegs, uint64_t& nw, DBuf<uint4>& csegs,
                   uint64_t& nc) {
  make_segments(g, PartRange{g.fr_in.get(), g.fr_e.get(), e0, e1}, wsegs, nw, csegs, nc, nullptr);
}

}  // namespace tcb
