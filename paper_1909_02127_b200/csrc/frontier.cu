// frontier.cu -- the level-1 frontier: useful in-edges grouped by pivot, built
// inside every tc_count (it is part of the timed step, like the reference's
// level-1 expand_level inside match()).
//
// The reference materialises level-1 rows (u, w) with expand_level
// (matcher.cpp:136-198: advance over N(u), accept w > u, 2-core membership,
// look-ahead) before its final level.  Here, for every oriented edge
// e = u->v of this part's edge range [e0, e1) that can close a triangle as a
// pivot in-edge (d+(v) > 0 and a non-empty suffix of N+(u) after v), one
// item, grouped by pivot v:
//   slots         one item slot per in-edge of every pivot with d+(v) > 0,
//                 deg(v) - d+(v) (no edge pass), scanned -> in[v]; a
//                 multi-GPU part fills only the slots of its own edges, and
//                 every pivot's item count is its scatter cursor
//   rowbase       per-vertex only: exclusive scan of each row's hit-mask
//                 bytes (closed form, graph.cuh RowMasks)
//   k_fr_scatter  item geometry computed in edge order (the row data u, off,
//                 offH are read coalesced) and scattered to the pivot's slot
//                 through an atomic cursor.  Item order inside a pivot is
//                 arbitrary: every count is an order-independent integer sum.
//   segments      per-bin work segments (warp bin / CTA bin)
// A part only ever sees its own edges, so multi-GPU ranks build disjoint
// frontiers with no exchange.
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
  unsigned long long W, J, hot, items_c, claims;
};

// The level-1 item of oriented edge e = u->v (u = src[e], v = col[e]).  Every
// in-edge of a pivot with d+(v) > 0 gets a slot (claim); the item is useful
// when the suffix of N+(u) after v is non-empty, else it stays all-zero.
// Warp-bin pivots (d+(v) <= kWarpMaxDeg): {b, e} range of the 32-bit col[].
// CTA-bin pivots: {hb, he, cb, ce} = the suffix split into its hot part
// (16-bit colH) and its cold part (32-bit col).
struct Geom {
  uint32_t v, dv, u, k, d, O, h;
  uint4 it;
  bool claim, useful;
};
struct ItemGeom {
  const uint32_t* off;
  const uint32_t* col;
  const uint32_t* src;
  const uint32_t* offH;
  __device__ __forceinline__ void operator()(uint64_t e, Geom& q) const {
    q.v = col[e];
    q.dv = off[q.v + 1] - off[q.v];
    q.u = src[e];
    const uint32_t beg = off[q.u], end = off[q.u + 1];
    q.k = (uint32_t)e - beg;
    q.d = end - beg;
    q.O = offH[q.u];
    q.h = offH[q.u + 1] - q.O;
    q.claim = q.dv > 0;
    q.useful = q.claim && (uint32_t)e + 1 < end;
    q.it = make_uint4(0, 0, 0, 0);
    if (!q.useful) return;
    if (q.dv <= kWarpMaxDeg) {
      q.it = make_uint4((uint32_t)e + 1, end, 0, 0);
    } else {
      const uint32_t cold_end = end - q.h;
      if ((uint32_t)e + 1 >= cold_end)  // v is in the hot part: the whole suffix is hot
        q.it = make_uint4(q.O + ((uint32_t)e + 1 - cold_end), q.O + q.h, 0, 0);
      else
        q.it = make_uint4(q.O, q.O + q.h, (uint32_t)e + 1, cold_end);
    }
  }
};

// Item slots of a whole-graph count: every in-edge of a pivot with d+(v) > 0,
// i.e. deg(v) - d+(v), with no pass over the edges.
struct InSlotsWhole {
  const uint32_t* off;
  const uint32_t* deg;
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const {
    const uint32_t dv = off[v + 1] - off[v];
    return dv ? deg[v] - dv : 0u;
  }
};

// Mask bytes of row u (rows [u_lo, u_hi] of the part).
struct RowBytes {
  const uint32_t* off;
  const uint32_t* offH;
  uint32_t u_lo;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    const uint32_t u = u_lo + (uint32_t)i;
    const uint32_t O = offH[u];
    return RowMasks(off[u + 1] - off[u], O, offH[u + 1] - O).total();
  }
};

// Edge order, kR edges per thread in flight: geometry (row data read
// coalesced), then the slot claims (atomic cursors), then the scattered item
// stores.
#ifndef TCB_SCATTER_R
#define TCB_SCATTER_R 4
#endif
#ifndef TCB_SCATTER_MINB
#define TCB_SCATTER_MINB 1
#endif
constexpr int kScatterR = TCB_SCATTER_R;
template <bool kPV>
__global__ void __launch_bounds__(kT, TCB_SCATTER_MINB) k_fr_scatter(ItemGeom geo, uint64_t e0, uint64_t e1,
                                                  uint32_t* __restrict__ cursor,
                                                  uint4* __restrict__ items,
                                                  const uint64_t* __restrict__ rowbase, uint32_t u_lo,
                                                  uint8_t* __restrict__ masks,
                                                  Sums* __restrict__ sums) {
  unsigned long long W = 0, J = 0, H = 0, IC = 0, CL = 0;
  for (uint64_t base = e0 + (uint64_t)blockIdx.x * (kT * kScatterR); base < e1;
       base += (uint64_t)gridDim.x * (kT * kScatterR)) {
    Geom q[kScatterR];
    uint32_t pos[kScatterR];
#pragma unroll
    for (int r = 0; r < kScatterR; ++r) {
      const uint64_t e = base + r * kT + threadIdx.x;
      if (e < e1) {
        geo(e, q[r]);
      } else {
        q[r].claim = q[r].useful = false;
        q[r].dv = 0;
      }
    }
#pragma unroll
    for (int r = 0; r < kScatterR; ++r)
      if (q[r].claim) pos[r] = atomicAdd(&cursor[q[r].v], 1u);  // cursors start at in[v]
#pragma unroll
    for (int r = 0; r < kScatterR; ++r) {
      W += q[r].dv;
      // per-vertex: the mask bytes of items the CTA/small-bin joins will not
      // write (warp-bin pivots, pivots with d+ = 0) are zeroed here, so the
      // mask buffer needs no memset
      if (kPV && base + r * kT + threadIdx.x < e1 && (!q[r].claim || q[r].dv <= kWarpMaxDeg) && q[r].h > 0 &&
          q[r].k + 1 < q[r].d) {
        const RowMasks rm(q[r].d, q[r].O, q[r].h);
        uint8_t* z = masks + rowbase[q[r].u - u_lo] + rm.P(q[r].k);
        const uint32_t nb = (uint32_t)(rm.c_hi - rm.first_chunk(q[r].k));
        for (uint32_t i = 0; i < nb; ++i) z[i] = 0;
      }
      if (!q[r].claim) continue;
      ++CL;
      constexpr int S = kPV ? 2 : kItemStrideTotal;  // uint4s per item record
      uint64_t mo = 0;
      if (kPV && q[r].useful && q[r].dv > kWarpMaxDeg && q[r].it.y > q[r].it.x)
        mo = rowbase[q[r].u - u_lo] + RowMasks(q[r].d, q[r].O, q[r].h).P(q[r].k);
      if (kPV) {  // the 32-byte record as one 256-bit store (one full L2 sector)
        const uint4 a = q[r].it;
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(items + (uint64_t)pos[r] * 2),
                     "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(q[r].u), "r"(0u), "r"((uint32_t)mo),
                     "r"((uint32_t)(mo >> 32))
                     : "memory");
      } else if (S == 2) {  // total-only records padded to a full 32-byte sector
        const uint4 a = q[r].it;
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(items + (uint64_t)pos[r] * 2),
                     "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
                     : "memory");
      } else {
        items[pos[r]] = q[r].it;
      }
      if (!q[r].useful) continue;
      if (q[r].dv <= kWarpMaxDeg) {
        J += q[r].it.y - q[r].it.x;
      } else {
        J += (q[r].it.y - q[r].it.x) + (q[r].it.w - q[r].it.z);
        H += q[r].it.y - q[r].it.x;
        ++IC;
      }
    }
  }
  W = warp_sum(W);
  J = warp_sum(J);
  H = warp_sum(H);
  IC = warp_sum(IC);
  CL = warp_sum(CL);
  if (lane_id() == 0) {
    if (CL) atomicAdd(&sums->claims, CL);
    if (W) atomicAdd(&sums->W, W);
    if (J) atomicAdd(&sums->J, J);
    if (H) atomicAdd(&sums->hot, H);
    if (IC) atomicAdd(&sums->items_c, IC);
  }
}

// Pivot class: 0 = warp bin (d+ <= kWarpMaxDeg), 1 = CTA bin, 2 = small CTA
// pivots (<= kSmallItems items and <= kSmallCold members below the hot
// window: one warp each, k_join_small), -1 = no work.
struct PivotClass {
  const uint32_t* off;
  const uint32_t* offH;
  const uint32_t* in;
  const uint32_t* end;  // in[v] + items of v (the spent scatter cursor)
  __device__ __forceinline__ int operator()(uint64_t v) const {
    const uint32_t dv = off[v + 1] - off[v];
    const uint32_t items = end[v] - in[v];
    if (dv == 0 || items == 0) return -1;
    if (dv <= kWarpMaxDeg) return 0;
    const uint32_t hv = offH[v + 1] - offH[v];
    return (items <= kSmallItems && dv - hv <= kSmallCold) ? 2 : 1;
  }
};

// One pass over the pivots: class + 1 (0 = no work), one byte each; the three
// per-class scans and segment fills then read 5 bytes per pivot.
// ... and the per-class segment totals + the pivot count (tot[0..3]), so the
// host sizes every segment list after one read and skips empty classes.
__global__ void k_fr_class(PivotClass pc, uint32_t n, uint8_t* __restrict__ cls,
                           unsigned long long* __restrict__ tot) {
  constexpr uint32_t per[3] = {kWarpSegItems, kCtaSegItems, kSmallItems};
  unsigned long long t[4] = {0, 0, 0, 0};
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const int c = pc(v);
    cls[v] = (uint8_t)(c + 1);
    if (c >= 0) {
      const uint32_t items = pc.end[v] - pc.in[v];
      const unsigned long long ns = (items + per[c] - 1) / per[c];
      t[0] += c == 0 ? ns : 0;
      t[1] += c == 1 ? ns : 0;
      t[2] += c == 2 ? ns : 0;
      t[3] += 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const unsigned long long w = warp_sum(t[i]);
    if (lane_id() == 0 && w) atomicAdd(&tot[i], w);
  }
}

struct SegCountBin {
  const uint8_t* cls;
  const uint32_t* in;
  const uint32_t* end;
  uint32_t c;  // PivotClass + 1
  uint32_t per;
  __device__ __forceinline__ uint32_t operator()(uint64_t v) const {
    return cls[v] == c ? (end[v] - in[v] + per - 1) / per : 0u;
  }
};

__global__ void k_fr_segs(const uint8_t* __restrict__ cls, const uint32_t* __restrict__ in,
                          const uint32_t* __restrict__ end, uint32_t n, uint32_t c, uint32_t per,
                          const uint32_t* __restrict__ seg_off, uint4* __restrict__ segs) {
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (cls[v] != c) continue;
    const uint32_t a = in[v], b = end[v];
    uint32_t s = seg_off[v];
    for (uint32_t i = a; i < b; i += per) segs[s++] = make_uint4((uint32_t)v, i, min(i + per, b), 0);
  }
}

}  // namespace

int build_frontier(tc_graph& g, uint64_t e0, uint64_t e1, bool per_vertex, Frontier& fr) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const int dev = g.device;
  const uint32_t nn = n ? n : 1;
  int kl = 0;
  PhaseLog pl(s);
  const ItemGeom geo{g.off.get(), g.col.get(), g.src.get(), g.offH.get()};
  Sums* sums = g.scratch[kSlotSums].get<Sums>(1, s);  // read only for stats (read_frontier_sums)
  TC_CUDA(cudaMemsetAsync(sums, 0, sizeof(Sums), s));
  fr.sums = sums;
  uint32_t* cnt = g.scratch[kSlotCnt].get<uint32_t>(nn, s);  // scatter cursors, from in[v]
  fr.in = g.scratch[kSlotIn].get<uint32_t>((uint64_t)n + 1, s);
  fr.e0 = e0;
  fr.e1 = e1;
  kl += scan_exclusive<uint32_t>(InSlotsWhole{g.off.get(), g.deg.get()}, fr.in, n, fr.in + n, s);
  if (n) TC_CUDA(cudaMemcpyAsync(cnt, fr.in, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
  pl.mark("fr_slots");
  // per-vertex: the rows the part's edges come from (the whole graph: all
  // rows) and their mask blocks; one read for the item and mask-byte totals
  fr.mask_bytes = 0;
  fr.u_lo = 0;
  fr.u_hi = n ? n - 1 : 0;
  uint64_t rows = 0;
  if (per_vertex && e1 > e0) {
    if (e0 != 0 || e1 != g.E) {
      fr.u_lo = read_scalar(g.src.get() + e0, s);
      fr.u_hi = read_scalar(g.src.get() + e1 - 1, s);
    }
    rows = (uint64_t)fr.u_hi - fr.u_lo + 1;
    fr.rowbase = g.scratch[kSlotRowBase].get<uint64_t>(rows + 1, s);
    kl += scan_exclusive<uint64_t>(RowBytes{g.off.get(), g.offH.get(), fr.u_lo}, fr.rowbase, rows, fr.rowbase + rows,
                                   s);
  }
  uint32_t NI32 = 0;
  if (n) TC_CUDA(cudaMemcpyAsync(&NI32, fr.in + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  if (rows) TC_CUDA(cudaMemcpyAsync(&fr.mask_bytes, fr.rowbase + rows, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  const uint64_t NI = NI32;
  fr.nitems = NI;
  fr.items = g.scratch[kSlotItems].get<uint4>(NI * (per_vertex ? 2 : kItemStrideTotal), s);
  if (rows) fr.masks = g.scratch[kSlotMasks].get<uint8_t>(fr.mask_bytes + 32, s);
  pl.mark("fr_rowbase");
  if (NI) {
    const unsigned grid = grid_gs(ceil_div64(e1 - e0, kScatterR), dev);
    if (per_vertex)
      k_fr_scatter<true><<<grid, kT, 0, s>>>(geo, e0, e1, cnt, fr.items, fr.rowbase,
                                             fr.u_lo, fr.masks, sums);
    else
      k_fr_scatter<false><<<grid, kT, 0, s>>>(geo, e0, e1, cnt, fr.items, nullptr, 0,
                                              nullptr, sums);
    TC_LAUNCH();
    ++kl;
  }
  pl.mark("fr_scatter");
  // per-bin work segments
  {
    const PivotClass pc{g.off.get(), g.offH.get(), fr.in, cnt};
    // one offsets array, reused class by class (n can be 2^32 - 1)
    uint32_t* segoff = g.scratch[kSlotWoff].get<uint32_t>((uint64_t)nn + 1, s);
    const uint32_t per[3] = {kWarpSegItems, kCtaSegItems, kSmallItems};
    DBuf<uint32_t> tot(1, s);
    DBuf<unsigned long long> ctot(4, s);
    TC_CUDA(cudaMemsetAsync(ctot.get(), 0, 4 * sizeof(unsigned long long), s));
    uint8_t* cls = g.scratch[kSlotPacked].get<uint8_t>(nn, s);
    if (n) {
      k_fr_class<<<grid_gs(n, dev), kT, 0, s>>>(pc, n, cls, ctot.get());
      TC_LAUNCH();
      ++kl;
    }
    unsigned long long h[4] = {0, 0, 0, 0};
    TC_CUDA(cudaMemcpyAsync(h, ctot.get(), sizeof(h), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    const ScratchSlot slot[3] = {kSlotWsegs, kSlotCsegs, kSlotSsegs};
    uint64_t* nseg[3] = {&fr.nw, &fr.nc, &fr.ns};
    uint4** segs[3] = {&fr.wsegs, &fr.csegs, &fr.ssegs};
    for (int c = 0; c < 3; ++c) {
      *nseg[c] = h[c];
      *segs[c] = g.scratch[slot[c]].get<uint4>(*nseg[c], s);
      if (!*nseg[c]) continue;  // (empty classes: no scan, no fill)
      kl += scan_exclusive<uint32_t>(SegCountBin{cls, fr.in, cnt, (uint32_t)c + 1, per[c]}, segoff, n, tot.get(), s);
      k_fr_segs<<<grid_gs(n, dev), kT, 0, s>>>(cls, fr.in, cnt, n, (uint32_t)c + 1, per[c], segoff, *segs[c]);
      TC_LAUNCH();
      ++kl;
    }
    fr.pivots = h[3];
  }
  pl.mark("fr_segs");
  return kl;
}

void read_frontier_sums(Frontier& fr, cudaStream_t s) {
  const Sums hs = read_scalar(static_cast<const Sums*>(fr.sums), s);
  fr.W = hs.W;
  fr.J = hs.J;
  fr.hot = hs.hot;
  fr.items_c = hs.items_c;
  fr.nitems = hs.claims;  // this part's items (the slots of other parts' edges stay empty)
}

}  // namespace tcb
