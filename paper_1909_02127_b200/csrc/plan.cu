// plan.cu -- the level-1 frontier of one count as a work plan over |V|.
//
// The reference materialises level-1 rows (u, w) with expand_level
// (matcher.cpp:136-198: advance over N(u), accept w > u, 2-core membership,
// look-ahead) before its final level.  Here the level-1 rows of pivot v are
// exactly its in-edges u->v, which the graph holds grouped by head (the
// in-edge index ine, build.cu finish_graph), so the frontier of a count is
// only a plan: every pivot in the part's rank range [v_lo, v_hi) is
// classified (graph.cuh PivotClass) and cut into work segments {v, i0, i1}
// over its in-edge positions.  The joins compute each item's geometry when
// they stage the segment (count.cu).
//   k_plan_class   class + 1 per pivot (one byte)
//   two scans      segment offsets: warp|CTA packed in a u64, small in a u32
//   k_plan_segs    segment lists; the list lengths go to device memory
// No host synchronisation: list capacities are the graph's seg_cap.
#include <cstdio>
#include <cuda_runtime.h>

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

struct Sums {
  unsigned long long W, J, hot, items, pivots;
  unsigned long long cta_hot, cta_cold, cta_items, cta_mask, cta_seg_members, cta_segs;
  unsigned long long dense_items, dense_segs;
};

__global__ void k_plan_class(PivotClass pc, uint32_t v_lo, uint32_t v_hi, uint8_t* __restrict__ cls) {
  for (uint64_t v = v_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < v_hi;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t din = 0;
    cls[v - v_lo] = (uint8_t)(pc((uint32_t)v, din) + 1);
  }
}

// Segment counts of pivot v_lo + i: warp bin in the low 32 bits, CTA bin in
// the high 32 (SegWC); small bin (SegS).
struct SegWC {
  const uint8_t* cls;
  const uint32_t* inoff;
  uint32_t v_lo;
  __device__ __forceinline__ unsigned long long operator()(uint64_t i) const {
    const uint32_t c = cls[i];
    if (c != 1 && c != 2) return 0ull;
    const uint32_t din = inoff[v_lo + i + 1] - inoff[v_lo + i];
    return c == 1 ? (unsigned long long)((din + kWarpSegItems - 1) / kWarpSegItems)
                  : (unsigned long long)((din + kCtaSegItems - 1) / kCtaSegItems) << 32;
  }
};
struct SegS {
  const uint8_t* cls;
  __device__ __forceinline__ uint32_t operator()(uint64_t i) const { return cls[i] == 3 ? 1u : 0u; }
};

__global__ void k_plan_segs(const uint8_t* __restrict__ cls, const uint32_t* __restrict__ inoff, uint32_t v_lo,
                            uint32_t v_hi, const unsigned long long* __restrict__ off_wc,
                            const uint32_t* __restrict__ off_s, const unsigned long long* __restrict__ tot_wc,
                            const uint32_t* __restrict__ tot_s, uint4* __restrict__ wsegs, uint4* __restrict__ csegs,
                            uint4* __restrict__ ssegs, uint32_t* __restrict__ nseg) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    nseg[0] = (uint32_t)*tot_wc;
    nseg[1] = (uint32_t)(*tot_wc >> 32);
    nseg[2] = *tot_s;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (uint64_t)(v_hi - v_lo);
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = cls[i];
    if (c == 0) continue;
    const uint32_t v = v_lo + (uint32_t)i;
    const uint32_t a = inoff[v], b = inoff[v + 1];
    if (c == 3) {
      ssegs[off_s[i]] = make_uint4(v, a, b, 0);
      continue;
    }
    const uint32_t per = c == 1 ? kWarpSegItems : kCtaSegItems;
    uint4* out = c == 1 ? wsegs : csegs;
    uint32_t s = c == 1 ? (uint32_t)off_wc[i] : (uint32_t)(off_wc[i] >> 32);
    for (uint32_t j = a; j < b; j += per) out[s++] = make_uint4(v, j, min(j + per, b), 0);
  }
}

// Work counters of the part (stats only): per in-edge of the part's pivots
// its suffix length (J), hot share and usefulness (edge-parallel over the
// in-edge index), per pivot W = din * d+ (SURVEY 8d wedge stream) and
// whether it has work.
// k_join_cta's and k_join_dense's algorithmic work of the part (tc_count_stats
// cta_bytes / dense_bytes): per CTA-bin item its sparse hot and cold
// candidates and mask bytes, per CTA segment the pivot row it stages; dense
// items and segments.
__global__ void k_plan_work(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col, PivotClass pc,
                            const uint4* __restrict__ rowd, uint32_t r0, const uint32_t* __restrict__ inoff,
                            const uint4* __restrict__ irec, const uint32_t* __restrict__ dsoff, uint32_t v_lo,
                            uint32_t v_hi, Sums* __restrict__ sums) {
  unsigned long long W = 0, J = 0, H = 0, I = 0, P = 0;
  unsigned long long ch = 0, cc = 0, ci = 0, cm = 0, csm = 0, cs = 0, di = 0, ds = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t v = v_lo + t0; v < v_hi; v += stride) {
    const uint32_t dv = off[v + 1] - off[v], din = inoff[v + 1] - inoff[v];
    if (dsoff) ds += dsoff[v + 1] - dsoff[v];
    if (!dv || !din) continue;
    W += (unsigned long long)dv * din;
    ++P;
    uint32_t d2 = 0;
    if (pc((uint32_t)v, d2) == 1) {
      const uint32_t ns = (din + kCtaSegItems - 1) / kCtaSegItems;
      cs += ns;
      csm += (unsigned long long)ns * dv;
    }
  }
  const uint32_t i_lo = inoff[v_lo], i_hi = inoff[v_hi];
  for (uint64_t i = i_lo + t0; i < i_hi; i += stride) {
    const uint4 ax = irec[2 * (uint64_t)(i) + 1];
    const uint2 eu = make_uint2(ax.x, ax.y);
    const RowGeo rd = load_row(rowd, r0, eu.y);
    if (eu.x + 1 >= rd.end) continue;
    ++I;
    const uint32_t suf = rd.end - eu.x - 1, h = rd.h();
    J += suf;
    H += suf < h ? suf : h;
    if (rd.didx != kNoDense) ++di;
    uint32_t din = 0;
    if (pc(col[eu.x], din) == 1) {
      // the CTA bin's share: sparse hot part [hb, Ht) of colH, cold part
      const uint32_t a = eu.x + 1, ce = rd.cold_end();
      const uint32_t hb = a >= ce ? rd.O + (a - ce) : rd.O;
      if (rd.Ht > hb) {
        ch += rd.Ht - hb;
        cm += ((rd.Ht + 7) >> 3) - (hb >> 3);
      }
      if (ce > a) cc += ce - a;
      ++ci;
    }
  }
  unsigned long long* dst = &sums->W;
  unsigned long long vals[13] = {W, J, H, I, P, ch, cc, ci, cm, csm, cs, di, ds};
#pragma unroll
  for (int k = 0; k < 13; ++k) {
    const unsigned long long x = warp_sum(vals[k]);
    if (lane_id() == 0 && x) atomicAdd(dst + k, x);
  }
}

}  // namespace

int build_plan(tc_graph& g, uint32_t v_lo, uint32_t v_hi, bool per_vertex, bool masks, bool want_sums, Plan& p) {
  cudaStream_t s = g.stream;
  const uint32_t n = g.n;
  const int dev = g.device;
  int kl = 0;
  PhaseLog pl(s);
  v_lo = v_lo < g.r0 ? (g.r0 < v_hi ? g.r0 : v_hi) : v_lo;  // isolated ranks [0, r0) have no work
  p.v_lo = v_lo;
  p.v_hi = v_hi;
  p.core_words = g.core_words;
  const uint32_t np = v_hi - v_lo;
  p.nseg = g.scratch[kSlotCounters].get<uint32_t>(16, s);  // [0..3] segment counts, [4..11] join queues
  for (int c = 0; c < 3; ++c) p.cap[c] = g.seg_cap[c];
  p.wsegs = g.scratch[kSlotWsegs].get<uint4>(p.cap[0], s);
  p.csegs = g.scratch[kSlotCsegs].get<uint4>(p.cap[1], s);
  p.ssegs = g.scratch[kSlotSsegs].get<uint4>(p.cap[2], s);
  if (np == 0) {
    TC_CUDA(cudaMemsetAsync(p.nseg, 0, 4 * sizeof(uint32_t), s));
  } else {
    uint8_t* cls = g.scratch[kSlotCls].get<uint8_t>(np, s);
    // d+(v) = 0 pivots join the warp bin only to zero their items' mask bytes
    const PivotClass pc{g.off.get(), g.offH.get(), g.inoff.get(), masks};
    k_plan_class<<<grid_gs(np, dev), kT, 0, s>>>(pc, v_lo, v_hi, cls);
    TC_LAUNCH();
    ++kl;
    // [0, np) u64 warp|CTA offsets, then [np, 2np) u32 small offsets, totals at the end
    unsigned long long* off_wc = g.scratch[kSlotSegOff].get<unsigned long long>(2 * (uint64_t)np + 2, s);
    uint32_t* off_s = reinterpret_cast<uint32_t*>(off_wc + np);
    unsigned long long* tot_wc = off_wc + 2 * (uint64_t)np;
    uint32_t* tot_s = reinterpret_cast<uint32_t*>(off_wc + 2 * (uint64_t)np + 1);
    // the scans' workspace is handle scratch too: a count allocates nothing
    unsigned long long* ws = g.scratch[kSlotScanWs].get<unsigned long long>(scan_ws_elems(np) + 1, s);
    kl += scan_exclusive<unsigned long long>(SegWC{cls, g.inoff.get(), v_lo}, off_wc, np, tot_wc, s, ws);
    kl += scan_exclusive<uint32_t>(SegS{cls}, off_s, np, tot_s, s, reinterpret_cast<uint32_t*>(ws));
    k_plan_segs<<<grid_gs(np, dev), kT, 0, s>>>(cls, g.inoff.get(), v_lo, v_hi, off_wc, off_s, tot_wc, tot_s,
                                                p.wsegs, p.csegs, p.ssegs, p.nseg);
    TC_LAUNCH();
    ++kl;
  }
  pl.mark("plan_segs");
  p.masks = nullptr;
  (void)per_vertex;
  if (masks && n) p.masks = g.scratch[kSlotMasks].get<uint8_t>(g.mask_total + 32, s);
  p.sums = nullptr;
  if (want_sums) {
    Sums* sums = g.scratch[kSlotSums].get<Sums>(1, s);
    TC_CUDA(cudaMemsetAsync(sums, 0, sizeof(Sums), s));
    if (np) {
      k_plan_work<<<(unsigned)num_sms(dev) * 8, kT, 0, s>>>(
          g.off.get(), g.col.get(), PivotClass{g.off.get(), g.offH.get(), g.inoff.get(), masks}, g.rowd.get(), g.r0,
          g.inoff.get(), g.irec.get(), g.ndine ? g.dsoff.get() : nullptr, v_lo, v_hi, sums);
      TC_LAUNCH();
    }
    p.sums = sums;
  }
  return kl;
}

void read_plan_sums(Plan& p, cudaStream_t s) {
  if (!p.sums) return;
  Sums h;
  TC_CUDA(cudaMemcpyAsync(&h, p.sums, sizeof(Sums), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  if (getenv("TCB_PHASES"))
    fprintf(stderr,
            "[tcb] plan sums: W=%llu J=%llu hot=%llu items=%llu pivots=%llu cta_hot=%llu cta_cold=%llu "
            "cta_items=%llu cta_mask=%llu cta_seg_members=%llu cta_segs=%llu dense_items=%llu dense_segs=%llu\n",
            h.W, h.J, h.hot, h.items, h.pivots, h.cta_hot, h.cta_cold, h.cta_items, h.cta_mask, h.cta_seg_members,
            h.cta_segs, h.dense_items, h.dense_segs);
  p.W = h.W;
  p.J = h.J;
  p.hot = h.hot;
  p.items = h.items;
  p.pivots = h.pivots;
  p.cta_bytes = 2.0 * h.cta_hot + 4.0 * h.cta_cold + 32.0 * h.cta_items + (p.masks ? (double)h.cta_mask : 0.0) +
                4.0 * h.cta_seg_members + 16.0 * h.cta_segs;
  p.dense_bytes = (p.masks ? 8.0 : 4.0) * h.dense_items + 4.0 * p.core_words * h.dense_items +
                  (32.0 + 4.0 * p.core_words) * h.dense_segs;
}

}  // namespace tcb
