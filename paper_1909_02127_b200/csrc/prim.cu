// prim.cu -- radix sort kernels (see prim.cuh).
#include "prim.cuh"

#ifndef TCB_RS_MATCH
#define TCB_RS_MATCH 0
#endif

namespace tcb {

int num_sms(int device) {
  int v = 0;
  TC_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

namespace {

// Lanes of the warp holding the same 8-bit digit as this lane (d = 256:
// invalid lane, never matched): eight ballots instead of a match_any, whose
// MIO-pipe cost bounded the passes (profiles/README.md).
__device__ __forceinline__ unsigned digit_peers(unsigned d) {
#if TCB_RS_MATCH
  return __match_any_sync(0xffffffffu, d);
#else
  unsigned peers = __ballot_sync(0xffffffffu, d < 256u);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return d < 256u ? peers : (1u << (threadIdx.x & 31u));
#endif
}

__global__ void __launch_bounds__(kRsThreads) k_rs_hist(const uint64_t* __restrict__ keys, uint64_t n,
                                                        int shift, uint32_t* __restrict__ hist,
                                                        uint32_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  const unsigned lane = lane_id();
#pragma unroll 4
  for (int it = 0; it < kRsKpt; ++it) {
    const uint64_t idx = base + (uint64_t)it * kRsThreads + threadIdx.x;
    const bool valid = idx < n;
    const unsigned d = valid ? (unsigned)((keys[idx] >> shift) & 255u) : 256u;
    const unsigned peers = digit_peers(d);
    if (valid && lane == (unsigned)(__ffs(peers) - 1)) atomicAdd(&h[d], (uint32_t)__popc(peers));
  }
  __syncthreads();
  hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kRsThreads) k_rs_scatter(const uint64_t* __restrict__ in,
                                                           uint64_t* __restrict__ out, uint64_t n,
                                                           int shift, const uint32_t* __restrict__ offs,
                                                           uint32_t ntiles) {
  __shared__ uint64_t stage[kRsTile];
  __shared__ uint32_t wh[kRsWarps][256];
  __shared__ uint32_t dstart[256];
  __shared__ uint32_t gofs[256];
  __shared__ uint32_t wtot[kRsWarps];

  const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
  const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
  const uint64_t wbase = base + (uint64_t)warp * kRsWarpKeys;

  uint64_t k[kRsKpt];
  unsigned d[kRsKpt];
#pragma unroll
  for (int it = 0; it < kRsKpt; ++it) {
    const uint64_t idx = wbase + (uint64_t)it * 32 + lane;
    const bool valid = idx < n;
    k[it] = valid ? in[idx] : 0ull;
    d[it] = valid ? (unsigned)((k[it] >> shift) & 255u) : 256u;
  }
#pragma unroll
  for (int w = 0; w < kRsWarps; ++w) wh[w][threadIdx.x] = 0;
  __syncthreads();

  // pass 1: per-warp digit counts, in key order (the peer masks are kept for
  // pass 2)
  unsigned pm[kRsKpt];
#pragma unroll
  for (int it = 0; it < kRsKpt; ++it) {
    pm[it] = digit_peers(d[it]);
    if (d[it] < 256u && lane == (unsigned)(__ffs(pm[it]) - 1)) wh[warp][d[it]] += __popc(pm[it]);
    __syncwarp();
  }
  __syncthreads();

  // per digit: warp-exclusive offsets, tile-local digit starts
  {
    const unsigned dg = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const uint32_t t = wh[w][dg];
      wh[w][dg] = run;
      run += t;
    }
    // block exclusive scan of run over the 256 digits
    uint32_t inc = warp_inclusive_scan(run);
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) wpre += (w < (int)warp) ? wtot[w] : 0u;
    const uint32_t ds = wpre + inc - run;
    dstart[dg] = ds;
    gofs[dg] = offs[(uint64_t)dg * ntiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) wh[w][dg] += ds;
  }
  __syncthreads();

  // pass 2: stable local ranks -> SMEM staging in tile-sorted order
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kRsKpt; ++it) {
    const unsigned peers = pm[it];
    if (d[it] < 256u) {
      const uint32_t pos = wh[warp][d[it]] + __popc(peers & lt);
      stage[pos] = k[it];
    }
    __syncwarp();
    if (d[it] < 256u && lane == (unsigned)(__ffs(peers) - 1)) wh[warp][d[it]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // pass 3: coalesced write-out, digit run by digit run
  const uint32_t cnt = (uint32_t)((n - base) < (uint64_t)kRsTile ? (n - base) : (uint64_t)kRsTile);
  for (uint32_t j = threadIdx.x; j < cnt; j += kRsThreads) {
    const uint64_t key = stage[j];
    const unsigned dg = (unsigned)((key >> shift) & 255u);
    out[(uint64_t)gofs[dg] + (j - dstart[dg])] = key;
  }
}

}  // namespace

uint64_t* radix_sort_u64(uint64_t* a, uint64_t* b, uint64_t n, int lo_bit, int hi_bit, cudaStream_t s) {
  if (n <= 1 || hi_bit <= lo_bit) return a;
  if (n >= (1ull << 32)) fail(TC_ERANGE, "radix_sort_u64: more than 2^32-1 keys");
  const uint32_t ntiles = (uint32_t)ceil_div64(n, kRsTile);
  DBuf<uint32_t> hist((uint64_t)ntiles * 256, s), offs((uint64_t)ntiles * 256, s);
  uint64_t* src = a;
  uint64_t* dst = b;
  for (int shift = lo_bit; shift < hi_bit; shift += 8) {
    k_rs_hist<<<ntiles, kRsThreads, 0, s>>>(src, n, shift, hist.get(), ntiles);
    TC_LAUNCH();
    scan_exclusive<uint32_t>(LoadArray<uint32_t>{hist.get()}, offs.get(), (uint64_t)ntiles * 256,
                             (uint32_t*)nullptr, s);
    k_rs_scatter<<<ntiles, kRsThreads, 0, s>>>(src, dst, n, shift, offs.get(), ntiles);
    TC_LAUNCH();
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

}  // namespace tcb
