// prim.cuh -- hand-written device primitives for sm_100a: exclusive scan and
// an LSD radix sort of u64 keys.  These replace the reference's serial
// detail::exclusive_scan (frontier.hpp:80-89, the offsets/compaction step of
// advance/filter) and its per-vertex std::sort (graph.cpp:65).
#pragma once

#include "common.cuh"

namespace tcb {

// ---------------------------------------------------------------------------
// Exclusive scan: out[i] = sum_{j<i} load(j), optional grand total to d_total.
// Reduce-then-scan over 4096-element tiles (256 threads x 16 items), with the
// tile partials scanned recursively.  load is a device functor (index -> T), so
// predicates (unique flags, suffix lengths, ...) fuse into the scan read.
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ __forceinline__ T block_exclusive_scan(T v, T* block_total) {
  __shared__ T warp_tot[kScanThreads / 32];
  const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_inclusive_scan(v);
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kScanThreads / 32 ? warp_tot[lane] : T(0);
    T wi = warp_inclusive_scan(w);
    if (lane < kScanThreads / 32) warp_tot[lane] = wi - w;
    if (lane == kScanThreads / 32 - 1) *block_total = wi;
  }
  __syncthreads();
  T r = inc - v + warp_tot[warp];
  __syncthreads();
  return r;
}

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(Load load, uint64_t n, T* partial) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i)
    if (base + i < n) s += load(base + i);
  s = warp_sum(s);
  __shared__ T ws[kScanThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
    partial[blockIdx.x] = t;
  }
}

template <typename T, typename Load>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(Load load, T* out, uint64_t n,
                                                             const T* tile_offset, T* d_total) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? load(base + i) : T(0);
    s += v[i];
  }
  __shared__ T btot;
  T run = block_exclusive_scan(s, &btot);
  const T off = tile_offset ? tile_offset[blockIdx.x] : T(0);
  run += off;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (d_total && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *d_total = off + btot;
}

template <typename T>
struct LoadArray {
  const T* p;
  __device__ __forceinline__ T operator()(uint64_t i) const { return p[i]; }
};

// Workspace elements scan_exclusive needs for n elements (tile partials and
// their scans, recursively).
inline uint64_t scan_ws_elems(uint64_t n) {
  const uint64_t tiles = ceil_div64(n, kScanTile);
  return tiles <= 1 ? 0 : 2 * tiles + scan_ws_elems(tiles);
}

// Returns the number of kernels launched.  ws (optional, scan_ws_elems(n)
// elements): caller-owned workspace -- no allocation, so the scan can be
// captured into a CUDA graph (the count plan passes the handle's scratch).
template <typename T, typename Load>
int scan_exclusive(Load load, T* out, uint64_t n, T* d_total, cudaStream_t s, T* ws = nullptr) {
  if (n == 0) {
    if (d_total) TC_CUDA(cudaMemsetAsync(d_total, 0, sizeof(T), s));
    return 0;
  }
  const uint64_t tiles = ceil_div64(n, kScanTile);
  if (tiles == 1) {
    k_scan_tiles<T><<<1, kScanThreads, 0, s>>>(load, out, n, (const T*)nullptr, d_total);
    TC_LAUNCH();
    return 1;
  }
  DBuf<T> own;
  if (!ws) {
    own.alloc(scan_ws_elems(n), s);
    ws = own.get();
  }
  T* partial = ws;
  T* partial_scan = ws + tiles;
  k_scan_reduce<T><<<(unsigned)tiles, kScanThreads, 0, s>>>(load, n, partial);
  TC_LAUNCH();
  const int inner = scan_exclusive<T>(LoadArray<T>{partial}, partial_scan, tiles, (T*)nullptr, s, ws + 2 * tiles);
  k_scan_tiles<T><<<(unsigned)tiles, kScanThreads, 0, s>>>(load, out, n, partial_scan, d_total);
  TC_LAUNCH();
  return 2 + inner;
}

// ---------------------------------------------------------------------------
// LSD radix sort of u64 keys over bits [lo_bit, hi_bit), 8-bit digits.
// Per pass: per-tile digit histograms (match_any-aggregated SMEM counters) ->
// exclusive scan over the digit-major histogram table -> stable scatter: each
// warp ranks its 512 keys in order with __match_any_sync, the tile is
// re-ordered in SMEM, then written out digit-run by digit-run so global stores
// are coalesced.  Bits outside the range must be zero.  Keys < 2^32.
// Returns the buffer (a or b) that holds the sorted keys.
// ---------------------------------------------------------------------------
constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
#ifndef TCB_RS_KPT
#define TCB_RS_KPT 8
#endif
constexpr int kRsKpt = TCB_RS_KPT;               // keys per thread
constexpr int kRsTile = kRsThreads * kRsKpt;     // 4096 keys per tile
constexpr int kRsWarpKeys = 32 * kRsKpt;         // 512 keys per warp

uint64_t* radix_sort_u64(uint64_t* a, uint64_t* b, uint64_t n, int lo_bit, int hi_bit, cudaStream_t s);

}  // namespace tcb
