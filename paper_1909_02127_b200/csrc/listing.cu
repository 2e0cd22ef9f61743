// listing.cu -- triangle listings on the GPU: the rows
// count_triangles(keep_listings = true) returns (matcher.hpp:92,
// matcher.cpp:169-181, :295-296): every triangle once, as its three vertex ids
// in ascending order (the reference's UMO u < w < x).
//
// One warp per oriented edge u->v of the degree-ordered DAG (a CTA-free,
// output-bound pass, not the counting join): lanes take the suffix of N+(u)
// after v 32 at a time, binary-search each id in N+(v) (rows are sorted), and
// the hits of a step claim output rows with one warp-aggregated atomic.  Rows
// past the caller's capacity are counted but not written, so a first call
// with capacity 0 sizes the buffer.  Row order is unspecified (as the
// reference's is a property of its parallel schedule); each row is sorted.
//
// Streamed output: a triangle is listed from exactly one oriented edge (its
// lowest-ranked vertex u -> its middle one v), so edge ranges [e0, e1) of the
// oriented CSR partition the listing; a caller with a bounded buffer walks the
// edges range by range (tc_list_triangles_range).
#include <cuda_runtime.h>

#include "graph.cuh"

namespace tcb {
namespace {

__device__ __forceinline__ bool in_sorted(const uint32_t* __restrict__ a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo < n && a[lo] == x;
}

__global__ void __launch_bounds__(256) k_list(const uint32_t* __restrict__ off, const uint32_t* __restrict__ col,
                                              const uint32_t* __restrict__ src, const uint32_t* __restrict__ id_of,
                                              uint64_t e0, uint64_t e1, uint64_t cap, uint32_t* __restrict__ rows,
                                              unsigned long long* __restrict__ cursor) {
  const unsigned lane = lane_id();
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x / 32);
  for (uint64_t e = e0 + (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); e < e1; e += warps) {
    const uint32_t u = src[e], v = col[e];
    const uint32_t end = off[u + 1];
    const uint32_t vb = off[v], dv = off[v + 1] - vb;
    if (dv == 0) continue;
    const uint32_t iu = id_of[u], iv = id_of[v];
    for (uint32_t p0 = (uint32_t)e + 1; p0 < end; p0 += 32) {
      const uint32_t p = p0 + lane;
      uint32_t x = 0;
      bool hit = false;
      if (p < end) {
        x = col[p];
        hit = in_sorted(col + vb, dv, x);
      }
      const uint32_t m = __ballot_sync(0xffffffffu, hit);
      if (!m) continue;
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(cursor, (unsigned long long)__popc(m));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (hit) {
        const unsigned long long r = base + __popc(m & lanemask_lt());
        if (r < cap) {
          const uint32_t ix = id_of[x];
          uint32_t a = iu, b = iv, c = ix;  // sort the three ids
          if (a > b) { const uint32_t t = a; a = b; b = t; }
          if (b > c) { const uint32_t t = b; b = c; c = t; }
          if (a > b) { const uint32_t t = a; a = b; b = t; }
          rows[3 * r] = a;
          rows[3 * r + 1] = b;
          rows[3 * r + 2] = c;
        }
      }
    }
  }
}

}  // namespace

uint64_t list_triangles(tc_graph& g, uint32_t* d_rows, uint64_t cap, uint64_t e0, uint64_t e1) {
  cudaStream_t s = g.stream;
  DBuf<unsigned long long> cursor(1, s);
  TC_CUDA(cudaMemsetAsync(cursor.get(), 0, sizeof(unsigned long long), s));
  if (e1 > g.E) e1 = g.E;
  if (e0 < e1) {
    const unsigned grid = (unsigned)num_sms(g.device) * 8;
    k_list<<<grid, 256, 0, s>>>(g.off.get(), g.col.get(), g.src.get(), g.id_of.get(), e0, e1, cap, d_rows,
                                cursor.get());
    TC_LAUNCH();
  }
  unsigned long long T = 0;
  TC_CUDA(cudaMemcpyAsync(&T, cursor.get(), sizeof(T), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  return T;
}

}  // namespace tcb
