// gen.cu -- deterministic synthetic edge lists on the device.
//
// Counter-based splitmix64 streams: edge i depends only on i, so the device
// output is bit-identical to the host restatement in oracle/oracle.c for any
// launch shape.  RMAT/Kronecker use Graph500 (a,b,c) = (.57,.19,.19) with IEEE
// double compares (no FMA can contract a multiply by 2^-53 and a compare).
#include <cuda_runtime.h>

#include <vector>

#include "graph.cuh"

namespace tcb {
namespace {

__host__ __device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

__global__ void k_gen_rmat(int scale, uint64_t m, double A, double AB, double ABC, uint2* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t st = sm64(i * 0x100000001ull + 12345ull);
    uint32_t u = 0, v = 0;
    for (int b = 0; b < scale; ++b) {
      st = sm64(st);
      const double p = __dmul_rn((double)(st >> 11), 0x1.0p-53);
      const uint32_t ub = p > AB;
      const uint32_t vb = (p > A && p <= AB) || p > ABC;
      u |= ub << b;
      v |= vb << b;
    }
    out[i] = make_uint2(u, v);
  }
}

__global__ void k_gen_er(int scale, uint64_t m, uint2* __restrict__ out) {
  const uint64_t mask = (1ull << scale) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t st = sm64(i * 0x100000001ull + 12345ull);
    st = sm64(st);
    const uint32_t u = (uint32_t)(st & mask);
    st = sm64(st);
    const uint32_t v = (uint32_t)(st & mask);
    out[i] = make_uint2(u, v);
  }
}

__global__ void k_permute(uint32_t* __restrict__ a, uint64_t n, const uint32_t* __restrict__ perm) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = perm[a[i]];
}

}  // namespace

uint64_t gen_num_edges(int kind, int scale, int param) {
  if (scale < 1 || scale > 32 || param < 1) return 0;
  if (kind == 2) return ((uint64_t)param << scale) / 2;
  return (uint64_t)param << scale;
}

void generate(int kind, int scale, int param, uint32_t* d_pairs, cudaStream_t s) {
  if (kind < 0 || kind > 2) fail(TC_EINVAL, "tc_generate: kind must be 0 (RMAT), 1 (Kronecker) or 2 (ER)");
  if (scale < 1 || scale > 31 || param < 1) fail(TC_EINVAL, "tc_generate: scale in [1,31], param >= 1");
  const uint64_t m = gen_num_edges(kind, scale, param);
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div64(m, 256), (uint64_t)num_sms(dev) * 32);
  if (kind == 2) {
    k_gen_er<<<grid, 256, 0, s>>>(scale, m, reinterpret_cast<uint2*>(d_pairs));
  } else {
    const double A = .57, B = .19, C = .19;
    const double AB = A + B, ABC = AB + C;
    k_gen_rmat<<<grid, 256, 0, s>>>(scale, m, A, AB, ABC, reinterpret_cast<uint2*>(d_pairs));
  }
  TC_LAUNCH();
  if (kind == 1) {
    // Fisher-Yates label permutation: inherently sequential, done on the
    // host (n steps), applied on the device.
    const uint64_t n = 1ull << scale;
    std::vector<uint32_t> perm(n);
    for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    for (uint64_t i = n - 1; i >= 1; --i) {
      const uint64_t j = sm64(0xABCDEFull ^ i) % (i + 1);
      std::swap(perm[i], perm[j]);
    }
    DBuf<uint32_t> dperm(n, s);
    TC_CUDA(cudaMemcpyAsync(dperm.get(), perm.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    k_permute<<<grid, 256, 0, s>>>(d_pairs, 2 * m, dperm.get());
    TC_LAUNCH();
    TC_CUDA(cudaStreamSynchronize(s));
  }
}

}  // namespace tcb
