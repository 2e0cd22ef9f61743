// common.cuh -- shared host/device plumbing for libtcb200.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <stdexcept>
#include <string>

#include "../../include/tcb200.h"

namespace tcb {

// Library-internal error; converted to a tc_status at the C boundary.
struct Error : std::runtime_error {
  tc_status code;
  Error(tc_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(tc_status c, const std::string& m) { throw Error(c, m); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const tc_status c = (e == cudaErrorMemoryAllocation) ? TC_ENOMEM : TC_ECUDA;
    fail(c, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                std::to_string(line) + ")");
  }
}
#define TC_CUDA(x) ::tcb::cuda_check((x), #x, __FILE__, __LINE__)
#define TC_LAUNCH() ::tcb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

// Caching device allocator (alloc.cu): freed blocks are kept per device and
// size class and handed back to the next request of the same class; a block
// reused on another stream first waits on the event recorded at its free.
// Repeated calls (a count per step, a graph per e2e step) therefore never
// remap device memory.
void* dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void* p, size_t bytes, cudaStream_t s);
// Return every cached (free) block of `device` (-1 = all devices) to
// cudaFree; returns the bytes released (tc_release_cached_memory).
size_t release_cached(int device);

// Stream-ordered device buffer on the caching allocator.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T) + 64, st));
  }
  void release() {
    if (p) dev_free(p, n * sizeof(T) + 64, s);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  T* get() const { return p; }
  operator T*() const { return p; }
};

// Diagnostics: TCB_PHASES=1 records a CUDA event at every mark() on the stream
// and prints the intervals to stderr when the log goes out of scope.
struct PhaseLog {
  static constexpr int kMax = 32;
  bool on = false;
  cudaStream_t s = nullptr;
  int n = 0;
  cudaEvent_t ev[kMax];
  const char* name[kMax];
  explicit PhaseLog(cudaStream_t st);
  void mark(const char* what);
  ~PhaseLog();
};

// Tuning / test knobs read from the environment (unset = default).
inline uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* v = getenv(name);
  return v ? (uint32_t)strtoul(v, nullptr, 10) : dflt;
}

inline unsigned ceil_div(uint64_t a, uint64_t b) { return (unsigned)((a + b - 1) / b); }
inline uint64_t ceil_div64(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

inline int bits_for(uint64_t max_value) {  // bits needed to represent values <= max_value
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b;
}

int num_sms(int device);

// ---- device helpers -------------------------------------------------------

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- bulk async copy (TMA, cp.async.bulk) + mbarrier, CTA scope ---------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Generic-proxy accesses of shared memory before this point are ordered
// before later async-proxy (bulk copy) writes to it.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// One thread: arm the barrier for `bytes` and start the bulk copy global ->
// shared (dst/src 16-byte aligned, bytes a multiple of 16); the TMA unit
// completes the transaction on the barrier when the bytes land.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* mbar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mbar))
               : "memory");
}
// One 256-bit store (STG.E.ENL2.256): a whole 32-byte sector, no partial write.
__device__ __forceinline__ void st256(void* p, const uint4& a, const uint4& b) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
               "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
// L2 prefetch of the line holding p (a hint: no completion, no register).
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
// TMA bulk prefetch of a global byte range into L2 (no SMEM, no completion
// to wait on): src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// The 16-byte aligned cover of [p, p + bytes) prefetched into L2.
__device__ __forceinline__ void prefetch_range_l2(const void* p, uint64_t bytes) {
  if (!bytes) return;
  const uint64_t a = reinterpret_cast<uint64_t>(p) & ~15ull;
  const uint64_t b = (reinterpret_cast<uint64_t>(p) + bytes + 15) & ~15ull;
  bulk_prefetch_l2(reinterpret_cast<const void*>(a), (uint32_t)(b - a));
}
// Ampere-style per-thread async copy (LDGSTS), 16 bytes, L1-bypassing.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Streaming (read-once) data, e.g. the in-edge item records of the warp and
// small bins: loaded with L2 evict-first (ld.global.cs) so a pass over them
// does not evict the adjacency the join probes.  Measured (profiles/README.md):
// C2 warp bin 0.679 -> 0.659 ms; the CTA bin (records staged per segment) is
// neutral and keeps plain loads.
#ifndef TCB_IREC_EF
#define TCB_IREC_EF 1
#endif
__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
#if TCB_IREC_EF
  return __ldcs(p);
#else
  return *p;
#endif
}
// Ampere-style per-thread async copy (LDGSTS), 8 bytes, L1-bypassing.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(unsigned long long* mbar, uint32_t parity) {
  const uint32_t a = smem_u32(mbar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (unsigned)o) v += t;
  }
  return v;
}

}  // namespace tcb
