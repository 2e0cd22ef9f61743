// alloc.cu -- the caching device allocator behind DBuf (common.cuh).
//
// Size classes: 512-byte granules below 1 MiB, 2 MiB granules above.  A freed
// block keeps the stream it was last used on and an event recorded at the
// free; dev_alloc takes a cached block of the same class and device, making
// the new stream wait on that event when the streams differ.  On
// cudaErrorMemoryAllocation the cache is drained (device synchronised, every
// cached block returned) and the request retried once.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace tcb {
namespace {

struct Block {
  void* p;
  cudaStream_t s;
  cudaEvent_t ev;
};

struct Cache {
  std::mutex mu;
  std::map<std::pair<int, size_t>, std::vector<Block>> free;  // (device, class) -> blocks
};

Cache& cache() {
  static Cache* c = new Cache();  // never destroyed: blocks may outlive static teardown order
  return *c;
}

size_t size_class(size_t bytes) {
  const size_t g = bytes < (1u << 20) ? 512 : (2u << 20);
  return (bytes + g - 1) / g * g;
}

void drain_locked(Cache& c) {
  cudaDeviceSynchronize();
  for (auto& kv : c.free) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(kv.first.first);
    for (Block& b : kv.second) {
      cudaEventDestroy(b.ev);
      cudaFree(b.p);
    }
    cudaSetDevice(prev);
  }
  c.free.clear();
}

}  // namespace

void* dev_alloc(size_t bytes, cudaStream_t s) {
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  const size_t cls = size_class(bytes);
  Cache& c = cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free.find({dev, cls});
    if (it != c.free.end() && !it->second.empty()) {
      Block b = it->second.back();
      it->second.pop_back();
      if (b.s != s) TC_CUDA(cudaStreamWaitEvent(s, b.ev, 0));
      cudaEventDestroy(b.ev);
      return b.p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, cls);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(c.mu);
    drain_locked(c);
    e = cudaMalloc(&p, cls);
  }
  TC_CUDA(e);
  return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  Block b{p, s, nullptr};
  if (cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(b.ev, s) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamSynchronize(s);
    cudaFree(p);
    return;
  }
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  c.free[{dev, size_class(bytes)}].push_back(b);
}

}  // namespace tcb
