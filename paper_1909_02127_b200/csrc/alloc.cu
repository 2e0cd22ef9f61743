// alloc.cu -- the caching device allocator behind DBuf (common.cuh).
//
// Size classes: 512-byte granules below 1 MiB, 2 MiB granules above.  A freed
// block keeps the stream it was last used on and an event recorded at the
// free; dev_alloc takes the smallest cached block of a fitting class (the
// exact class below 1 MiB, up to 1.25x the request above: best fit, so a
// graph of another size still reuses the cache) on the same device, making the
// new stream wait on that event when the streams differ.  The real class of
// every live block is tracked, so a block handed out for a smaller request
// goes back under its own class.
//
// The cache is bounded: freed bytes above the per-device limit (TCB_CACHE_MB,
// default 40% of the device's memory) go straight back to cudaFree, oldest
// first, and tc_release_cached_memory() returns everything on demand -- a host
// framework in the same process (PyTorch) can always reclaim what the library
// is not using.  On cudaErrorMemoryAllocation the cache is drained (device
// synchronised, every cached block returned) and the request retried once.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <deque>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace tcb {
namespace {

struct Block {
  void* p;
  size_t cls;
  cudaStream_t s;
  cudaEvent_t ev;
  uint64_t seq;  // free order (oldest first when trimming)
};

struct DevCache {
  std::map<size_t, std::vector<Block>> free;  // class -> blocks
  size_t cached = 0;                          // bytes held in `free`
  size_t limit = 0;                           // 0 = not yet initialised
};

struct Cache {
  std::mutex mu;
  std::map<int, DevCache> dev;
  std::unordered_map<void*, size_t> live;  // pointer -> real class
  std::vector<void*> parked;  // freed inside a stream capture (dev_free)
  uint64_t seq = 0;
};

Cache& cache() {
  static Cache* c = new Cache();  // never destroyed: blocks may outlive static teardown order
  return *c;
}

size_t size_class(size_t bytes) {
  const size_t g = bytes < (1u << 20) ? 512 : (2u << 20);
  return (bytes + g - 1) / g * g;
}

size_t cache_limit(int dev) {
  if (const char* e = getenv("TCB_CACHE_MB")) return (size_t)strtoull(e, nullptr, 10) << 20;
  size_t fr = 0, tot = 0;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev);
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    tot = 0;
  }
  cudaSetDevice(prev);
  return tot ? tot / 5 * 2 : ((size_t)16 << 30);
}

void release_block(int dev, Block& b) {
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(dev);
  cudaEventSynchronize(b.ev);
  cudaEventDestroy(b.ev);
  cudaFree(b.p);
  cudaSetDevice(prev);
}

void drain_locked(Cache& c, int only_dev) {
  for (auto& d : c.dev) {
    if (only_dev >= 0 && d.first != only_dev) continue;
    for (auto& kv : d.second.free)
      for (Block& b : kv.second) release_block(d.first, b);
    d.second.free.clear();
    d.second.cached = 0;
  }
}

// Oldest cached blocks of the device back to cudaFree until the cache fits.
void trim_locked(Cache& c, int dev) {
  DevCache& d = c.dev[dev];
  while (d.cached > d.limit) {
    auto oldest = d.free.end();
    size_t idx = 0;
    uint64_t best = UINT64_MAX;
    for (auto it = d.free.begin(); it != d.free.end(); ++it)
      for (size_t i = 0; i < it->second.size(); ++i)
        if (it->second[i].seq < best) {
          best = it->second[i].seq;
          oldest = it;
          idx = i;
        }
    if (oldest == d.free.end()) break;
    Block b = oldest->second[idx];
    oldest->second.erase(oldest->second.begin() + idx);
    if (oldest->second.empty()) d.free.erase(oldest);
    d.cached -= b.cls;
    release_block(dev, b);
  }
}

}  // namespace

void* dev_alloc(size_t bytes, cudaStream_t s) {
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  const size_t cls = size_class(bytes);
  Cache& c = cache();
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (s && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
    fail(TC_ECUDA, "device allocation of " + std::to_string(bytes) +
                       " bytes inside a CUDA-graph capture (warm the handle up with one count first)");
  {
    std::lock_guard<std::mutex> lk(c.mu);
    if (!c.parked.empty()) {
      for (void* q : c.parked) cudaFree(q);
      c.parked.clear();
    }
    DevCache& d = c.dev[dev];
    const size_t max_cls = cls < (1u << 20) ? cls : cls + cls / 4;
    auto it = d.free.lower_bound(cls);
    if (it != d.free.end() && it->first <= max_cls && !it->second.empty()) {
      Block b = it->second.back();
      it->second.pop_back();
      if (it->second.empty()) d.free.erase(it);
      d.cached -= b.cls;
      if (b.s != s && cudaStreamWaitEvent(s, b.ev, 0) != cudaSuccess) {
        cudaGetLastError();  // the freeing stream's event is unusable: order by a device sync
        TC_CUDA(cudaDeviceSynchronize());
      }
      cudaEventDestroy(b.ev);
      c.live[b.p] = b.cls;
      return b.p;
    }
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, cls);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    std::lock_guard<std::mutex> lk(c.mu);
    cudaDeviceSynchronize();
    drain_locked(c, -1);
    e = cudaMalloc(&p, cls);
  }
  TC_CUDA(e);
  std::lock_guard<std::mutex> lk(c.mu);
  c.live[p] = cls;
  return p;
}

void dev_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  Cache& c = cache();
  size_t cls = size_class(bytes);
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.live.find(p);
    if (it != c.live.end()) {
      cls = it->second;
      c.live.erase(it);
    }
  }
  // A free inside a CUDA-graph capture (a count's scratch never reallocates
  // at steady state, so this is a caller error): the block cannot be
  // recycled through an event recorded into the capture; it is parked and
  // returned to the driver at the next allocation outside a capture.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (s && cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
    if (getenv("TCB_ALLOC_DEBUG")) fprintf(stderr, "[tcb] free of %zu bytes during stream capture (parked)\n", cls);
    std::lock_guard<std::mutex> lk(c.mu);
    c.parked.push_back(p);
    return;
  }
  cudaGetLastError();
  Block b{p, cls, s, nullptr, 0};
  if (cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventRecord(b.ev, s) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamSynchronize(s);
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lk(c.mu);
  DevCache& d = c.dev[dev];
  if (!d.limit) d.limit = cache_limit(dev);
  b.seq = ++c.seq;
  d.free[cls].push_back(b);
  d.cached += cls;
  if (d.cached > d.limit) trim_locked(c, dev);
}

size_t release_cached(int device) {
  Cache& c = cache();
  std::lock_guard<std::mutex> lk(c.mu);
  size_t n = 0;
  for (auto& d : c.dev)
    if (device < 0 || d.first == device) n += d.second.cached;
  drain_locked(c, device);
  return n;
}

}  // namespace tcb
