// feed.cu -- host->device feed of the CSR neighbour array in pieces, for the
// build that orients and sorts the rows of each piece as soon as it lands
// (build.cu build_from_csr, tc_graph_from_csr with host arrays).
//
// Pinned sources (cudaHostAlloc / cudaHostRegister / torch pin_memory): one
// DMA per piece on a side stream, issued a few pieces ahead.
// Pageable sources (the reference's Graph holds std::vectors): the driver's
// own pageable path measured ~5x below the link (202 vs 42 ms for C4's 2.1 GB),
// so worker threads copy pieces into pinned bounce slots (two per worker,
// process-wide, reused across calls) and DMA from there on their own streams;
// host memcpy of piece k+W overlaps the DMA of piece k.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "graph.cuh"

namespace tcb {

bool pageable_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

namespace {

// Process-wide pinned bounce slots (grow-only); one feed uses them at a time.
struct Slots {
  std::mutex use;  // held by the feed that owns the slots
  std::vector<void*> p;
  size_t bytes = 0;
  void ensure(size_t n_slots, size_t slot_bytes) {
    if (p.size() >= n_slots && bytes >= slot_bytes) return;
    for (void* q : p) cudaFreeHost(q);
    p.assign(n_slots, nullptr);
    bytes = slot_bytes;
    for (auto& q : p) TC_CUDA(cudaHostAlloc(&q, slot_bytes, cudaHostAllocDefault));
  }
};
Slots& slots() {
  static Slots* s = new Slots();  // never destroyed (pinned memory outlives static teardown)
  return *s;
}

}  // namespace

PieceFeed::PieceFeed(const uint32_t* h, uint32_t* d, uint64_t total, uint64_t piece, cudaStream_t after)
    : h_(h), d_(d), total_(total), piece_(piece) {
  K_ = (uint32_t)((total + piece - 1) / piece);
  pageable_ = pageable_host(h);
  TC_CUDA(cudaGetDevice(&dev_));  // (worker threads start on device 0)
  ev_.assign(K_, nullptr);
  for (auto& e : ev_) TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cudaEvent_t ready;  // the destination was allocated on `after`
  TC_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  TC_CUDA(cudaEventRecord(ready, after));
  const uint32_t hw = std::max(2u, std::thread::hardware_concurrency());
  W_ = pageable_ ? std::min<uint32_t>({8u, hw / 2, K_}) : 1u;
  if (W_ < 1) W_ = 1;
  streams_.assign(W_, nullptr);
  for (auto& st : streams_) {
    TC_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    TC_CUDA(cudaStreamWaitEvent(st, ready, 0));
  }
  TC_CUDA(cudaEventDestroy(ready));
  if (!pageable_) {
    issue(2);
    return;
  }
  lock_ = std::unique_lock<std::mutex>(slots().use);
  slots().ensure(2 * (size_t)W_, (size_t)piece * sizeof(uint32_t));
  slot_done_.assign(2 * (size_t)W_, nullptr);
  for (auto& e : slot_done_) TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  recorded_.assign(K_, 0);
  for (uint32_t t = 0; t < W_; ++t) workers_.emplace_back([this, t] { work(t); });
}

// pinned: DMA pieces [issued_, upto) straight from the caller's buffer
void PieceFeed::issue(uint32_t upto) {
  for (; issued_ < upto && issued_ < K_; ++issued_) {
    const uint64_t a = (uint64_t)issued_ * piece_, b = std::min(total_, a + piece_);
    TC_CUDA(cudaMemcpyAsync(d_ + a, h_ + a, (b - a) * sizeof(uint32_t), cudaMemcpyHostToDevice, streams_[0]));
    TC_CUDA(cudaEventRecord(ev_[issued_], streams_[0]));
  }
}

// pageable: worker t stages pieces t, t+W, ... through slots t and t+W
void PieceFeed::work(uint32_t t) {
  try {
    TC_CUDA(cudaSetDevice(dev_));
    for (uint32_t k = t; k < K_ && !abort_; k += W_) {
      const size_t sl = k % (2 * W_);
      void* buf = slots().p[sl];
      TC_CUDA(cudaEventSynchronize(slot_done_[sl]));  // the slot's previous DMA has drained
      const uint64_t a = (uint64_t)k * piece_, b = std::min(total_, a + piece_);
      std::memcpy(buf, h_ + a, (b - a) * sizeof(uint32_t));
      TC_CUDA(cudaMemcpyAsync(d_ + a, buf, (b - a) * sizeof(uint32_t), cudaMemcpyHostToDevice, streams_[t]));
      TC_CUDA(cudaEventRecord(slot_done_[sl], streams_[t]));
      TC_CUDA(cudaEventRecord(ev_[k], streams_[t]));
      {
        std::lock_guard<std::mutex> lk(mu_);
        recorded_[k] = 1;
      }
      cv_.notify_all();
    }
  } catch (...) {
    std::lock_guard<std::mutex> lk(mu_);
    if (!err_) err_ = std::current_exception();
    cv_.notify_all();
  }
}

void PieceFeed::wait_piece(uint32_t k, cudaStream_t s) {
  if (!pageable_) {
    issue(k + 3);
  } else {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return recorded_[k] || err_; });
    if (err_) std::rethrow_exception(err_);
  }
  TC_CUDA(cudaStreamWaitEvent(s, ev_[k], 0));
}

// Large host<->device copies of pageable buffers (the offsets of a host CSR,
// per-vertex counts and exported CSR arrays into numpy / std::vector memory)
// through the same pinned bounce slots: worker t moves chunks t, t+W, ...,
// each chunk's host memcpy overlapping the other workers' DMAs on their own
// streams (the driver's pageable path runs several times below the link).
// Synchronous: returns when the host buffer (d2h) or the device buffer (h2d)
// holds the data; small or pinned buffers take one cudaMemcpyAsync on s.
namespace {
constexpr size_t kBounceMin = 16u << 20;    // below: the driver's own path
constexpr size_t kBounceChunk = 32u << 20;  // bytes per chunk = the pageable feed's slot size (one slot allocation serves both)

void bounce(void* dst, const void* src, size_t bytes, bool h2d, cudaStream_t s) {
  const size_t K = (bytes + kBounceChunk - 1) / kBounceChunk;
  const uint32_t hw = std::max(2u, std::thread::hardware_concurrency());
  const uint32_t W = (uint32_t)std::max<size_t>(1, std::min<size_t>({8u, hw / 2, K}));
  int dev = 0;
  TC_CUDA(cudaGetDevice(&dev));
  std::unique_lock<std::mutex> lock(slots().use);
  slots().ensure(2 * (size_t)W, kBounceChunk);
  cudaEvent_t ready;
  TC_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  TC_CUDA(cudaEventRecord(ready, s));  // d2h: the producer's work; h2d: the destination's allocation
  std::vector<cudaStream_t> st(W, nullptr);
  for (auto& x : st) {
    TC_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    TC_CUDA(cudaStreamWaitEvent(x, ready, 0));
  }
  std::exception_ptr err;
  std::mutex emu;
  std::vector<std::thread> th;
  for (uint32_t t = 0; t < W; ++t)
    th.emplace_back([&, t] {
      try {
        TC_CUDA(cudaSetDevice(dev));
        cudaEvent_t done[2];
        for (auto& e : done) TC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        bool used[2] = {false, false};
        uint32_t j = 0;  // this worker's chunk counter (slot = j & 1)
        for (size_t k = t; k < K; k += W, ++j) {
          void* buf = slots().p[2 * t + (j & 1)];
          const size_t a = k * kBounceChunk, n = std::min(bytes, a + kBounceChunk) - a;
          if (h2d) {
            if (used[j & 1]) TC_CUDA(cudaEventSynchronize(done[j & 1]));  // the slot's last DMA drained
            std::memcpy(buf, static_cast<const char*>(src) + a, n);
            TC_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + a, buf, n, cudaMemcpyHostToDevice, st[t]));
            TC_CUDA(cudaEventRecord(done[j & 1], st[t]));
            used[j & 1] = true;
          } else {
            TC_CUDA(cudaMemcpyAsync(buf, static_cast<const char*>(src) + a, n, cudaMemcpyDeviceToHost, st[t]));
            TC_CUDA(cudaStreamSynchronize(st[t]));
            std::memcpy(static_cast<char*>(dst) + a, buf, n);
          }
        }
        TC_CUDA(cudaStreamSynchronize(st[t]));
        for (auto& e : done) cudaEventDestroy(e);
      } catch (...) {
        std::lock_guard<std::mutex> lk(emu);
        if (!err) err = std::current_exception();
      }
    });
  for (auto& x : th) x.join();
  for (auto& x : st) cudaStreamDestroy(x);
  cudaEventDestroy(ready);
  if (err) std::rethrow_exception(err);
}
}  // namespace

void copy_h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
  if (bytes < kBounceMin || !pageable_host(h)) {
    TC_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    return;
  }
  bounce(d, h, bytes, true, s);
}

void copy_d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
  if (bytes < kBounceMin || !pageable_host(h)) {
    TC_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
    return;
  }
  bounce(h, d, bytes, false, s);
}

PieceFeed::~PieceFeed() {  // an error path may leave pieces in flight into the caller's buffers
  abort_ = true;
  for (auto& w : workers_) w.join();
  for (cudaStream_t st : streams_)
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  for (cudaEvent_t e : ev_)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : slot_done_)
    if (e) cudaEventDestroy(e);
}

}  // namespace tcb
