// multi.cu -- the multi-GPU count behind the C-ABI (SURVEY 8e, 8b tc_count_multi).
//
// The oriented graph is replicated on every GPU (each builds it from the same
// edge list or CSR: no communication).  Part p of P counts the triangles whose
// middle vertex has rank in its degree-weighted range (count.cu
// partition_bounds), then ONE ncclAllReduce(ncclUint64, ncclSum) of the
// [per-vertex | total] buffer combines the parts on the count stream -- the
// only exchange the path has.  Two launch shapes, the same kernels:
//   tc_comm_init_rank + tc_count_allreduce   one process per GPU (torchrun
//       style; the host framework passes the 128-byte NCCL id around)
//   tc_multi_create  + tc_count_multi        one process driving every GPU
//       (ncclCommInitAll over the distinct devices, one stream per GPU).  A
//       device listed more than once runs its parts back to back and sums them
//       locally before the allreduce, so a P-part split is testable on 1 GPU.
//
// NCCL is bound at first use (dlopen of libnccl.so.2, or $TCB_NCCL_LIB), not
// at link time: libtcb200.so loaded before a host framework that ships its own
// libnccl.so.2 (PyTorch) must not pin the system copy under that soname, and
// single-GPU users need no NCCL at all.  When the framework has already loaded
// its NCCL, dlopen returns that same library, so both share one NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <map>
#include <mutex>
#include <vector>

#include "graph.cuh"

struct tc_comm {
  ncclComm_t comm = nullptr;
  int device = 0, rank = 0, nranks = 1;
  tcb::DBuf<uint64_t> buf;  // [per-vertex n | total]
  std::mutex mu;
};

struct tc_multi {
  std::vector<int> part_dev;   // device of part p
  std::vector<int> udev;       // distinct devices, comm order
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;  // one per distinct device
  std::vector<tcb::DBuf<uint64_t>> acc, tmp;
  std::mutex mu;
};

namespace tcb {
namespace {

// The NCCL entry points this file uses, resolved once.
struct NcclApi {
  decltype(&::ncclGetErrorString) GetErrorString = nullptr;
  decltype(&::ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&::ncclCommInitRank) CommInitRank = nullptr;
  decltype(&::ncclCommInitAll) CommInitAll = nullptr;
  decltype(&::ncclCommDestroy) CommDestroy = nullptr;
  decltype(&::ncclAllReduce) AllReduce = nullptr;
  decltype(&::ncclGroupStart) GroupStart = nullptr;
  decltype(&::ncclGroupEnd) GroupEnd = nullptr;
  std::string error;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("TCB_NCCL_LIB");
    const char* name = env && *env ? env : "libnccl.so.2";
    void* h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      a.error = std::string("cannot load NCCL (") + name + "): " + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fp, const char* s) {
      fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, s));
      if (!fp && a.error.empty()) a.error = std::string("NCCL symbol missing: ") + s;
    };
    sym(a.GetErrorString, "ncclGetErrorString");
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    return a;
  }();
  if (!api.error.empty()) fail(TC_ENCCL, api.error);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(TC_ENCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

__global__ void k_add_u64(uint64_t* __restrict__ a, const uint64_t* __restrict__ b, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] += b[i];
}

struct Dev {
  int prev = 0;
  explicit Dev(int d) {
    TC_CUDA(cudaGetDevice(&prev));
    TC_CUDA(cudaSetDevice(d));
  }
  ~Dev() { cudaSetDevice(prev); }
};

}  // namespace

// One part's count into buf = [per-vertex n | total] on g's stream.
static void count_part(tc_graph& g, const tc_count_opts& o, uint32_t part, uint32_t parts, bool pv, uint64_t* buf,
                       tc_count_stats* st) {
  tc_count_opts q = o;
  q.part_index = part;
  q.part_count = parts;
  std::lock_guard<std::mutex> lk(g.mu);
  count_triangles(g, q, buf + g.n, pv ? buf : nullptr, st);
}

void comm_unique_id(void* id) {
  ncclUniqueId u;
  nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
}

tc_comm* comm_init_rank(const void* id, int nranks, int rank, int device) {
  Dev d(device);
  auto* c = new tc_comm();
  c->device = device;
  c->rank = rank;
  c->nranks = nranks;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  const ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    nccl_check(r, "ncclCommInitRank");
  }
  return c;
}

void comm_destroy(tc_comm* c) {
  if (!c) return;
  {
    Dev d(c->device);
    cudaDeviceSynchronize();
    c->buf.release();
    if (c->comm) nccl().CommDestroy(c->comm);
  }
  delete c;
}

void count_allreduce(tc_comm* c, tc_graph& g, const tc_count_opts& o, uint64_t* d_total, uint64_t* d_pv,
                     tc_count_stats* st) {
  if (g.device != c->device) fail(TC_EINVAL, "tc_count_allreduce: graph and communicator on different devices");
  std::lock_guard<std::mutex> lk(c->mu);
  Dev d(c->device);
  cudaStream_t s = g.stream;
  const bool pv = d_pv != nullptr;
  const uint64_t cnt = (uint64_t)g.n + 1;
  if (c->buf.n < cnt) c->buf.alloc(cnt, s);
  c->buf.s = s;
  uint64_t* buf = c->buf.get();
  count_part(g, o, (uint32_t)c->rank, (uint32_t)c->nranks, pv, buf, st);
  // the one exchange: per-vertex + total (or the total alone), on the count stream
  if (pv)
    nccl_check(nccl().AllReduce(buf, buf, cnt, ncclUint64, ncclSum, c->comm, s), "ncclAllReduce");
  else
    nccl_check(nccl().AllReduce(buf + g.n, buf + g.n, 1, ncclUint64, ncclSum, c->comm, s), "ncclAllReduce");
  TC_CUDA(cudaMemcpyAsync(d_total, buf + g.n, sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
  if (pv && g.n) TC_CUDA(cudaMemcpyAsync(d_pv, buf, sizeof(uint64_t) * g.n, cudaMemcpyDeviceToDevice, s));
}

tc_multi* multi_create(const int* devices, int nparts) {
  auto* m = new tc_multi();
  m->part_dev.assign(devices, devices + nparts);
  for (int p = 0; p < nparts; ++p)
    if (std::find(m->udev.begin(), m->udev.end(), devices[p]) == m->udev.end()) m->udev.push_back(devices[p]);
  const int nd = (int)m->udev.size();
  m->comms.resize(nd, nullptr);
  const ncclResult_t r = nccl().CommInitAll(m->comms.data(), nd, m->udev.data());
  if (r != ncclSuccess) {
    delete m;
    nccl_check(r, "ncclCommInitAll");
  }
  m->streams.resize(nd, nullptr);
  m->acc.resize(nd);
  m->tmp.resize(nd);
  for (int i = 0; i < nd; ++i) {
    Dev d(m->udev[i]);
    TC_CUDA(cudaStreamCreateWithFlags(&m->streams[i], cudaStreamNonBlocking));
  }
  return m;
}

void multi_destroy(tc_multi* m) {
  if (!m) return;
  for (size_t i = 0; i < m->udev.size(); ++i) {
    Dev d(m->udev[i]);
    cudaStreamSynchronize(m->streams[i]);
    m->acc[i].release();
    m->tmp[i].release();
    if (m->comms[i]) nccl().CommDestroy(m->comms[i]);
    cudaStreamDestroy(m->streams[i]);
  }
  delete m;
}

int multi_parts(const tc_multi* m) { return (int)m->part_dev.size(); }
int multi_part_device(const tc_multi* m, int p) { return m->part_dev[p]; }

// graphs[p] lives on part_dev[p] (the same handle may serve several parts of
// one device).  Outputs (device pointers on part 0's device) are final on
// return of the stream work; stats (nullable) = part 0's, total_ms = slowest part.
void count_multi(tc_multi* m, tc_graph* const* graphs, const tc_count_opts& o, uint64_t* d_total, uint64_t* d_pv,
                 tc_count_stats* st) {
  std::lock_guard<std::mutex> lk(m->mu);
  const int P = (int)m->part_dev.size(), nd = (int)m->udev.size();
  const uint32_t n = graphs[0]->n;
  for (int p = 0; p < P; ++p) {
    if (graphs[p]->device != m->part_dev[p]) fail(TC_EINVAL, "tc_count_multi: graph not on its part's device");
    if (graphs[p]->n != n || graphs[p]->E != graphs[0]->E)
      fail(TC_EINVAL, "tc_count_multi: the graphs are not replicas of one graph");
  }
  const bool pv = d_pv != nullptr;
  const uint64_t cnt = (uint64_t)n + 1;
  double max_ms = 0;
  std::vector<cudaEvent_t> evs;
  for (int i = 0; i < nd; ++i) {
    Dev d(m->udev[i]);
    cudaStream_t ds = m->streams[i];
    if (m->acc[i].n < cnt) m->acc[i].alloc(cnt, ds);
    bool first = true;
    for (int p = 0; p < P; ++p) {
      if (m->part_dev[p] != m->udev[i]) continue;
      tc_graph& g = *graphs[p];
      // the graph's stream waits for the device stream (acc / tmp reuse), counts, and hands back
      cudaEvent_t e0, e1;
      TC_CUDA(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
      TC_CUDA(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
      evs.push_back(e0);
      evs.push_back(e1);
      TC_CUDA(cudaEventRecord(e0, ds));
      TC_CUDA(cudaStreamWaitEvent(g.stream, e0, 0));
      uint64_t* out = m->acc[i].get();
      if (!first) {
        if (m->tmp[i].n < cnt) m->tmp[i].alloc(cnt, ds);
        out = m->tmp[i].get();
      }
      tc_count_stats ps{};
      count_part(g, o, (uint32_t)p, (uint32_t)P, pv, out, st ? &ps : nullptr);
      if (st) {
        if (p == 0) *st = ps;
        max_ms = std::max(max_ms, ps.total_ms);
      }
      TC_CUDA(cudaEventRecord(e1, g.stream));
      TC_CUDA(cudaStreamWaitEvent(ds, e1, 0));
      if (!first) {
        const uint64_t off = pv ? 0 : n;  // without per-vertex counts only the total is live
        k_add_u64<<<num_sms(m->udev[i]) * 4, 256, 0, ds>>>(m->acc[i].get() + off, m->tmp[i].get() + off, cnt - off);
        TC_LAUNCH();
      }
      first = false;
    }
  }
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (int i = 0; i < nd; ++i) {
    Dev d(m->udev[i]);
    uint64_t* a = pv ? m->acc[i].get() : m->acc[i].get() + n;  // [per-vertex | total] or the total alone
    nccl_check(nccl().AllReduce(a, a, pv ? cnt : 1, ncclUint64, ncclSum, m->comms[i], m->streams[i]), "ncclAllReduce");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  // part 0's device holds the result
  const int i0 = (int)(std::find(m->udev.begin(), m->udev.end(), m->part_dev[0]) - m->udev.begin());
  {
    Dev d(m->udev[i0]);
    cudaStream_t ds = m->streams[i0];
    TC_CUDA(cudaMemcpyAsync(d_total, m->acc[i0].get() + n, sizeof(uint64_t), cudaMemcpyDeviceToDevice, ds));
    if (pv && n) TC_CUDA(cudaMemcpyAsync(d_pv, m->acc[i0].get(), sizeof(uint64_t) * n, cudaMemcpyDeviceToDevice, ds));
    TC_CUDA(cudaStreamSynchronize(ds));
  }
  for (int i = 0; i < nd; ++i) {
    Dev d(m->udev[i]);
    TC_CUDA(cudaStreamSynchronize(m->streams[i]));
  }
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  if (st) st->total_ms = max_ms;
}

}  // namespace tcb
