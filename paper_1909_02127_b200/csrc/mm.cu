// mm.cu -- MatrixMarket entry tokenizer on the GPU: the
// bulk of parse_matrix_market (io.cpp:124-158) for load_graph, so a text file
// goes host bytes -> device -> EdgeList -> device graph without a host pass
// over the entries.
//
// The banner and size line are parsed on the host (io_host.cpp
// parse_mm_header, a few bytes).  The entry body, on the device:
//   k_mm_block_lines   lines starting in each 4 KiB block of the body
//   scan               -> block line offsets
//   k_mm_line_starts   byte offset of every line (getline semantics: split at
//                      '\n'; a final '\n' does not start an empty line)
//   k_mm_parse         one thread per line: trim, skip blank and '%' lines,
//                      two whitespace-separated decimal u64 tokens (the
//                      from_chars rules: digits only, no sign, overflow is an
//                      error), the declared-range check; trailing fields are
//                      ignored -- status per line
//   scan               -> entry index per line
//   k_mm_emit          the first nnz entries -> 0-based (i, j) pairs; records
//                      the line of the nnz-th entry and the first bad line
// Any malformed input (a bad line before the nnz-th entry, non-comment
// content after it, fewer than nnz entries) is reported by re-running the
// host parser, which throws the reference's exact ParseError and line.
#include <cuda_runtime.h>

#include "graph.cuh"
#include "io_host.h"
#include "prim.cuh"

namespace tcb {
namespace {

constexpr uint32_t kBlockBytes = 4096;
constexpr int kT = 256;

__device__ __forceinline__ bool mm_space(unsigned char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// number of line starts in block b: byte i starts a line iff i == 0 or
// t[i-1] == '\n' (and i < len)
__global__ void k_mm_block_lines(const unsigned char* __restrict__ t, uint64_t len, uint32_t* __restrict__ cnt) {
  const uint64_t b = blockIdx.x;
  const uint64_t base = b * kBlockBytes;
  uint32_t c = 0;
  for (uint32_t k = threadIdx.x; k < kBlockBytes; k += blockDim.x) {
    const uint64_t i = base + k;
    if (i < len && (i == 0 || t[i - 1] == '\n')) ++c;
  }
  c = warp_sum(c);
  __shared__ uint32_t ws[kT / 32];
  if (lane_id() == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kT / 32; ++w) s += ws[w];
    cnt[b] = s;
  }
}

// line start offsets, in order (block-local ballot ranks + block offsets)
__global__ void k_mm_line_starts(const unsigned char* __restrict__ t, uint64_t len,
                                 const uint32_t* __restrict__ boff, uint64_t* __restrict__ starts) {
  const uint64_t b = blockIdx.x;
  const uint64_t base = b * kBlockBytes;
  __shared__ uint32_t s_run;
  __shared__ uint32_t ws[kT / 32];
  if (threadIdx.x == 0) s_run = boff[b];
  __syncthreads();
  for (uint32_t k0 = 0; k0 < kBlockBytes; k0 += kT) {
    const uint64_t i = base + k0 + threadIdx.x;
    const bool st = i < len && (i == 0 || t[i - 1] == '\n');
    const uint32_t m = __ballot_sync(0xffffffffu, st);
    if (lane_id() == 0) ws[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int w = 0; w < kT / 32; ++w) {
      before += (w < (int)(threadIdx.x >> 5)) ? ws[w] : 0u;
      tot += ws[w];
    }
    if (st) starts[s_run + before + __popc(m & lanemask_lt())] = i;
    __syncthreads();
    if (threadIdx.x == 0) s_run += tot;
    __syncthreads();
  }
}

// per line: 0 blank/comment, 1 entry (i, j returned), 2 malformed
__global__ void k_mm_parse(const unsigned char* __restrict__ t, uint64_t len, const uint64_t* __restrict__ starts,
                           uint64_t nlines, uint64_t rows, uint64_t cols, uint8_t* __restrict__ status,
                           uint2* __restrict__ ij) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t p = starts[k];
    const uint64_t e = (k + 1 < nlines) ? starts[k + 1] : len;  // includes the '\n'
    while (p < e && mm_space(t[p])) ++p;
    if (p >= e || t[p] == '%') {
      status[k] = 0;
      continue;
    }
    uint64_t v[2] = {0, 0};
    bool ok = true;
    int ntok = 0;
    while (ntok < 2 && p < e && ok) {
      uint64_t x = 0;
      bool any = false;
      while (p < e && !mm_space(t[p])) {
        const unsigned c = t[p];
        if (c < '0' || c > '9') {
          ok = false;
          break;
        }
        if (x > (0xFFFFFFFFFFFFFFFFull - (c - '0')) / 10) {  // from_chars: result_out_of_range
          ok = false;
          break;
        }
        x = x * 10 + (c - '0');
        any = true;
        ++p;
      }
      if (!ok || !any) break;
      v[ntok++] = x;
      while (p < e && mm_space(t[p])) ++p;
    }
    if (!ok || ntok < 2 || v[0] < 1 || v[0] > rows || v[1] < 1 || v[1] > cols) {
      status[k] = 2;
      continue;
    }
    status[k] = 1;
    ij[k] = make_uint2((uint32_t)(v[0] - 1), (uint32_t)(v[1] - 1));
  }
}

struct IsEntry {
  const uint8_t* status;
  __device__ __forceinline__ uint64_t operator()(uint64_t k) const { return status[k] == 1 ? 1ull : 0ull; }
};

// res[0] = line of the nnz-th entry (or ~0), res[1] = first malformed line
// before it, res[2] = first non-blank line after it
__global__ void k_mm_emit(const uint8_t* __restrict__ status, const uint2* __restrict__ ij,
                          const uint64_t* __restrict__ eidx, uint64_t nlines, uint64_t nnz,
                          uint32_t* __restrict__ pairs, unsigned long long* __restrict__ res) {
  for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t st = status[k];
    if (st == 1) {
      const uint64_t x = eidx[k];
      if (x < nnz) {
        pairs[2 * x] = ij[k].x;
        pairs[2 * x + 1] = ij[k].y;
      }
      if (x + 1 == nnz) atomicMin(&res[0], (unsigned long long)k);
    }
    if (st == 2) atomicMin(&res[1], (unsigned long long)k);
  }
}

__global__ void k_mm_after(const uint8_t* __restrict__ status, uint64_t from, uint64_t nlines,
                           unsigned long long* __restrict__ res) {
  for (uint64_t k = from + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines;
       k += (uint64_t)gridDim.x * blockDim.x)
    if (status[k] != 0) atomicMin(&res[2], (unsigned long long)k);
}

template <typename T>
T read1(const T* d, cudaStream_t s) {
  T h;
  TC_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

// Returns true and fills d_pairs (device, 2*nnz u32) when the entry body is
// well formed; false when the host parser must produce the error.
bool mm_tokenize(const unsigned char* d_body, uint64_t len, const MmHeader& h, DBuf<uint32_t>& d_pairs,
                 int device, cudaStream_t s) {
  const uint64_t nblocks = (len + kBlockBytes - 1) / kBlockBytes;
  uint64_t nlines = 0;
  DBuf<uint64_t> starts;
  if (len) {
    DBuf<uint32_t> cnt(nblocks, s), boff(nblocks + 1, s);
    k_mm_block_lines<<<(unsigned)nblocks, kT, 0, s>>>(d_body, len, cnt.get());
    TC_LAUNCH();
    scan_exclusive<uint32_t>(LoadArray<uint32_t>{cnt.get()}, boff.get(), nblocks, boff.get() + nblocks, s);
    nlines = read1(boff.get() + nblocks, s);
    starts.alloc(nlines ? nlines : 1, s);
    k_mm_line_starts<<<(unsigned)nblocks, kT, 0, s>>>(d_body, len, boff.get(), starts.get());
    TC_LAUNCH();
  }
  d_pairs.alloc(2 * (h.nnz ? h.nnz : 1), s);
  if (h.nnz == 0) {
    if (!nlines) return true;
    // only blank/comment lines may follow the size line
  }
  DBuf<uint8_t> status(nlines ? nlines : 1, s);
  DBuf<uint2> ij(nlines ? nlines : 1, s);
  DBuf<uint64_t> eidx(nlines + 1, s);
  DBuf<unsigned long long> res(3, s);
  TC_CUDA(cudaMemsetAsync(res.get(), 0xff, 3 * sizeof(unsigned long long), s));
  const uint64_t cap = (uint64_t)num_sms(device) * 16;
  const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cap, (nlines + kT - 1) / kT));
  if (nlines) {
    k_mm_parse<<<grid, kT, 0, s>>>(d_body, len, starts.get(), nlines, h.rows, h.cols, status.get(), ij.get());
    TC_LAUNCH();
    scan_exclusive<uint64_t>(IsEntry{status.get()}, eidx.get(), nlines, eidx.get() + nlines, s);
    k_mm_emit<<<grid, kT, 0, s>>>(status.get(), ij.get(), eidx.get(), nlines, h.nnz, d_pairs.get(), res.get());
    TC_LAUNCH();
  }
  unsigned long long r[3];
  TC_CUDA(cudaMemcpyAsync(r, res.get(), sizeof(r), cudaMemcpyDeviceToHost, s));
  TC_CUDA(cudaStreamSynchronize(s));
  const uint64_t last = h.nnz ? r[0] : (uint64_t)-1;  // line of the nnz-th entry
  if (h.nnz && last == ~0ull) return false;          // fewer than nnz entries
  if (h.nnz && r[1] < last) return false;            // malformed line before it
  const uint64_t from = h.nnz ? last + 1 : 0;
  if (from < nlines) {
    k_mm_after<<<grid, kT, 0, s>>>(status.get(), from, nlines, res.get());
    TC_LAUNCH();
    TC_CUDA(cudaMemcpyAsync(r, res.get(), sizeof(r), cudaMemcpyDeviceToHost, s));
    TC_CUDA(cudaStreamSynchronize(s));
    if (r[2] != ~0ull) return false;  // content after the last entry
  }
  return true;
}

}  // namespace tcb
