// graph.cuh -- the device-resident graph handle behind the opaque tc_graph.
//
// HBM layout (all arrays in degree-rank space, rank = position of (deg, id) in
// ascending order, so the north-star orientation u->v iff (deg u,u) < (deg v,v)
// is simply rank(u) < rank(v)):
//   off[n+1]  u32  oriented CSR row offsets (|E+| = |E| < 2^32)
//   col[|E|]  u32  N+(r) as ranks, strictly ascending per row, +16 B tail pad
//   src[|E|]  u32  source rank of each oriented edge (COO companion of col)
//   deg[n]    u32  undirected degree by rank
//   id_of[n]  u32  rank -> original vertex id
//   rank_of[n]u32  original vertex id -> rank
// 16 B per oriented edge + 16 B per vertex: C4 (RMAT s24) = 4.4 GB,
// C5 (RMAT s26 ef32) = 34 GB of 180 GB.
#pragma once

#include <atomic>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tcb {
// Grow-only device scratch owned by a graph handle: the per-count frontier,
// hit masks and counters are rebuilt by every tc_count in the same buffers,
// so repeated counts do not remap memory (a cuBLAS-style workspace).
struct Scratch {
  DBuf<uint8_t> buf;
  template <typename T>
  T* get(uint64_t count, cudaStream_t s) {
    const uint64_t need = (count ? count : 1) * sizeof(T);
    if (buf.n < need) {
      buf.s = s;  // free the old block on the stream that uses it now
      buf.alloc(need + need / 8, s);
    }
    return reinterpret_cast<T*>(buf.get());
  }
  void release(cudaStream_t s) {
    buf.s = s;
    buf.release();
  }
};
enum ScratchSlot {
  kSlotSegOff, kSlotWsegs, kSlotCsegs, kSlotSsegs, kSlotMasks, kSlotSlab, kSlotTRank,
  kSlotHeavy, kSlotCls, kSlotSums, kSlotCounters, kSlotAcc, kSlotScanWs, kSlotCount
};
}  // namespace tcb

struct tc_graph {
  int device = 0;
  cudaStream_t own_stream = nullptr;
  // count fork/join (count.cu): the CTA join on a high-priority stream, the
  // warp / small / dense joins on a low-priority one, so they fill its tail
  cudaStream_t hi_stream = nullptr, lo_stream = nullptr;
  cudaEvent_t fork_ev = nullptr, join_hi = nullptr, join_lo = nullptr;
  cudaStream_t stream = nullptr;
  uint32_t n = 0;
  uint64_t E = 0;
  uint32_t max_deg = 0;
  uint32_t max_dplus = 0;
  uint32_t max_din = 0;  // largest in-degree in the orientation (in-edge items of one pivot)
  int id_bits = 1;  // bits_for(n-1)
  double build_ms = 0;
  tcb::DBuf<uint32_t> off, col, src, deg, id_of, rank_of;
  // Hot window: the top kHotBits ranks [h0, n), where ~97% of wedge endpoints
  // of a power-law DAG fall (n-x < 2^16 for 97% of probes).  Each
  // row's members >= h0 form its sorted suffix; they are mirrored as 16-bit
  // offsets x - h0 in colH (row r at [offH[r], offH[r+1])), halving the bytes
  // the join streams and letting a probe index the pivot bitmap directly.
  uint32_t h0 = 0;
  tcb::DBuf<uint16_t> colH;
  tcb::DBuf<uint32_t> offH;
  // In-edge index: the oriented edges grouped by head, slots [inoff[v],
  // inoff[v+1]) for every u->v.  Together with off/col this is the
  // reference's symmetric adjacency split by orientation (N+(v) and N-(v));
  // it is what makes the level-1 frontier of a count a plan over |V| instead
  // of a scatter over |E| (plan.cu).  Each slot is a 32-byte level-1 item
  // record (one DRAM sector, written once at build by k_in_scatter with one
  // 256-bit store) so a join stages an item with one coalesced load and no
  // row lookup:
  //   irec[2 slot]     = {hb, he, cb, ce}  sparse hot suffix colH[hb, he),
  //                                        cold suffix col[cb, ce) (empty:
  //                                        end <= begin)
  //   irec[2 slot + 1] = {e, u, mo_lo, mo_hi}  edge position, source, first
  //                                        per-vertex mask byte
  tcb::DBuf<uint32_t> inoff;
  tcb::DBuf<uint4> irec;
  // Row descriptors, one 32-byte record (two uint4, one DRAM sector) per rank
  // of the non-isolated ranks [r0, n) (isolated vertices have the lowest
  // ranks and no work): tcb::RowGeo -- a join stages an item's whole row
  // geometry (offsets, hot/core split, dense index, per-vertex mask base)
  // with one sector read.
  tcb::DBuf<uint4> rowd;
  uint32_t r0 = 0;
  // Dense core: the top core_bits ranks [cb, n) (inside the hot window).  A
  // row with at least core_min members there ("dense row") keeps them as a
  // core_bits-bit bitmap (cbits + didx * core_words) instead of in its
  // sparse hot suffix: a join intersects such an item's core part with the
  // pivot's core words word-parallel (count.cu dense step).  At RMAT s24,
  // 1.9e5 rows (49 MB of bitmaps) carry 45% of the candidate wedges.
  uint32_t cb = 0, core_words = 0;  // core_words = 0: no dense rows
  uint32_t ndense = 0, core_min = 0;
  tcb::DBuf<uint32_t> cbits;
  // Dense in-edge list (graph-static, like ine): for every pivot v, the
  // dense index of each in-neighbour u whose row is dense and whose suffix
  // after v is non-empty -- the items k_join_dense intersects -- grouped by
  // pivot (dine), cut into segments of <= kDenseSeg items {v, i0, i1}
  // (dseg; pivot v's are [dsoff[v], dsoff[v+1])); drow[didx] = the row's rank.
  tcb::DBuf<uint32_t> dine, dsoff, drow;
  tcb::DBuf<uint4> dseg;
  uint64_t ndine = 0;
  // Count-plan capacities (graph properties, recorded once at build): work
  // segments per pivot class over the whole graph (any part has at most as
  // many) and the per-vertex mask bytes of all rows (RowGeo::rowbase is the
  // exclusive scan of the rows' mask bytes).
  uint64_t seg_cap[3] = {0, 0, 0};
  uint64_t mask_total = 0;
  // multi-GPU work partition (count.cu): pivot rank ranges [b[p], b[p+1])
  // with ~equal join work; computed on the first P-part count, then reused
  std::vector<uint64_t> part_bounds;
  uint32_t part_bounds_P = 0;
  // per part of the last P-way split: each row's item range {k_lo, k_hi}
  // (per-vertex row pass of a split count), built on first use
  std::vector<tcb::DBuf<uint2>> part_kr;
  uint32_t part_kr_P = 0;
  tcb::Scratch scratch[tcb::kSlotCount];
  // Every call that touches the handle's scratch, stream or partition state
  // (count, listings, export, degrees, partition bounds, set_stream) holds
  // this for its whole duration: concurrent calls on one Graph (allowed by the
  // reference, graph.hpp:33-34) are serialised, never interleaved on the
  // shared per-count buffers.
  std::mutex mu;
};

namespace tcb {

constexpr uint32_t kHotBits = 1u << 16;
#ifndef TCB_WARP_MAX_DEG
#define TCB_WARP_MAX_DEG 64
#endif
// warp bin: d+(v) <= 64 (128-slot warp table; A/B at C4: 48 -> 64 saves 0.4 ms,
// 96 costs 0.5 ms at C3)
constexpr uint32_t kWarpMaxDeg = TCB_WARP_MAX_DEG;
#ifndef TCB_WARP_SEG_ITEMS
#define TCB_WARP_SEG_ITEMS 64
#endif
constexpr uint32_t kWarpSegItems = TCB_WARP_SEG_ITEMS;  // items per warp-bin segment
#ifndef TCB_CTA_SEG_ITEMS
#define TCB_CTA_SEG_ITEMS 512
#endif
constexpr uint32_t kCtaSegItems = TCB_CTA_SEG_ITEMS;  // items per CTA-bin segment
#ifndef TCB_ITEM_STRIDE_TOTAL
#define TCB_ITEM_STRIDE_TOTAL 1
#endif
// uint4s per level-1 item record without per-vertex counts (A/B: padding the
// 16-byte record to a full 32-byte sector is slower, 10.2 vs 9.6 ms at C4)
constexpr int kItemStrideTotal = TCB_ITEM_STRIDE_TOTAL;
// small CTA-bin pivots (d+ > kWarpMaxDeg but few in-edge items and few
// members below the hot window) are joined one warp each: at RMAT s24 they
// are 60% of the CTA-bin segments and 2% of the candidate wedges
#ifndef TCB_SMALL_ITEMS
#define TCB_SMALL_ITEMS 32
#endif
#ifndef TCB_SMALL_COLD
#define TCB_SMALL_COLD 256
#endif
constexpr uint32_t kSmallItems = TCB_SMALL_ITEMS;  // multiple of 32
constexpr uint32_t kSmallCold = TCB_SMALL_COLD;    // power of two

// Count plan of one part (plan.cu): the pivots v in the part's rank range
// [v_lo, v_hi) that can close a triangle, classified and cut into work
// segments {v, i0, i1, 0} over the in-edge index positions
// [inoff[v], inoff[v+1]).  An item of pivot v is in-edge ine[i] = {e, u}: the
// reference's level-1 row (u, v) (matcher.cpp:136-198), whose wedge suffix is
// col[e+1 .. off[u+1]) -- its geometry (hot part in colH, cold part in col,
// per-vertex mask offset) is computed by the join when it stages the segment.
// Everything here is built inside every tc_count (timed) with no host
// synchronisation: list lengths live in device memory (nseg), list capacities
// are graph properties recorded at build (tc_graph::seg_cap).
//   wsegs  warp bin   (d+(v) <= kWarpMaxDeg, and d+(v) = 0 pivots whose
//                      per-vertex mask bytes must be zeroed)
//   csegs  CTA bin    (kCtaSegItems items per segment)
//   ssegs  small bin  (<= kSmallItems items, <= kSmallCold cold members)
//   masks  per-vertex hit masks (row u's block at RowGeo::rowbase)
struct Plan {
  uint4* wsegs = nullptr;
  uint4* csegs = nullptr;
  uint4* ssegs = nullptr;
  uint32_t* nseg = nullptr;  // device: [0] warp, [1] CTA, [2] small segment counts
  uint8_t* masks = nullptr;
  uint32_t v_lo = 0, v_hi = 0;
  uint64_t cap[3] = {0, 0, 0};
  uint64_t W = 0, J = 0, hot = 0, items = 0, pivots = 0;  // stats (read_plan_sums)
  double cta_bytes = 0, dense_bytes = 0;  // per-kernel algorithmic bytes (tc_count_stats)
  uint32_t core_words = 0;
  void* sums = nullptr;
};
// Returns the number of kernels launched.
// masks: per-vertex hit masks (d+ = 0 pivots' items zeroed by the warp bin)
int build_plan(tc_graph& g, uint32_t v_lo, uint32_t v_hi, bool per_vertex, bool masks, bool want_sums, Plan& p);
// The plan's work counters (W, J, hot, items, pivots) -- a read, only for stats.
void read_plan_sums(Plan& p, cudaStream_t s);

// Pivot class (graph property): 0 = warp bin (d+(v) <= kWarpMaxDeg; with
// per-vertex counts also d+(v) = 0 pivots, whose items' mask bytes the warp
// join zeroes), 1 = CTA bin, 2 = small CTA pivots (<= kSmallItems in-edges
// and <= kSmallCold members below the hot window: one warp each), -1 = none.
__host__ __device__ __forceinline__ uint32_t segs_per_class(int c) {
  return c == 0 ? kWarpSegItems : c == 1 ? kCtaSegItems : kSmallItems;
}
struct PivotClass {
  const uint32_t* off;
  const uint32_t* offH;
  const uint32_t* inoff;
  bool pv;
  __device__ __forceinline__ int operator()(uint32_t v, uint32_t& din) const {
    const uint32_t dv = off[v + 1] - off[v];
    din = inoff[v + 1] - inoff[v];
    if (din == 0 || (dv == 0 && !pv)) return -1;
    if (dv <= kWarpMaxDeg) return 0;
    const uint32_t hv = offH[v + 1] - offH[v];
    return (din <= kSmallItems && dv - hv <= kSmallCold) ? 2 : 1;
  }
};

// Per-vertex hit-mask layout of row u (closed form, no per-edge scan).  Row u
// has d = d+(u) out-edges, the last h of them hot (colH[O, O+h), O = offH[u]),
// c0 = d - h cold.  Item k (edge off[u]+k, suffix positions k+1..d-1) starts
// its hot part at s_k = max(k+1-c0, 0) and owns one mask byte per chunk
// cs_k = (O+s_k)>>3 .. c_hi-1, c_hi = (O+h+7)>>3.  The row's block holds the
// items k = 0..d-2 back to back: P(k) = bytes of items < k.
struct RowMasks {
  uint64_t O;
  uint32_t d, h, c0;
  uint64_t c_lo, c_hi;
  __host__ __device__ __forceinline__ RowMasks(uint32_t d_, uint64_t O_, uint32_t h_)
      : O(O_), d(d_), h(h_), c0(d_ - h_), c_lo(O_ >> 3), c_hi((O_ + h_ + 7) >> 3) {}
  // sum_{t < x} floor(t/8)
  __host__ __device__ static __forceinline__ uint64_t F(uint64_t x) {
    const uint64_t q = x >> 3, r = x & 7;
    return 4 * q * (q ? q - 1 : 0) + r * q;
  }
  __host__ __device__ __forceinline__ uint64_t P(uint32_t k) const {
    const uint64_t C = c_hi - c_lo;
    if (k <= c0) return (uint64_t)k * C;
    const uint64_t S = k - c0;
    return (uint64_t)c0 * C + S * c_hi - (F(O + S + 1) - F(O + 1));
  }
  // total bytes of the row (0 when it has no hot member or < 2 out-edges)
  __host__ __device__ __forceinline__ uint64_t total() const { return (h == 0 || d < 2) ? 0 : P(d - 1); }
  __host__ __device__ __forceinline__ uint64_t first_chunk(uint32_t k) const {
    const uint64_t sk = k + 1 > c0 ? (uint64_t)(k + 1 - c0) : 0;
    return (O + sk) >> 3;
  }
};

// Dense-core parameters: core_bits ranks (a multiple of 32, <= 32 * 32 *
// kCoreWordsMax), rows with >= core_min core members are dense.
#ifndef TCB_CORE_BITS
#define TCB_CORE_BITS 2048
#endif
constexpr uint32_t kCoreBits = TCB_CORE_BITS;
constexpr int kCoreWordsMax = 3;  // core words per lane of a warp the dense join is instantiated for (2, 3)
static_assert(kCoreBits <= 32u * 32u * kCoreWordsMax, "default core larger than the dense join supports");
constexpr uint32_t kDenseSeg = 64;  // dense items per k_join_dense segment

// Row descriptor of rank u (tc_graph::rowd[2(u - r0)], [2(u - r0) + 1]):
//   a = {beg = off[u], end = off[u+1], O = offH[u], Ht}
//   b = {Hf = offH[u+1], didx, rowbase lo, rowbase hi}
// The row's members: cold col[beg, beg + c0), hot colH[O, Hf) (ids >= h0,
// sorted); of the hot ones the sparse part is colH[O, Ht) and, for a dense
// row, the core part colH[Ht, Hf) (ids >= cb) lives in its core bitmap
// (didx; kNoDense otherwise, Ht = Hf).  Per-vertex hit masks cover the sparse
// hot part only: RowMasks(d - cc, O, Ht - O) at rowbase.
constexpr uint32_t kNoDense = 0xffffffffu;
struct RowGeo {
  uint32_t beg, end, O, Ht, Hf, didx;
  uint64_t rowbase;
  __host__ __device__ __forceinline__ RowGeo(const uint4& a, const uint4& b)
      : beg(a.x), end(a.y), O(a.z), Ht(a.w), Hf(b.x), didx(b.y), rowbase(b.z | ((uint64_t)b.w << 32)) {}
  __host__ __device__ __forceinline__ uint32_t d() const { return end - beg; }
  __host__ __device__ __forceinline__ uint32_t h() const { return Hf - O; }   // hot members
  __host__ __device__ __forceinline__ uint32_t cc() const { return Hf - Ht; }  // core members cut out
  __host__ __device__ __forceinline__ uint32_t cold_end() const { return end - (Hf - O); }
  __host__ __device__ __forceinline__ RowMasks masks() const { return RowMasks(d() - cc(), O, Ht - O); }
};
#ifdef __CUDACC__
__device__ __forceinline__ RowGeo load_row(const uint4* __restrict__ rowd, uint32_t r0, uint32_t u) {
  const uint4* p = rowd + 2 * (uint64_t)(u - r0);
  return RowGeo(__ldg(p), __ldg(p + 1));
}
#endif

// Build pipeline entry points (build.cu).
void build_from_pairs(tc_graph& g, const uint32_t* d_pairs, uint64_t m, uint32_t n,
                      tc_build_report* rep);
// strict: TRIMCSR1 ingest -- reject bad offsets / self-loops / unsorted rows
// with the reference's ParseError messages (io.cpp:206-218)
// Host-resident neighbour array for build_from_csr: copied into d_dst (which
// is then the d_nbrs argument) in kFeedChunk-entry pieces on a side stream
// while the rows that have arrived are oriented.  h_off (host copy of the
// offsets, or null = one piece) places the row boundaries.
constexpr uint64_t kFeedChunk = 1ull << 25;
struct CsrFeed {
  const uint32_t* h_nbrs;
  const uint64_t* h_off;
  uint32_t* d_dst;
};
void build_from_csr(tc_graph& g, const uint64_t* d_off, const uint32_t* d_nbrs, uint32_t n,
                    uint64_t num_edges, bool strict = false, const CsrFeed* feed = nullptr);

// Host memory that is neither pinned nor registered with CUDA.
bool pageable_host(const void* p);
// host<->device copies that take pageable buffers through pinned bounce slots
// when large (feed.cu); synchronous on that path
void copy_h2d(void* d, const void* h, size_t bytes, cudaStream_t s);
void copy_d2h(void* h, const void* d, size_t bytes, cudaStream_t s);

// The piece-by-piece host->device copy behind build_from_csr (feed.cu):
// pinned sources are DMA'd directly; pageable ones go through pinned bounce
// slots filled by worker threads.  wait_piece(k, s) makes s wait for piece k;
// the destructor waits for every piece in flight.
class PieceFeed {
 public:
  PieceFeed(const uint32_t* h, uint32_t* d, uint64_t total, uint64_t piece, cudaStream_t after);
  ~PieceFeed();
  PieceFeed(const PieceFeed&) = delete;
  PieceFeed& operator=(const PieceFeed&) = delete;
  uint32_t pieces() const { return K_; }
  bool pageable() const { return pageable_; }
  void wait_piece(uint32_t k, cudaStream_t s);

 private:
  void issue(uint32_t upto);
  void work(uint32_t t);
  const uint32_t* h_;
  uint32_t* d_;
  uint64_t total_, piece_;
  uint32_t K_ = 0, W_ = 1, issued_ = 0;
  int dev_ = 0;
  bool pageable_ = false;
  std::vector<cudaEvent_t> ev_, slot_done_;
  std::vector<cudaStream_t> streams_;
  std::vector<std::thread> workers_;
  std::unique_lock<std::mutex> lock_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<char> recorded_;
  std::exception_ptr err_;
  std::atomic<bool> abort_{false};
};
void export_csr(tc_graph& g, uint64_t* d_off, uint32_t* d_nbrs);
void export_degrees(tc_graph& g, uint32_t* d_deg);

// Count pipeline (count.cu).
void count_triangles(tc_graph& g, const tc_count_opts& opts, uint64_t* d_total,
                     uint64_t* d_per_vertex, tc_count_stats* stats);
// Degree-weighted oriented-edge ranges of a P-way split.
const std::vector<uint64_t>& partition_bounds(tc_graph& g, uint32_t parts);

// Multi-GPU (multi.cu).
void comm_unique_id(void* id);
tc_comm* comm_init_rank(const void* id, int nranks, int rank, int device);
void comm_destroy(tc_comm* c);
void count_allreduce(tc_comm* c, tc_graph& g, const tc_count_opts& o, uint64_t* d_total, uint64_t* d_pv,
                     tc_count_stats* st);
tc_multi* multi_create(const int* devices, int nparts);
void multi_destroy(tc_multi* m);
int multi_parts(const tc_multi* m);
int multi_part_device(const tc_multi* m, int p);
void count_multi(tc_multi* m, tc_graph* const* graphs, const tc_count_opts& o, uint64_t* d_total, uint64_t* d_pv,
                 tc_count_stats* st);

// MatrixMarket entry tokenizer (mm.cu): true and device pairs when the body is
// well formed, false when the host parser must report the error.
struct MmHeader;
bool mm_tokenize(const unsigned char* d_body, uint64_t len, const MmHeader& h, DBuf<uint32_t>& d_pairs,
                 int device, cudaStream_t s);

// Triangle listings (listing.cu): writes min(T, cap) rows (3 u32 ids,
// ascending) to d_rows, returns T.
uint64_t list_triangles(tc_graph& g, uint32_t* d_rows, uint64_t cap, uint64_t e0, uint64_t e1);

// Generators (gen.cu).
uint64_t gen_num_edges(int kind, int scale, int param);
void generate(int kind, int scale, int param, uint32_t* d_pairs, cudaStream_t s);

}  // namespace tcb
