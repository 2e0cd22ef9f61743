/* dag_stats.c -- workload statistics of the degree-ordered pivot join on a
 * synthetic config (design evidence for count.cu; not product, not oracle).
 *   dag_stats <rmat|kron|er> <scale> <param>
 * Builds the symmetric CSR with oracle.c, orients by (deg,id) in rank space,
 * then enumerates every candidate wedge (in-edge u->v of pivot v, x in the
 * suffix of N+(u) after v) and histograms candidates and hits by top
 * distance n-1-x. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>
#include "../oracle/oracle.h"

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}
#define NB 9
static const uint32_t edges_[NB] = {256, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 0xffffffffu};

int main(int argc, char** argv) {
  const int kind = strcmp(argv[1], "er") == 0 ? 1 : 0, permute = strcmp(argv[1], "kron") == 0;
  const int scale = atoi(argv[2]), param = atoi(argv[3]);
  const uint32_t n = 1u << scale;
  const uint64_t m = kind ? oracle_er_num_edges(scale, param) : oracle_rmat_num_edges(scale, param);
  uint32_t* pairs = malloc(m * 8);
  if (kind) oracle_gen_er(scale, param, pairs); else oracle_gen_rmat(scale, param, permute, pairs);
  uint64_t *off, E, L, D; uint32_t* nb;
  oracle_build_graph(pairs, m, n, &off, &nb, &E, &L, &D);
  free(pairs);
  /* rank by (deg,id) */
  uint32_t* order = malloc(n * 4); uint32_t* rank = malloc(n * 4);
  { uint64_t maxd = 0; for (uint32_t v = 0; v < n; ++v) if (off[v+1]-off[v] > maxd) maxd = off[v+1]-off[v];
    uint64_t* b = calloc(maxd + 2, 8);
    for (uint32_t v = 0; v < n; ++v) ++b[off[v+1]-off[v]+1];
    for (uint64_t d = 0; d <= maxd; ++d) b[d+1] += b[d];
    for (uint32_t v = 0; v < n; ++v) { uint64_t r = b[off[v+1]-off[v]]++; order[r] = v; rank[v] = r; }
    free(b); }
  uint64_t* oo = calloc(n + 1, 8); uint64_t* io = calloc(n + 1, 8);
  for (uint32_t r = 0; r < n; ++r) { uint32_t v = order[r]; uint64_t c = 0;
    for (uint64_t k = off[v]; k < off[v+1]; ++k) c += rank[nb[k]] > r;
    oo[r+1] = c; io[r+1] = off[v+1]-off[v]-c; }
  for (uint32_t r = 0; r < n; ++r) { oo[r+1] += oo[r]; io[r+1] += io[r]; }
  uint32_t* oc = malloc(E * 4); uint32_t* ic = malloc(E * 4); uint64_t* cur = malloc(n * 8);
  memcpy(cur, io, n * 8);
  for (uint32_t r = 0; r < n; ++r) { uint32_t v = order[r]; uint64_t p = oo[r];
    for (uint64_t k = off[v]; k < off[v+1]; ++k) { uint32_t x = rank[nb[k]]; if (x > r) { oc[p++] = x; ic[cur[x]++] = r; } }
    qsort(oc + oo[r], p - oo[r], 4, cmp_u32); }
  free(off); free(nb);
  const uint32_t h0 = n > 65536 ? n - 65536 : 0;
  double cand[NB] = {0}, hits[NB] = {0}, J = 0, T = 0, items = 0, items_hot = 0;
  double core_c[3] = {0}, core_elig_items[3] = {0}, core_elig_c[3] = {0}; const uint32_t K[3] = {1024, 2048, 4096};
  double words_hot = 0, words64_hot = 0, cand_hot = 0;  /* distinct 32-bit bitmap words touched per item's hot suffix, summed */
  double segs512 = 0, piv = 0, dplus_hist[6] = {0}; /* J by pivot d+ class: <=64, <=256, <=1024, >1024 */
  const uint64_t W = (n + 63) / 64;
#pragma omp parallel reduction(+:cand[:NB], hits[:NB], J, T, items, items_hot, core_c[:3], core_elig_items[:3], core_elig_c[:3], words_hot, words64_hot, cand_hot, segs512, piv, dplus_hist[:6])
  { uint64_t* bm = calloc(W, 8);
#pragma omp for schedule(dynamic, 64)
    for (int64_t bb = n - 1; bb >= 0; --bb) { uint32_t b = bb;
      uint64_t dv = oo[b+1]-oo[b], din = io[b+1]-io[b];
      if (!dv || !din) continue;
      ++piv; segs512 += (din + 511) / 512;
      for (uint64_t k = oo[b]; k < oo[b+1]; ++k) bm[oc[k]>>6] |= 1ull << (oc[k]&63);
      double jb = 0;
      for (uint64_t q = io[b]; q < io[b+1]; ++q) { uint32_t a = ic[q]; const uint32_t* na = oc + oo[a]; uint64_t da = oo[a+1]-oo[a];
        uint64_t lo = 0, hi = da; while (lo < hi) { uint64_t mid = (lo+hi)/2; if (na[mid] <= b) lo = mid+1; else hi = mid; }
        if (lo >= da) continue;
        ++items; uint32_t lastw = 0xffffffffu; uint64_t cc[3] = {0,0,0}; int anyhot = 0;
        for (uint64_t k = lo; k < da; ++k) { uint32_t x = na[k]; uint32_t td = n - 1 - x; int bi = 0; while (td >= edges_[bi]) ++bi;
          cand[bi] += 1; J += 1; jb += 1;
          if (x >= h0) { anyhot = 1; cand_hot += 1; uint32_t w = (x - h0) >> 5; if (w != lastw) { words_hot += 1; if ((w >> 1) != (lastw >> 1) || lastw == 0xffffffffu) words64_hot += 1; lastw = w; } }
          for (int t = 0; t < 3; ++t) if (td < K[t]) cc[t]++;
          if ((bm[x>>6] >> (x&63)) & 1) { hits[bi] += 1; T += 1; } }
        items_hot += anyhot;
        for (int t = 0; t < 3; ++t) { core_c[t] += cc[t]; if (cc[t] >= K[t] / 32) { core_elig_items[t] += 1; core_elig_c[t] += cc[t]; } } }
      int cl = dv <= 64 ? 0 : dv <= 256 ? 1 : dv <= 1024 ? 2 : 3; dplus_hist[cl] += jb;
      for (uint64_t k = oo[b]; k < oo[b+1]; ++k) bm[oc[k]>>6] = 0; }
    free(bm); }
  printf("n=%u E=%llu J=%.4g T=%.4g items=%.4g items_hot=%.4g pivots=%.4g segs512=%.4g words_hot=%.4g\n", n,
         (unsigned long long)E, J, T, items, items_hot, piv, segs512, words_hot);
  printf("hot cands=%.4g words32=%.4g (%.2f ids/word) words64=%.4g (%.2f ids/word)\n", cand_hot, words_hot, cand_hot/words_hot, words64_hot, cand_hot/words64_hot);
  printf("top-distance buckets (<256 <1K <2K <4K <8K <16K <32K <64K cold):\n cand%%:");
  for (int i = 0; i < NB; ++i) printf(" %.2f", 100 * cand[i] / J);
  printf("\n hits%%:");
  for (int i = 0; i < NB; ++i) printf(" %.2f", 100 * hits[i] / T);
  printf("\nJ by pivot d+ (<=64 <=256 <=1024 >1024) %%: %.2f %.2f %.2f %.2f\n", 100*dplus_hist[0]/J, 100*dplus_hist[1]/J, 100*dplus_hist[2]/J, 100*dplus_hist[3]/J);
  for (int t = 0; t < 3; ++t) printf("core K=%u: cand in core %.2f%% of J; items with >=K/32 core cands: %.4g carrying %.2f%% of J\n", K[t], 100*core_c[t]/J, core_elig_items[t], 100*core_elig_c[t]/J);
  return 0;
}
