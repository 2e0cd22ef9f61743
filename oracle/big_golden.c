/*
 * big_golden.c -- goldens for the configs too large for make_golden.py's
 * in-memory path (C4 per-vertex from the reference, C5 RMAT s26 ef32).
 *
 * TEST INFRASTRUCTURE ONLY (run in the build container; the product never
 * links it).  Usage:
 *   big_golden <rmat|kron|er> <scale> <param> <mode> [threads]
 *     mode  ref     the reference's own segmented_intersect with listings
 *                   (oracle/_ref, frontier.cpp:51-81, chunked by source rows)
 *           oracle  oracle_count (the id-order restatement, oracle.c)
 *           dag     oracle_count_dag (degree-ordered pivot join, oracle.c)
 *           none    graph fingerprints only
 * Prints one JSON object with the fields tests/golden/synthetic.json holds.
 *
 * The symmetric CSR is built exactly as build_graph does (graph.cpp:33-85:
 * drop loops, both orientations, per-row sort + unique, dups/2) but streamed:
 * the counter-based generator (oracle_gen_range) runs twice -- once to count
 * degrees and hash the pair array, once to scatter -- so C5's 17 GB pair array
 * is never held, and rows are compacted in place.  Peak memory is the CSR
 * (2m u32 before dedup) plus the offsets.
 */
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "oracle.h"

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

static uint64_t fnv_step(uint64_t h, const void* data, uint64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

#define BLOCK (1ULL << 24)

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s <rmat|kron|er> <scale> <param> <ref|oracle|dag|none> [threads]\n", argv[0]);
    return 2;
  }
  const char* kname = argv[1];
  const int scale = atoi(argv[2]), param = atoi(argv[3]);
  const char* mode = argv[4];
  const int threads = argc > 5 ? atoi(argv[5]) : 0;
#ifdef _OPENMP
  if (threads > 0) omp_set_num_threads(threads);
#endif
  const int kind = strcmp(kname, "er") == 0 ? 1 : 0;
  const int permute = strcmp(kname, "kron") == 0;
  const uint32_t n = 1u << scale;
  const uint64_t m = kind == 1 ? oracle_er_num_edges(scale, param) : oracle_rmat_num_edges(scale, param);
  uint32_t* perm = NULL;
  if (permute) {
    perm = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    oracle_kron_perm(scale, perm);
  }
  double t0 = now_s();
  /* pass 1: pair fingerprint, loops, degree counts (graph.cpp:38-49) */
  uint32_t* blk = (uint32_t*)malloc(2 * BLOCK * sizeof(uint32_t));
  uint64_t* deg = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t hp = 0xcbf29ce484222325ULL, loops = 0;
  for (uint64_t i0 = 0; i0 < m; i0 += BLOCK) {
    const uint64_t i1 = i0 + BLOCK < m ? i0 + BLOCK : m;
    oracle_gen_range(kind, scale, param, i0, i1, perm, blk);
    hp = fnv_step(hp, blk, (i1 - i0) * 8);
    uint64_t lp = 0;
#pragma omp parallel for schedule(static) reduction(+ : lp)
    for (int64_t k = 0; k < (int64_t)(i1 - i0); ++k) {
      const uint32_t u = blk[2 * k], v = blk[2 * k + 1];
      if (u == v) {
        ++lp;
        continue;
      }
      __atomic_fetch_add(&deg[u + 1], 1, __ATOMIC_RELAXED);
      __atomic_fetch_add(&deg[v + 1], 1, __ATOMIC_RELAXED);
    }
    loops += lp;
  }
  for (uint64_t u = 0; u < n; ++u) deg[u + 1] += deg[u]; /* now offsets (graph.cpp:50) */
  uint64_t* off = deg;
  const uint64_t slots = off[n];
  uint32_t* adj = (uint32_t*)malloc((slots ? slots : 1) * sizeof(uint32_t));
  uint64_t* cur = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  memcpy(cur, off, (size_t)n * sizeof(uint64_t));
  /* pass 2: scatter both orientations (graph.cpp:52-58; row order is fixed by
   * the sort below, so the scatter may run in parallel) */
  for (uint64_t i0 = 0; i0 < m; i0 += BLOCK) {
    const uint64_t i1 = i0 + BLOCK < m ? i0 + BLOCK : m;
    oracle_gen_range(kind, scale, param, i0, i1, perm, blk);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < (int64_t)(i1 - i0); ++k) {
      const uint32_t u = blk[2 * k], v = blk[2 * k + 1];
      if (u == v) continue;
      adj[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
      adj[__atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED)] = u;
    }
  }
  free(blk);
  free(perm);
  /* per-row sort + unique (graph.cpp:61-76), then in-place compaction */
  uint64_t* nd = cur; /* reuse: unique length per row */
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t uu = 0; uu < (int64_t)n; ++uu) {
    uint32_t* r = adj + off[uu];
    const uint64_t d = off[uu + 1] - off[uu];
    if (d > 1) qsort(r, d, sizeof(uint32_t), cmp_u32);
    uint64_t w = 0;
    for (uint64_t i = 0; i < d; ++i)
      if (w == 0 || r[w - 1] != r[i]) r[w++] = r[i];
    nd[uu] = w;
  }
  uint64_t write = 0;
  for (uint64_t u = 0; u < n; ++u) {
    const uint64_t b = off[u], d = nd[u];
    if (write != b) memmove(adj + write, adj + b, d * sizeof(uint32_t));
    off[u] = write;
    write += d;
  }
  off[n] = write;
  free(nd);
  const uint64_t E = write / 2;
  const uint64_t dups = (slots - write) / 2; /* graph.cpp:80-81 */
  const double t_build = now_s() - t0;
  const uint64_t off_fnv = oracle_fnv1a64(off, ((uint64_t)n + 1) * 8);
  const uint64_t nb_fnv = oracle_fnv1a64(adj, write * 4);
  fprintf(stderr, "built: E=%llu loops=%llu dups=%llu in %.1f s\n", (unsigned long long)E,
          (unsigned long long)loops, (unsigned long long)dups, t_build);

  uint64_t T = 0;
  uint64_t* pv = NULL;
  double t_count = 0;
  const char* source = "none";
  if (strcmp(mode, "none") != 0) {
    pv = (uint64_t*)calloc((size_t)n, sizeof(uint64_t));
    const double t1 = now_s();
    if (strcmp(mode, "dag") == 0) {
      T = oracle_count_dag(off, adj, n, pv, threads);
      source = "oracle_count_dag (degree-ordered pivot join, oracle.c; pinned to the reference goldens)";
    } else if (strcmp(mode, "oracle") == 0) {
      T = oracle_count(off, adj, n, pv, threads);
      source = "oracle_count (id-order segmented-intersect restatement, oracle.c)";
    } else if (strcmp(mode, "ref") == 0) {
      char path[4096];
      const char* self = argv[0];
      const char* slash = strrchr(self, '/');
      snprintf(path, sizeof path, "%.*s/libtrimatch_ref.so", slash ? (int)(slash - self) : 1, slash ? self : ".");
      void* h = dlopen(path, RTLD_NOW);
      if (!h) {
        fprintf(stderr, "dlopen %s: %s\n", path, dlerror());
        return 1;
      }
      void* (*gnew)(const uint64_t*, const uint32_t*, uint32_t, uint64_t) =
          (void* (*)(const uint64_t*, const uint32_t*, uint32_t, uint64_t))dlsym(h, "ref_graph_new");
      int (*sipv)(void*, int, uint64_t*, uint64_t*) =
          (int (*)(void*, int, uint64_t*, uint64_t*))dlsym(h, "ref_segmented_intersect_pv");
      /* trimatch::Graph takes its own copies (graph.cpp:9-21 validates them) */
      void* g = gnew(off, adj, n, E);
      if (!g) {
        fprintf(stderr, "ref_graph_new failed\n");
        return 1;
      }
      free(adj);
      adj = NULL;
      if (sipv(g, threads, &T, pv) != 0) {
        fprintf(stderr, "ref_segmented_intersect_pv failed\n");
        return 1;
      }
      source = "reference segmented_intersect with listings (frontier.cpp:51-81), chunked";
    } else {
      fprintf(stderr, "unknown mode %s\n", mode);
      return 2;
    }
    t_count = now_s() - t1;
  }
  printf("{\"kind\": \"%s\", \"scale\": %d, \"edgefactor\": %d, \"permute\": %s, \"n\": %u, \"m\": %llu, "
         "\"pairs_fnv\": \"%016llx\", \"E\": %llu, \"loops\": %llu, \"dups\": %llu, "
         "\"offsets_fnv\": \"%016llx\", \"nbrs_fnv\": \"%016llx\"",
         kind == 1 ? "er" : "rmat", scale, param, permute ? "true" : "false", n, (unsigned long long)m,
         (unsigned long long)hp, (unsigned long long)E, (unsigned long long)loops, (unsigned long long)dups,
         (unsigned long long)off_fnv, (unsigned long long)nb_fnv);
  if (pv) {
    uint64_t s = 0, mx = 0, am = 0;
    for (uint64_t v = 0; v < n; ++v) {
      s += pv[v];
      if (pv[v] > mx) {
        mx = pv[v];
        am = v;
      }
    }
    printf(", \"T\": %llu, \"pv_fnv\": \"%016llx\", \"pv_sum\": %llu, \"pv_max\": %llu, \"pv_argmax\": %llu, "
           "\"source\": \"%s\", \"count_s\": %.1f, \"build_s\": %.1f",
           (unsigned long long)T, (unsigned long long)oracle_fnv1a64(pv, (uint64_t)n * 8),
           (unsigned long long)s, (unsigned long long)mx, (unsigned long long)am, source, t_count, t_build);
  }
  printf("}\n");
  free(pv);
  free(adj);
  free(off);
  return 0;
}
