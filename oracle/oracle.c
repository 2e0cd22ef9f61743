/*
 * oracle.c -- CPU restatement of the reference triangle-counting path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  The product never links this file.
 * Each function cites the reference file:line it follows (relative to
 * /root/reference/proj).  Parity of this restatement with the reference is
 * pinned by tests/test_oracle.py against oracle/_ref (the reference sources
 * compiled unmodified except for the 2-token compile fix documented in
 * oracle/Makefile) and against the fixtures under tests/golden/.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- generators: SURVEY.md section 8d, bit-exact ------------------------ */

static inline uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t oracle_rmat_num_edges(int scale, int edgefactor) {
  return (uint64_t)edgefactor << scale;
}

uint64_t oracle_er_num_edges(int scale, int avg_degree) {
  return ((uint64_t)avg_degree << scale) / 2;
}

void oracle_gen_rmat(int scale, int edgefactor, int permute, uint32_t* pairs) {
  const uint64_t m = oracle_rmat_num_edges(scale, edgefactor);
  const double A = .57, B = .19, C = .19;
  const double AB = A + B, ABC = AB + C; /* left-to-right IEEE double sums */
#pragma omp parallel for schedule(static)
  for (int64_t ii = 0; ii < (int64_t)m; ++ii) {
    const uint64_t i = (uint64_t)ii;
    uint64_t st = sm64(i * 0x100000001ULL + 12345ULL);
    uint32_t u = 0, v = 0;
    for (int b = 0; b < scale; ++b) {
      st = sm64(st);
      const double p = (double)(st >> 11) * 0x1.0p-53;
      const uint32_t ub = p > AB;
      const uint32_t vb = (p > A && p <= AB) || p > ABC;
      u |= ub << b;
      v |= vb << b;
    }
    pairs[2 * i] = u;
    pairs[2 * i + 1] = v;
  }
  if (permute) {
    const uint64_t n = 1ULL << scale;
    uint32_t* perm = (uint32_t*)malloc(n * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    for (uint64_t i = n - 1; i >= 1; --i) {
      const uint64_t j = sm64(0xABCDEFULL ^ i) % (i + 1);
      const uint32_t t = perm[i];
      perm[i] = perm[j];
      perm[j] = t;
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)(2 * m); ++i) pairs[i] = perm[pairs[i]];
    free(perm);
  }
}

void oracle_gen_er(int scale, int avg_degree, uint32_t* pairs) {
  const uint64_t m = oracle_er_num_edges(scale, avg_degree);
  const uint64_t mask = (1ULL << scale) - 1;
#pragma omp parallel for schedule(static)
  for (int64_t ii = 0; ii < (int64_t)m; ++ii) {
    const uint64_t i = (uint64_t)ii;
    uint64_t st = sm64(i * 0x100000001ULL + 12345ULL);
    st = sm64(st);
    const uint32_t u = (uint32_t)(st & mask);
    st = sm64(st);
    const uint32_t v = (uint32_t)(st & mask);
    pairs[2 * i] = u;
    pairs[2 * i + 1] = v;
  }
}

/* ---- build_graph: graph.cpp:33-85 --------------------------------------- */

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

int oracle_build_graph(const uint32_t* pairs, uint64_t m, uint32_t n,
                       uint64_t** offsets_out, uint32_t** nbrs_out, uint64_t* num_edges,
                       uint64_t* self_loops, uint64_t* dups) {
  /* graph.cpp:38-49: count both orientations, skip loops, range check. */
  uint64_t* offsets = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t loops = 0;
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u >= n || v >= n) {
      free(offsets);
      return -1; /* std::invalid_argument, graph.cpp:40-42 */
    }
    if (u == v) {
      ++loops;
      continue;
    }
    ++offsets[u + 1];
    ++offsets[v + 1];
  }
  /* graph.cpp:50 serial prefix */
  for (uint64_t u = 0; u < n; ++u) offsets[u + 1] += offsets[u];
  /* graph.cpp:52-58 scatter both orientations */
  uint32_t* adj = (uint32_t*)malloc((offsets[n] ? offsets[n] : 1) * sizeof(uint32_t));
  uint64_t* cursor = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
  memcpy(cursor, offsets, ((size_t)n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    if (u == v) continue;
    adj[cursor[u]++] = v;
    adj[cursor[v]++] = u;
  }
  free(cursor);
  /* graph.cpp:61-76 per-vertex sort + unique; rows sorted independently
   * (parallel), then compacted serially exactly as the reference does. */
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t u = 0; u < (int64_t)n; ++u) {
    const uint64_t b = offsets[u], e = offsets[u + 1];
    if (e - b > 1) qsort(adj + b, e - b, sizeof(uint32_t), cmp_u32);
  }
  uint64_t* new_off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t write = 0, dup = 0;
  for (uint64_t u = 0; u < n; ++u) {
    const uint64_t b = offsets[u], e = offsets[u + 1];
    uint64_t out = write;
    for (uint64_t i = b; i < e; ++i) {
      if (out == write || adj[out - 1] != adj[i]) {
        adj[out++] = adj[i];
      } else {
        ++dup;
      }
    }
    write = out;
    new_off[u + 1] = write;
  }
  free(offsets);
  /* graph.cpp:80-81: each duplicate directed entry was inserted twice */
  dup /= 2;
  *offsets_out = new_off;
  *nbrs_out = adj;
  *num_edges = write / 2;
  if (self_loops) *self_loops = loops;
  if (dups) *dups = dup;
  return 0;
}

void oracle_free(void* p) { free(p); }

/* ---- segmented intersection count: frontier.cpp:14-81 ------------------- */

static uint64_t upper_bound_u32(const uint32_t* a, uint64_t n, uint32_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] <= key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

static int binary_search_u32(const uint32_t* a, uint64_t n, uint32_t key) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo < n && a[lo] == key;
}

/* frontier.cpp:10 kProbeRatio */
#define ORACLE_PROBE_RATIO 32

/* intersect_sorted (frontier.cpp:14-47) with bounded=true, floor=dst.
 * Common vertices are reported to `out` (nullable) in ascending order. */
static uint64_t intersect_above(const uint32_t* a, uint64_t na, const uint32_t* b, uint64_t nb,
                                uint32_t floor, uint32_t* out) {
  const uint64_t sa = upper_bound_u32(a, na, floor), sb = upper_bound_u32(b, nb, floor);
  a += sa; na -= sa;
  b += sb; nb -= sb;
  if (na > nb) {
    const uint32_t* t = a; a = b; b = t;
    const uint64_t tn = na; na = nb; nb = tn;
  }
  uint64_t count = 0;
  if (na * ORACLE_PROBE_RATIO < nb) { /* frontier.cpp:23-31 probe */
    for (uint64_t i = 0; i < na; ++i)
      if (binary_search_u32(b, nb, a[i])) {
        if (out) out[count] = a[i];
        ++count;
      }
    return count;
  }
  uint64_t i = 0, j = 0; /* frontier.cpp:33-45 merge */
  while (i < na && j < nb) {
    if (a[i] < b[j]) ++i;
    else if (b[j] < a[i]) ++j;
    else {
      if (out) out[count] = a[i];
      ++count; ++i; ++j;
    }
  }
  return count;
}

uint64_t oracle_count(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n,
                      uint64_t* per_vertex, int threads) {
  uint64_t total = 0;
  if (per_vertex) memset(per_vertex, 0, (size_t)n * sizeof(uint64_t));
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#else
  (void)threads;
#endif
  /* Pairs {(u,v): v in N(u), u<v} in (u, adjacency) order, exactly the
   * edge frontier SPEC.md:376 feeds segmented_intersect with
   * above_dst_only=true.  Listings (when per_vertex) give triangles
   * (u, v, w) with u<v<w (frontier.cpp:65-79). */
#pragma omp parallel num_threads(threads) reduction(+ : total)
  {
    uint32_t* buf = NULL;
    uint64_t cap = 0;
#pragma omp for schedule(dynamic, 64)
    for (int64_t uu = 0; uu < (int64_t)n; ++uu) {
      const uint32_t u = (uint32_t)uu;
      const uint32_t* nu = nbrs + offsets[u];
      const uint64_t du = offsets[u + 1] - offsets[u];
      uint64_t tu = 0;
      if (per_vertex && du > cap) {
        free(buf);
        cap = du;
        buf = (uint32_t*)malloc(cap * sizeof(uint32_t));
      }
      for (uint64_t k = upper_bound_u32(nu, du, u); k < du; ++k) {
        const uint32_t v = nu[k];
        const uint32_t* nv = nbrs + offsets[v];
        const uint64_t dv = offsets[v + 1] - offsets[v];
        const uint64_t c = intersect_above(nu, du, nv, dv, v, per_vertex ? buf : NULL);
        total += c;
        if (per_vertex && c) {
          tu += c;
#pragma omp atomic
          per_vertex[v] += c;
          for (uint64_t i = 0; i < c; ++i) {
#pragma omp atomic
            per_vertex[buf[i]] += 1;
          }
        }
      }
      if (per_vertex && tu) {
#pragma omp atomic
        per_vertex[u] += tu;
      }
    }
    free(buf);
  }
  return total;
}

/* ---- brute force: SPEC.md:347-365 --------------------------------------- */

static int has_edge(const uint64_t* offsets, const uint32_t* nbrs, uint32_t u, uint32_t v) {
  /* graph.cpp:23-31 binary search in N(u) */
  return binary_search_u32(nbrs + offsets[u], offsets[u + 1] - offsets[u], v);
}

uint64_t oracle_brute_force(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n) {
  if (n > 5000) return UINT64_MAX;
  uint64_t count = 0;
  for (uint32_t a = 0; a < n; ++a)
    for (uint32_t b = a + 1; b < n; ++b) {
      if (!has_edge(offsets, nbrs, a, b)) continue;
      for (uint32_t c = b + 1; c < n; ++c)
        if (has_edge(offsets, nbrs, a, c) && has_edge(offsets, nbrs, b, c)) ++count;
    }
  return count;
}

uint64_t oracle_fnv1a64(const void* data, uint64_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ---- CPU-baseline sampling support --------------------------------------- */

/* cost[u] = deg(u) * |{w in N(u): w > u}| -- the visits the reference's final
 * level makes for seed u (matcher.cpp:215-228 visits N(u) for each level-1
 * row (u,w), w > u).  Used to stratify and extrapolate the bounded sample. */
void oracle_seed_costs(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n, double* cost) {
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t uu = 0; uu < (int64_t)n; ++uu) {
    const uint32_t u = (uint32_t)uu;
    const uint64_t b = offsets[u], e = offsets[u + 1];
    const uint64_t up = e - b - upper_bound_u32(nbrs + b, e - b, u);
    cost[u] = (double)(e - b) * (double)up;
  }
}

/* ---- DAG statistics for the work model ------------------- */

void oracle_dag_stats(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n,
                      double* W, double* S2, double* J, uint32_t* max_dplus) {
  /* (deg,id) orientation: u->v iff (deg u, u) < (deg v, v). */
  uint32_t* dplus = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
  uint32_t mx = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(max : mx)
  for (int64_t uu = 0; uu < (int64_t)n; ++uu) {
    const uint32_t u = (uint32_t)uu;
    const uint64_t du = offsets[u + 1] - offsets[u];
    uint32_t c = 0;
    for (uint64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
      const uint32_t v = nbrs[k];
      const uint64_t dv = offsets[v + 1] - offsets[v];
      if (du < dv || (du == dv && u < v)) ++c;
    }
    dplus[u] = c;
    if (c > mx) mx = c;
  }
  double w = 0, s2 = 0, j = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : w, s2, j)
  for (int64_t uu = 0; uu < (int64_t)n; ++uu) {
    const uint32_t u = (uint32_t)uu;
    const uint64_t du = offsets[u + 1] - offsets[u];
    s2 += (double)dplus[u] * dplus[u];
    for (uint64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
      const uint32_t v = nbrs[k];
      const uint64_t dv = offsets[v + 1] - offsets[v];
      if (du < dv || (du == dv && u < v)) w += dplus[v];
    }
  }
  /* J = sum over oriented (u->v) with d+(v)>0 of #{x in N+(u): x after v in
   * rank order}; computed per u by sorting its out-list ranks implicitly:
   * the suffix length of v in N+(u) ordered by (deg,id). */
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : j)
  for (int64_t uu = 0; uu < (int64_t)n; ++uu) {
    const uint32_t u = (uint32_t)uu;
    const uint64_t du = offsets[u + 1] - offsets[u];
    for (uint64_t k = offsets[u]; k < offsets[u + 1]; ++k) {
      const uint32_t v = nbrs[k];
      const uint64_t dv = offsets[v + 1] - offsets[v];
      if (!(du < dv || (du == dv && u < v)) || dplus[v] == 0) continue;
      /* count out-neighbours x of u ranked above v */
      uint64_t after = 0;
      for (uint64_t q = offsets[u]; q < offsets[u + 1]; ++q) {
        const uint32_t x = nbrs[q];
        const uint64_t dx = offsets[x + 1] - offsets[x];
        if ((du < dx || (du == dx && u < x)) && (dv < dx || (dv == dx && v < x))) ++after;
      }
      j += (double)after;
    }
  }
  free(dplus);
  *W = w;
  *S2 = s2;
  *J = j;
  if (max_dplus) *max_dplus = mx;
}

/* ---- degree-ordered DAG count: the independent big-config checker -------- */

/* SURVEY.md 8c "planned GPU algorithm, validated on the host": orient by
 * (deg, id), every triangle a<b<c (ranks) is found once with pivot b -- for
 * each in-edge a->b scan the suffix of N+(a) after b and test membership in
 * N+(b).  Same counts as segmented_intersect with above_dst_only
 * (frontier.cpp:51-81) because both are total orders; the
 * per-vertex histogram is t[a], t[b], t[c] += 1 per triangle, as the
 * reference's listings give it (frontier.cpp:65-79, matcher.hpp:92).  It
 * exists because the id-order restatement above needs hours at C5 (RMAT s26
 * ef32); tests/test_oracle.py pins it against the reference goldens before it
 * is trusted.  J = sum_a C(d+(a),2) bitmap probes instead of the id-order
 * merge's sum over id-ordered pairs. */
static int cmp_u32b(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

uint64_t oracle_count_dag(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n,
                          uint64_t* per_vertex, int threads) {
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_max_threads();
#else
  threads = 1;
#endif
  if (per_vertex) memset(per_vertex, 0, (size_t)n * sizeof(uint64_t));
  if (n == 0) return 0;
  /* rank = position of (deg, id): counting sort by degree, stable in id */
  uint64_t maxd = 0;
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t d = offsets[v + 1] - offsets[v];
    if (d > maxd) maxd = d;
  }
  uint64_t* bucket = (uint64_t*)calloc(maxd + 2, sizeof(uint64_t));
  for (uint64_t v = 0; v < n; ++v) ++bucket[offsets[v + 1] - offsets[v] + 1];
  for (uint64_t d = 0; d <= maxd; ++d) bucket[d + 1] += bucket[d];
  uint32_t* order = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  uint32_t* rank = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t r = bucket[offsets[v + 1] - offsets[v]]++;
    order[r] = (uint32_t)v;
    rank[v] = (uint32_t)r;
  }
  free(bucket);
  /* oriented CSR in rank space (rows sorted) and its transpose (in-edges) */
  uint64_t* oo = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
  uint64_t* io = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4096)
  for (int64_t rr = 0; rr < (int64_t)n; ++rr) {
    const uint32_t v = order[rr];
    uint64_t c = 0;
    for (uint64_t k = offsets[v]; k < offsets[v + 1]; ++k) c += rank[nbrs[k]] > (uint32_t)rr;
    oo[rr + 1] = c;
    io[rr + 1] = (offsets[v + 1] - offsets[v]) - c;
  }
  for (uint64_t r = 0; r < n; ++r) {
    oo[r + 1] += oo[r];
    io[r + 1] += io[r];
  }
  const uint64_t E = oo[n];
  uint32_t* oc = (uint32_t*)malloc((E ? E : 1) * sizeof(uint32_t));
  uint32_t* ic = (uint32_t*)malloc((E ? E : 1) * sizeof(uint32_t));
  uint64_t* icur = (uint64_t*)malloc((size_t)n * sizeof(uint64_t));
  memcpy(icur, io, (size_t)n * sizeof(uint64_t));
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1024)
  for (int64_t rr = 0; rr < (int64_t)n; ++rr) {
    const uint32_t v = order[rr];
    uint64_t p = oo[rr];
    for (uint64_t k = offsets[v]; k < offsets[v + 1]; ++k) {
      const uint32_t x = rank[nbrs[k]];
      if (x > (uint32_t)rr) {
        oc[p++] = x;
        const uint64_t q = __atomic_fetch_add(&icur[x], 1, __ATOMIC_RELAXED);
        ic[q] = (uint32_t)rr;
      }
    }
    if (p - oo[rr] > 1) qsort(oc + oo[rr], p - oo[rr], sizeof(uint32_t), cmp_u32b);
  }
  free(icur);
  free(rank);
  /* pivot join: per-thread membership bitmap and per-vertex counters */
  const uint64_t words = ((uint64_t)n + 63) / 64;
  uint64_t total = 0;
  uint64_t** tl = (uint64_t**)calloc((size_t)threads, sizeof(uint64_t*));
#pragma omp parallel num_threads(threads) reduction(+ : total)
  {
#ifdef _OPENMP
    const int tid = omp_get_thread_num();
#else
    const int tid = 0;
#endif
    uint64_t* bm = (uint64_t*)calloc(words, sizeof(uint64_t));
    uint64_t* t = per_vertex ? (uint64_t*)calloc((size_t)n, sizeof(uint64_t)) : NULL;
    tl[tid] = t;
#pragma omp for schedule(dynamic, 64)
    for (int64_t bb = (int64_t)n - 1; bb >= 0; --bb) {
      const uint32_t b = (uint32_t)bb;
      const uint64_t b0 = oo[b], b1 = oo[b + 1];
      if (b1 == b0 || io[b + 1] == io[b]) continue;
      for (uint64_t k = b0; k < b1; ++k) bm[oc[k] >> 6] |= 1ull << (oc[k] & 63);
      uint64_t hb = 0;
      for (uint64_t q = io[b]; q < io[b + 1]; ++q) {
        const uint32_t a = ic[q];
        const uint32_t* na = oc + oo[a];
        const uint64_t da = oo[a + 1] - oo[a];
        uint64_t c = 0;
        for (uint64_t k = upper_bound_u32(na, da, b); k < da; ++k) {
          const uint32_t x = na[k];
          if ((bm[x >> 6] >> (x & 63)) & 1) {
            ++c;
            if (t) ++t[x];
          }
        }
        if (t) t[a] += c;
        hb += c;
      }
      if (t) t[b] += hb;
      total += hb;
      for (uint64_t k = b0; k < b1; ++k) bm[oc[k] >> 6] = 0;
    }
    free(bm);
  }
  if (per_vertex) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t rr = 0; rr < (int64_t)n; ++rr) {
      uint64_t s = 0;
      for (int t = 0; t < threads; ++t) s += tl[t][rr];
      per_vertex[order[rr]] = s;
    }
    for (int t = 0; t < threads; ++t) free(tl[t]);
  }
  free(tl);
  free(oo);
  free(io);
  free(oc);
  free(ic);
  free(order);
  return total;
}

/* ---- streamed generation for the big-config goldens ---------------------- */

/* Edges [i0, i1) of the SURVEY 8d generators (kind 0 = RMAT/Kronecker,
 * 1 = ER), bit-identical to oracle_gen_rmat / oracle_gen_er; perm (nullable)
 * is the Kronecker relabelling of oracle_kron_perm.  Lets a driver build a
 * 2^31-edge graph without holding the 17 GB pair array. */
void oracle_gen_range(int kind, int scale, int param, uint64_t i0, uint64_t i1, const uint32_t* perm,
                      uint32_t* pairs) {
  const double A = .57, B = .19, C = .19;
  const double AB = A + B, ABC = AB + C;
  const uint64_t mask = (1ULL << scale) - 1;
  (void)param;
#pragma omp parallel for schedule(static)
  for (int64_t ii = (int64_t)i0; ii < (int64_t)i1; ++ii) {
    const uint64_t i = (uint64_t)ii;
    uint64_t st = sm64(i * 0x100000001ULL + 12345ULL);
    uint32_t u = 0, v = 0;
    if (kind == 1) {
      st = sm64(st);
      u = (uint32_t)(st & mask);
      st = sm64(st);
      v = (uint32_t)(st & mask);
    } else {
      for (int b = 0; b < scale; ++b) {
        st = sm64(st);
        const double p = (double)(st >> 11) * 0x1.0p-53;
        u |= (uint32_t)(p > AB) << b;
        v |= (uint32_t)((p > A && p <= AB) || p > ABC) << b;
      }
      if (perm) {
        u = perm[u];
        v = perm[v];
      }
    }
    pairs[2 * (i - i0)] = u;
    pairs[2 * (i - i0) + 1] = v;
  }
}

void oracle_kron_perm(int scale, uint32_t* perm) {
  const uint64_t n = 1ULL << scale;
  for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
  for (uint64_t i = n - 1; i >= 1; --i) {
    const uint64_t j = sm64(0xABCDEFULL ^ i) % (i + 1);
    const uint32_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
}
