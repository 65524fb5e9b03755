/*
 * trilist_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference `trilist` AOT path
 * (/root/reference/proj, C++20).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker.  The product (paper_2006_11494_b200) never links it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks this restatement against
 * the reference's own known-answer tests (restated values) and
 * against the reference itself compiled from /root/reference by
 * oracle/Makefile into oracle/_ref/libtrilist_ref.so.
 *
 * Every function cites the reference file:line it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* splitmix64 -- ordering.cpp:13-19, testutil.hpp:79-85                      */
/* ------------------------------------------------------------------------ */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ull;

OR_API uint64_t or_fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* k-th output (0-based) of the sequential splitmix64 seeded with `seed`. */
OR_API uint64_t or_draw(uint64_t seed, uint64_t k) { return or_fmix64(seed + (k + 1) * kGolden); }

/* Order-independent triangle hash (round-2 definition,
 * the one oracle/ref_shim.cpp's HashSink applies to the reference's own
 * emissions): every vertex has the word Z(v) = fmix64(v + golden) of its
 * original id; a triangle adds Z(a) Z(b) Z(c) mod 2^64 to hash_sum and xors
 * Z(a) & Z(b) & Z(c) into hash_xor.  Both are symmetric in the three ids. */
OR_API uint64_t or_vertex_word(uint32_t v) { return or_fmix64((uint64_t)v + kGolden); }
OR_API uint64_t or_triangle_hash_xor(uint32_t a, uint32_t b, uint32_t c) {
  return or_vertex_word(a) & or_vertex_word(b) & or_vertex_word(c);
}
OR_API uint64_t or_triangle_hash(uint32_t a, uint32_t b, uint32_t c) {  /* the hash_sum term */
  return or_vertex_word(a) * or_vertex_word(b) * or_vertex_word(c);
}

static void canon3(uint32_t* x, uint32_t* y, uint32_t* z) { /* graph.cpp:148-153 */
  uint32_t t;
  if (*x > *y) { t = *x; *x = *y; *y = t; }
  if (*y > *z) { t = *y; *y = *z; *z = t; }
  if (*x > *y) { t = *x; *x = *y; *y = t; }
}

/* ------------------------------------------------------------------------ */
/* Synthetic generators.  The GPU library implements the same */
/* definitions; tests check them bit-for-bit.                                 */
/* ------------------------------------------------------------------------ */

/* ER config C1: acceptance.cpp:305-316 pair-draw pattern. */
OR_API void or_gen_er(uint64_t seed, uint32_t n, uint64_t npairs, uint32_t* pairs) {
  for (uint64_t i = 0; i < npairs; ++i) {
    uint64_t d = or_draw(seed, i);
    pairs[2 * i] = (uint32_t)((d >> 32) % n);
    pairs[2 * i + 1] = (uint32_t)((d & 0xFFFFFFFFull) % n);
  }
}

/* Bijection on [0, 2^bits): every step (xor, odd multiply, xorshift, add) is
 * invertible modulo 2^bits. */
OR_API uint32_t or_permute_id(uint64_t seed, uint32_t bits, uint32_t x) {
  const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  const uint32_t sh = (bits + 1) / 2;
  uint64_t k1 = or_fmix64(seed ^ 0xA5A5A5A5A5A5A5A5ull);
  uint64_t k2 = or_fmix64(seed ^ 0x5A5A5A5A5A5A5A5Aull);
  uint64_t v = ((uint64_t)x ^ k1) & mask;
  v = (v * 0x9E3779B1ull) & mask;
  v ^= v >> sh;
  v = (v * 0x85EBCA77ull) & mask;
  v ^= v >> sh;
  v = (v + k2) & mask;
  return (uint32_t)v;
}

/* R-MAT quadrant thresholds floor(p * 2^64) for p = 0.57, 0.76, 0.95. */
#define RMAT_T1 10514644122014444421ull
#define RMAT_T2 14019525496019259228ull
#define RMAT_T3 17524406870024074035ull

/* R-MAT (a,b,c,d)=(.57,.19,.19,.05), MSB-first; draw(seed, i*scale + level);
 * ids then scrambled by or_permute_id(seed, scale, .). */
OR_API void or_gen_rmat(uint64_t seed, uint32_t scale, uint64_t npairs, uint32_t* pairs) {
  for (uint64_t i = 0; i < npairs; ++i) {
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      uint64_t d = or_draw(seed, i * scale + l);
      uint32_t ub = d >= RMAT_T2;                           /* quadrants c, d */
      uint32_t vb = (d >= RMAT_T1 && d < RMAT_T2) || d >= RMAT_T3; /* b, d */
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    pairs[2 * i] = or_permute_id(seed, scale, u);
    pairs[2 * i + 1] = or_permute_id(seed, scale, v);
  }
}

/* Chung-Lu expected-degree weights: w_i = (1-U_i)^(-1/(gamma-1)), rescaled to
 * mean `avg`, capped at sqrt(n*avg), integerised to fixed point 2^20; the
 * output is the exclusive prefix (n+1 entries). */
OR_API void or_chung_lu_prefix(uint64_t seed, uint32_t n, double avg, double gamma,
                               uint64_t* prefix) {
  double* w = (double*)malloc(sizeof(double) * (n ? n : 1));
  double sum = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    double u = (double)(or_draw(seed, i) >> 11) * (1.0 / 9007199254740992.0);
    w[i] = pow(1.0 - u, -1.0 / (gamma - 1.0));
    sum += w[i];
  }
  double scale = (n && sum > 0) ? avg * (double)n / sum : 0.0;
  double cap = sqrt((double)n * avg);
  prefix[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    double x = w[i] * scale;
    if (x > cap) x = cap;
    prefix[i + 1] = prefix[i] + (uint64_t)(x * 1048576.0);
  }
  free(w);
}

static uint32_t upper_slot(const uint64_t* prefix, uint32_t n, uint64_t r) {
  /* the i with prefix[i] <= r < prefix[i+1] */
  uint32_t lo = 0, hi = n; /* invariant: prefix[lo] <= r < prefix[hi] */
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (prefix[mid] <= r) lo = mid; else hi = mid;
  }
  return lo;
}

OR_API void or_gen_chung_lu(uint64_t seed, uint32_t n, const uint64_t* prefix, uint64_t npairs,
                            uint32_t* pairs) {
  uint64_t total = prefix[n];
  uint64_t s2 = or_fmix64(seed ^ 0xC0FFEEull);
  for (uint64_t i = 0; i < npairs; ++i) {
    pairs[2 * i] = upper_slot(prefix, n, or_draw(s2, 2 * i) % total);
    pairs[2 * i + 1] = upper_slot(prefix, n, or_draw(s2, 2 * i + 1) % total);
  }
}

/* gnp(n, p, seed): testutil.hpp:89-97 -- one sequential splitmix64 draw per
 * pair u<v against floor(p * (2^64-1)).  Returns the pair count; writes up to
 * cap pairs. */
OR_API uint64_t or_gen_gnp(uint32_t n, double p, uint64_t seed, uint32_t* pairs, uint64_t cap) {
  uint64_t state = seed, cnt = 0;
  uint64_t threshold = (uint64_t)(p * 18446744073709551615.0);
  for (uint32_t u = 0; u < n; ++u)
    for (uint32_t v = u + 1; v < n; ++v) {
      state += kGolden;
      if (or_fmix64(state) < threshold) {
        if (cnt < cap) { pairs[2 * cnt] = u; pairs[2 * cnt + 1] = v; }
        ++cnt;
      }
    }
  return cnt;
}

/* ------------------------------------------------------------------------ */
/* Graph::from_edges / build_from_packed -- graph.cpp:158-206                */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint32_t n;
  uint64_t m;
  uint64_t* off; /* n+1 */
  uint32_t* adj; /* 2m, ascending per vertex */
  uint64_t duplicates;
} or_graph;

static void radix_sort_u64(uint64_t* a, uint64_t len) {
  if (len < 2) return;
  uint64_t* tmp = (uint64_t*)malloc(sizeof(uint64_t) * len);
  uint64_t* src = a;
  uint64_t* dst = tmp;
  for (int pass = 0; pass < 4; ++pass) {
    int sh = pass * 16;
    uint64_t* cnt = (uint64_t*)calloc(65537, sizeof(uint64_t));
    for (uint64_t i = 0; i < len; ++i) cnt[((src[i] >> sh) & 0xFFFF) + 1]++;
    for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
    for (uint64_t i = 0; i < len; ++i) dst[cnt[(src[i] >> sh) & 0xFFFF]++] = src[i];
    free(cnt);
    uint64_t* t = src; src = dst; dst = t;
  }
  /* 4 passes: result back in `a` */
  free(tmp);
}

OR_API or_graph* or_from_edges(uint32_t min_vertices, const uint32_t* pairs, uint64_t npairs) {
  uint64_t n = min_vertices;
  uint64_t* packed = (uint64_t*)malloc(sizeof(uint64_t) * (npairs ? npairs : 1));
  uint64_t k = 0;
  for (uint64_t i = 0; i < npairs; ++i) { /* graph.cpp:193-198 */
    uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
    uint32_t hi = u > v ? u : v, lo = u > v ? v : u;
    if ((uint64_t)hi + 1 > n) n = (uint64_t)hi + 1;
    if (u == v) continue;
    packed[k++] = ((uint64_t)lo << 32) | hi;
  }
  radix_sort_u64(packed, k); /* graph.cpp:160 */
  uint64_t m = 0;
  for (uint64_t i = 0; i < k; ++i) /* std::unique, graph.cpp:161 */
    if (i == 0 || packed[i] != packed[i - 1]) packed[m++] = packed[i];

  or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
  g->n = (uint32_t)n;
  g->m = m;
  g->duplicates = k - m;
  g->off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  g->adj = (uint32_t*)malloc(sizeof(uint32_t) * (2 * m ? 2 * m : 1));
  for (uint64_t i = 0; i < m; ++i) { /* graph.cpp:168-171 */
    g->off[(uint32_t)(packed[i] >> 32) + 1]++;
    g->off[(uint32_t)packed[i] + 1]++;
  }
  for (uint64_t i = 1; i <= n; ++i) g->off[i] += g->off[i - 1];
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  memcpy(cur, g->off, sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < m; ++i) { /* graph.cpp:179-185 */
    uint32_t lo = (uint32_t)(packed[i] >> 32), hi = (uint32_t)packed[i];
    g->adj[cur[lo]++] = hi;
    g->adj[cur[hi]++] = lo;
  }
  free(cur);
  free(packed);
  return g;
}

OR_API void or_graph_free(or_graph* g) {
  if (!g) return;
  free(g->off);
  free(g->adj);
  free(g);
}
OR_API uint32_t or_graph_n(const or_graph* g) { return g->n; }
OR_API uint64_t or_graph_m(const or_graph* g) { return g->m; }
OR_API uint64_t or_graph_duplicates(const or_graph* g) { return g->duplicates; }
OR_API void or_graph_csr(const or_graph* g, uint64_t* off, uint32_t* adj) {
  memcpy(off, g->off, sizeof(uint64_t) * (g->n + 1ull));
  memcpy(adj, g->adj, sizeof(uint32_t) * 2 * g->m);
}

static uint32_t gdeg(const or_graph* g, uint32_t u) { return (uint32_t)(g->off[u + 1] - g->off[u]); }

static int has_edge(const or_graph* g, uint32_t u, uint32_t v) { /* graph.cpp:213-217 */
  if (u >= g->n || v >= g->n) return 0;
  uint64_t lo = g->off[u], hi = g->off[u + 1];
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (g->adj[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo < g->off[u + 1] && g->adj[lo] == v;
}

/* ------------------------------------------------------------------------ */
/* degree_order -- ordering.cpp:69-84 (counting sort by degree, ties by id)  */
/* ------------------------------------------------------------------------ */
OR_API void or_degree_order(const or_graph* g, uint32_t* rank) {
  uint32_t maxd = 0;
  for (uint32_t u = 0; u < g->n; ++u) if (gdeg(g, u) > maxd) maxd = gdeg(g, u);
  uint64_t* start = (uint64_t*)calloc((size_t)maxd + 2, sizeof(uint64_t));
  for (uint32_t u = 0; u < g->n; ++u) start[gdeg(g, u) + 1]++;
  for (size_t d = 1; d < (size_t)maxd + 2; ++d) start[d] += start[d - 1];
  for (uint32_t u = 0; u < g->n; ++u) rank[u] = (uint32_t)(start[gdeg(g, u)]++);
  free(start);
}

/* ------------------------------------------------------------------------ */
/* orient -- ordering.cpp:185-227; OrientedGraph ordering.hpp:62-108          */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint32_t n;
  uint64_t m;
  uint64_t *out_off, *in_off;
  uint32_t *out, *in, *rank;
} or_oriented;

/* Returns NULL unless rank is a permutation of 0..n-1 (ordering.cpp:187-188). */
OR_API or_oriented* or_orient(const or_graph* g, const uint32_t* rank) {
  uint32_t n = g->n;
  uint32_t* by_rank = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  unsigned char* seen = (unsigned char*)calloc(n ? n : 1, 1);
  for (uint32_t u = 0; u < n; ++u) {
    if (rank[u] >= n || seen[rank[u]]) { free(seen); free(by_rank); return NULL; }
    seen[rank[u]] = 1;
    by_rank[rank[u]] = u;
  }
  free(seen);
  or_oriented* og = (or_oriented*)calloc(1, sizeof(or_oriented));
  og->n = n;
  og->m = g->m;
  og->out_off = (uint64_t*)calloc(n + 1ull, sizeof(uint64_t));
  og->in_off = (uint64_t*)calloc(n + 1ull, sizeof(uint64_t));
  og->out = (uint32_t*)malloc(sizeof(uint32_t) * (g->m ? g->m : 1));
  og->in = (uint32_t*)malloc(sizeof(uint32_t) * (g->m ? g->m : 1));
  og->rank = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  memcpy(og->rank, rank, sizeof(uint32_t) * n);
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
      uint32_t v = g->adj[i];
      if (rank[u] < rank[v]) { og->out_off[u + 1]++; og->in_off[v + 1]++; }
    }
  for (uint32_t u = 0; u < n; ++u) {
    og->out_off[u + 1] += og->out_off[u];
    og->in_off[u + 1] += og->in_off[u];
  }
  uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  memcpy(cur, og->out_off, sizeof(uint64_t) * n);
  for (uint32_t r = 0; r < n; ++r) { /* heads in ascending rank: rank-sorted lists */
    uint32_t head = by_rank[r];
    for (uint64_t i = g->off[head]; i < g->off[head + 1]; ++i) {
      uint32_t tail = g->adj[i];
      if (rank[tail] < r) og->out[cur[tail]++] = head;
    }
  }
  memcpy(cur, og->in_off, sizeof(uint64_t) * n);
  for (uint32_t r = 0; r < n; ++r) {
    uint32_t tail = by_rank[r];
    for (uint64_t i = g->off[tail]; i < g->off[tail + 1]; ++i) {
      uint32_t head = g->adj[i];
      if (rank[head] > r) og->in[cur[head]++] = tail;
    }
  }
  free(cur);
  free(by_rank);
  return og;
}

OR_API void or_oriented_free(or_oriented* og) {
  if (!og) return;
  free(og->out_off); free(og->in_off); free(og->out); free(og->in); free(og->rank);
  free(og);
}
OR_API uint64_t or_oriented_m(const or_oriented* og) { return og->m; }
OR_API void or_oriented_csr(const or_oriented* og, uint64_t* out_off, uint32_t* out,
                            uint64_t* in_off, uint32_t* in, uint32_t* rank) {
  uint64_t n1 = og->n + 1ull;
  if (out_off) memcpy(out_off, og->out_off, sizeof(uint64_t) * n1);
  if (in_off) memcpy(in_off, og->in_off, sizeof(uint64_t) * n1);
  if (out) memcpy(out, og->out, sizeof(uint32_t) * og->m);
  if (in) memcpy(in, og->in, sizeof(uint32_t) * og->m);
  if (rank) memcpy(rank, og->rank, sizeof(uint32_t) * og->n);
}

static uint32_t odeg(const or_oriented* g, uint32_t u) {
  return (uint32_t)(g->out_off[u + 1] - g->out_off[u]);
}
/* out_degree_before -- ordering.hpp:86-89: lexicographic (deg+, id). */
static int before(const or_oriented* g, uint32_t a, uint32_t b) {
  uint32_t da = odeg(g, a), db = odeg(g, b);
  return da != db ? da < db : a < b;
}

OR_API uint32_t or_max_out_degree(const or_oriented* og) { /* ordering.cpp:178-182 */
  uint32_t best = 0;
  for (uint32_t u = 0; u < og->n; ++u) if (odeg(og, u) > best) best = odeg(og, u);
  return best;
}

/* cost_model -- engine.cpp:37-49: out[0]=cf, out[1]=kclist, out[2]=aot. */
OR_API void or_cost_model(const or_oriented* og, uint64_t* out) {
  uint64_t cf = 0, kc = 0, aot = 0;
  for (uint32_t u = 0; u < og->n; ++u) {
    uint64_t du = odeg(og, u);
    for (uint64_t i = og->out_off[u]; i < og->out_off[u + 1]; ++i) {
      uint64_t dv = odeg(og, og->out[i]);
      cf += du + dv;
      kc += dv;
      aot += du < dv ? du : dv;
    }
  }
  out[0] = cf; out[1] = kc; out[2] = aot;
}

/* ------------------------------------------------------------------------ */
/* aot_pivot + sequential driver -- engine.hpp:238-276, :294-304             */
/* stats: [0]=triangles [1]=probes [2]=merge_comparisons [3]=table_builds     */
/*        [4]=positive [5]=negative [6]=hash_sum [7]=hash_xor                 */
/* Raw emissions (pivot, neighbor, witness) are written to out (if non-null)  */
/* up to cap triples; the return value is the emission count.                */
/* ------------------------------------------------------------------------ */
OR_API uint64_t or_aot(const or_oriented* g, int skip_negative, uint64_t* stats, uint32_t* out,
                       uint64_t cap) {
  uint64_t s[8] = {0};
  uint64_t words = ((uint64_t)g->n + 63) / 64;
  uint64_t* bm = (uint64_t*)calloc(words ? words : 1, sizeof(uint64_t)); /* bitmap.hpp:11-32 */
  uint64_t emitted = 0;
#define OR_EMIT(a, b, c, polarity)                                          \
  do {                                                                      \
    s[0]++; s[polarity]++;                                                  \
    uint32_t e0_ = (a), e1_ = (b), e2_ = (c);                               \
    if (out && emitted < cap) {                                             \
      out[3 * emitted] = e0_; out[3 * emitted + 1] = e1_; out[3 * emitted + 2] = e2_; \
    }                                                                       \
    emitted++;                                                              \
    canon3(&e0_, &e1_, &e2_);                                               \
    s[6] += or_triangle_hash(e0_, e1_, e2_);                                \
    s[7] ^= or_triangle_hash_xor(e0_, e1_, e2_);                            \
  } while (0)
  for (uint32_t u = 0; u < g->n; ++u) {
    uint64_t ub = g->out_off[u], ue = g->out_off[u + 1];
    for (uint64_t i = ub; i < ue; ++i) bm[g->out[i] >> 6] |= 1ull << (g->out[i] & 63);
    s[3] += ue - ub;
    for (uint64_t i = ub; i < ue; ++i) { /* positive phase, engine.hpp:247-257 */
      uint32_t v = g->out[i];
      if (!before(g, v, u)) continue;
      for (uint64_t j = g->out_off[v]; j < g->out_off[v + 1]; ++j) {
        uint32_t w = g->out[j];
        s[1]++;
        if ((bm[w >> 6] >> (w & 63)) & 1) OR_EMIT(u, v, w, 4);
      }
    }
    if (!skip_negative) { /* negative phase, engine.hpp:259-272 */
      for (uint64_t i = g->in_off[u]; i < g->in_off[u + 1]; ++i) {
        uint32_t x = g->in[i];
        if (!before(g, x, u)) continue;
        for (uint64_t j = g->out_off[x]; j < g->out_off[x + 1]; ++j) {
          uint32_t y = g->out[j];
          s[1]++;
          if ((bm[y >> 6] >> (y & 63)) & 1) OR_EMIT(u, x, y, 5);
        }
      }
    }
    for (uint64_t i = ub; i < ue; ++i) bm[g->out[i] >> 6] &= ~(1ull << (g->out[i] & 63));
  }
#undef OR_EMIT
  free(bm);
  memcpy(stats, s, sizeof(s));
  return emitted;
}

/* ------------------------------------------------------------------------ */
/* The comparison kernels -- engine.hpp:164-236 (cf merge, cf hash, kclist3), */
/* sequential driver engine.hpp:294-304.  algo: 0 = cf (merge), 1 = cf-hash,  */
/* 2 = kclist.  Same stats/emission conventions as or_aot; `reuse` is         */
/* RunOptions::cf_hash_reuse_last_table (engine.hpp:58).  The cf-hash probe   */
/* structure is a set; a bitmap gives the same membership answers, and the    */
/* counters only count insertions and look-ups (engine.hpp:200-215).          */
/* cf (merge) compares ranks (engine.hpp:168) on the current list layout.     */
/* ------------------------------------------------------------------------ */
OR_API uint64_t or_kernel(const or_oriented* g, int algo, int reuse, uint64_t* stats, uint32_t* out,
                          uint64_t cap) {
  uint64_t s[8] = {0};
  uint64_t words = ((uint64_t)g->n + 63) / 64;
  uint64_t* bm = (uint64_t*)calloc(words ? words : 1, sizeof(uint64_t));
  uint64_t emitted = 0;
#define OR_EMIT3(a, b, c)                                                   \
  do {                                                                      \
    s[0]++;                                                                 \
    uint32_t e0_ = (a), e1_ = (b), e2_ = (c);                               \
    if (out && emitted < cap) {                                             \
      out[3 * emitted] = e0_; out[3 * emitted + 1] = e1_; out[3 * emitted + 2] = e2_; \
    }                                                                       \
    emitted++;                                                              \
    canon3(&e0_, &e1_, &e2_);                                               \
    s[6] += or_triangle_hash(e0_, e1_, e2_);                                \
    s[7] ^= or_triangle_hash_xor(e0_, e1_, e2_);                            \
  } while (0)
#define OR_SET(list_b, list_e, on)                                          \
  for (uint64_t q_ = (list_b); q_ < (list_e); ++q_) {                       \
    uint32_t x_ = g->out[q_];                                               \
    if (on) bm[x_ >> 6] |= 1ull << (x_ & 63); else bm[x_ >> 6] &= ~(1ull << (x_ & 63)); \
  }
  for (uint32_t u = 0; u < g->n; ++u) {
    uint64_t ub = g->out_off[u], ue = g->out_off[u + 1];
    if (algo == 0) { /* cf_merge_pivot, engine.hpp:164-184 */
      for (uint64_t k = ub; k < ue; ++k) {
        uint32_t v = g->out[k];
        uint64_t i = ub, j = g->out_off[v], je = g->out_off[v + 1];
        while (i < ue && j < je) {
          s[2]++;
          uint32_t ri = g->rank[g->out[i]], rj = g->rank[g->out[j]];
          if (ri < rj) ++i;
          else if (rj < ri) ++j;
          else { OR_EMIT3(u, v, g->out[i]); ++i; ++j; }
        }
      }
    } else if (algo == 1) { /* cf_hash_pivot, engine.hpp:186-215 */
      int64_t cached = -1; /* kNoOwner: the cache never survives the pivot */
      for (uint64_t k = ub; k < ue; ++k) {
        uint32_t v = g->out[k];
        int hash_u = before(g, v, u);
        uint32_t owner = hash_u ? u : v;
        uint64_t bb = hash_u ? ub : g->out_off[v], be = hash_u ? ue : g->out_off[v + 1];
        uint64_t pb = hash_u ? g->out_off[v] : ub, pe = hash_u ? g->out_off[v + 1] : ue;
        if (!reuse || (int64_t)owner != cached) {
          if (cached >= 0) {
            uint32_t c = (uint32_t)cached;
            OR_SET(g->out_off[c], g->out_off[c + 1], 0);
          }
          OR_SET(bb, be, 1);
          s[3] += be - bb;
          cached = owner;
        }
        for (uint64_t q = pb; q < pe; ++q) {
          uint32_t w = g->out[q];
          s[1]++;
          if ((bm[w >> 6] >> (w & 63)) & 1) OR_EMIT3(u, v, w);
        }
        if (!reuse) { OR_SET(bb, be, 0); cached = -1; }
      }
      if (cached >= 0) {
        uint32_t c = (uint32_t)cached;
        OR_SET(g->out_off[c], g->out_off[c + 1], 0);
      }
    } else { /* kclist3_pivot, engine.hpp:217-236 */
      OR_SET(ub, ue, 1);
      s[3] += ue - ub;
      for (uint64_t k = ub; k < ue; ++k) {
        uint32_t v = g->out[k];
        for (uint64_t q = g->out_off[v]; q < g->out_off[v + 1]; ++q) {
          uint32_t w = g->out[q];
          s[1]++;
          if ((bm[w >> 6] >> (w & 63)) & 1) OR_EMIT3(u, v, w);
        }
      }
      OR_SET(ub, ue, 0);
    }
  }
#undef OR_SET
#undef OR_EMIT3
  free(bm);
  memcpy(stats, s, sizeof(s));
  return emitted;
}

/* Rewrites the out-lists of og in place: 0 = rank-asc, 1 = degree-desc,     */
/* 2 = random:seed (ordering.cpp:229-266, out-lists only: the kernels above  */
/* read no in-list).                                                          */
static uint64_t or_splitmix(uint64_t* state) { /* ordering.cpp:13-19 */
  *state += kGolden;
  return or_fmix64(*state);
}
static uint64_t or_bounded(uint64_t* state, uint64_t bound) { /* ordering.cpp:23-26 */
  return (uint64_t)(((unsigned __int128)or_splitmix(state) * bound) >> 64);
}
static void or_fisher_yates(uint32_t* a, uint64_t n, uint64_t seed) { /* ordering.cpp:28-34 */
  uint64_t state = seed;
  for (uint64_t i = n; i > 1; --i) {
    uint64_t j = or_bounded(&state, i);
    uint32_t t = a[i - 1]; a[i - 1] = a[j]; a[j] = t;
  }
}
static const or_oriented* g_sort_ctx;
static int g_sort_policy;
static int or_cmp_local(const void* pa, const void* pb) {
  uint32_t x = *(const uint32_t*)pa, y = *(const uint32_t*)pb;
  const or_oriented* g = g_sort_ctx;
  if (g_sort_policy == 1) {
    uint64_t dx = (g->out_off[x + 1] - g->out_off[x]) + (g->in_off[x + 1] - g->in_off[x]);
    uint64_t dy = (g->out_off[y + 1] - g->out_off[y]) + (g->in_off[y + 1] - g->in_off[y]);
    if (dx != dy) return dx > dy ? -1 : 1;
    return x < y ? -1 : (x > y);
  }
  return g->rank[x] < g->rank[y] ? -1 : (g->rank[x] > g->rank[y]);
}
OR_API void or_apply_local_order(or_oriented* g, int policy, uint64_t seed) {
  g_sort_ctx = g;
  g_sort_policy = policy == 1 ? 1 : 0;
  for (uint32_t u = 0; u < g->n; ++u) {
    uint64_t b = g->out_off[u], len = g->out_off[u + 1] - b;
    qsort(g->out + b, len, sizeof(uint32_t), or_cmp_local);
    if (policy == 2) {
      uint64_t mix = seed;
      uint64_t key = or_splitmix(&mix) ^ (((uint64_t)u << 1) | 0u);
      or_fisher_yates(g->out + b, len, key);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* degeneracy_order -- ordering.cpp:86-114: repeatedly remove the vertex of  */
/* least (current degree, id).  A binary heap over packed (deg << 32 | id)   */
/* with lazy deletion, as the reference.                                     */
/* ------------------------------------------------------------------------ */
static void heap_push(uint64_t* h, uint64_t* len, uint64_t x) {
  uint64_t i = (*len)++;
  h[i] = x;
  while (i) {
    uint64_t p = (i - 1) / 2;
    if (h[p] <= h[i]) break;
    uint64_t t = h[p]; h[p] = h[i]; h[i] = t;
    i = p;
  }
}
static uint64_t heap_pop(uint64_t* h, uint64_t* len) {
  uint64_t top = h[0];
  h[0] = h[--(*len)];
  uint64_t i = 0;
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, k = i;
    if (l < *len && h[l] < h[k]) k = l;
    if (r < *len && h[r] < h[k]) k = r;
    if (k == i) break;
    uint64_t t = h[k]; h[k] = h[i]; h[i] = t;
    i = k;
  }
  return top;
}
OR_API void or_degeneracy_order(const or_graph* g, uint32_t* rank) {
  uint32_t n = g->n;
  uint32_t* deg = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
  unsigned char* removed = (unsigned char*)calloc(n ? n : 1, 1);
  uint64_t* heap = (uint64_t*)malloc(sizeof(uint64_t) * ((uint64_t)n + 2 * g->m + 1));
  uint64_t len = 0;
  for (uint32_t u = 0; u < n; ++u) {
    deg[u] = gdeg(g, u);
    heap_push(heap, &len, ((uint64_t)deg[u] << 32) | u);
  }
  for (uint32_t r = 0; r < n; ++r) {
    uint32_t u;
    for (;;) {
      uint64_t top = heap_pop(heap, &len);
      u = (uint32_t)top;
      if (!removed[u] && (uint32_t)(top >> 32) == deg[u]) break;
    }
    removed[u] = 1;
    rank[u] = r;
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
      uint32_t v = g->adj[i];
      if (!removed[v]) heap_push(heap, &len, ((uint64_t)(--deg[v]) << 32) | v);
    }
  }
  free(heap); free(removed); free(deg);
}

/* random_order -- ordering.cpp:116-120: Fisher-Yates of the identity. */
OR_API void or_random_order(uint32_t n, uint64_t seed, uint32_t* rank) {
  for (uint32_t u = 0; u < n; ++u) rank[u] = u;
  or_fisher_yates(rank, n, seed);
}

/* ------------------------------------------------------------------------ */
/* brute_force_triangles -- oracle.cpp:8-25 (sorted, duplicate-free)          */
/* ------------------------------------------------------------------------ */
OR_API uint64_t or_brute_force(const or_graph* g, uint32_t* out, uint64_t cap) {
  uint64_t cnt = 0;
  for (uint32_t u = 0; u < g->n; ++u)
    for (uint64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
      uint32_t v = g->adj[i];
      if (v <= u) continue;
      for (uint64_t j = g->off[u]; j < g->off[u + 1]; ++j) {
        uint32_t w = g->adj[j];
        if (w <= v) continue;
        if (has_edge(g, v, w)) {
          if (out && cnt < cap) { out[3 * cnt] = u; out[3 * cnt + 1] = v; out[3 * cnt + 2] = w; }
          cnt++;
        }
      }
    }
  return cnt;
}
