/*
 * tcmis_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A sequential, plain-C restatement of the reference TC-MIS path.  Every
 * function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py only.  Its parity with the reference is pinned
 * by tests/test_oracle.py against oracle/_ref (the reference compiled from its
 * own sources by oracle/Makefile) and against tests/golden/.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off; the H2 priority and
 * the G(n,p) gap arithmetic must round exactly like the reference).
 */
#include "tcmis_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9e3779b97f4a7c15ULL

/* ---------------------------------------------------------------- hashing */

/* priorities.cpp:15-19 -- splitmix64 finalizer */
uint64_t orc_mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* priorities.cpp:21-23 */
uint64_t orc_vertex_hash(uint64_t v, uint64_t seed) {
  return orc_mix64(orc_mix64(seed) + (v + 1) * GOLDEN);
}

/* priorities.cpp:25-27 -- 53 high bits scaled by 2^-53 */
double orc_hash_to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

/* priorities.cpp:29-31 */
uint64_t orc_combine_seed(uint64_t seed, uint64_t round) {
  return orc_mix64(seed + orc_mix64(round + GOLDEN));
}

/* ------------------------------------------------------------- priorities */

/* priorities.cpp:33-41 */
int orc_h1_random(int32_t n, uint64_t seed, uint32_t *p) {
  if (n < 1) return 1;
  for (int32_t v = 0; v < n; ++v) p[v] = (uint32_t)(orc_vertex_hash((uint64_t)v, seed) >> 32);
  return 0;
}

/* priorities.cpp:43-51 (denominator floor 1/1024 from priorities.cpp:12) */
uint32_t orc_h2_priority_value(double avg, int32_t deg, double eps, int scale_bits) {
  double d = avg + (double)deg - eps;
  if (d < 1.0 / 1024.0) d = 1.0 / 1024.0;
  double s = floor(avg / d * ldexp(1.0, scale_bits));
  if (s < 0.0) return 0u;
  if (s >= 4294967295.0) return 0xffffffffu;
  return (uint32_t)s;
}

/* priorities.cpp:53-67 */
int orc_h2_degree_aware(int32_t n, const int64_t *off, uint64_t seed, int scale_bits,
                        uint32_t *p) {
  if (scale_bits < 8 || scale_bits > 30) return 1;
  if (n == 0) return 0;
  int64_t m = off[n] / 2; /* graph.hpp:23-25 num_edges */
  double avg = 2.0 * (double)m / (double)n;
  for (int32_t v = 0; v < n; ++v) {
    double eps = orc_hash_to_unit(orc_vertex_hash((uint64_t)v, seed));
    p[v] = orc_h2_priority_value(avg, (int32_t)(off[v + 1] - off[v]), eps, scale_bits);
  }
  return 0;
}

/* priorities.hpp:61-64 -- (p, id+1) key, never 0 */
static inline uint64_t key_of(const uint32_t *p, int32_t v) {
  return ((uint64_t)p[v] << 32) | ((uint64_t)(uint32_t)v + 1u);
}

/* ------------------------------------------------------------ phase funcs */

/* engine.cpp:86-103 */
void orc_compute_max_np(int32_t n, const int64_t *off, const int32_t *nbr, const uint32_t *p,
                        const uint8_t *st, uint64_t *out) {
  for (int32_t v = 0; v < n; ++v) {
    uint64_t best = 0; /* kNoNeighborKey, priorities.hpp:57 */
    if (st[v] == 0) {
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int32_t u = nbr[e];
        if (st[u] != 0) continue;
        uint64_t k = key_of(p, u);
        if (k > best) best = k;
      }
    }
    out[v] = best;
  }
}

/* spmv.cpp:61-73 */
void orc_csr_neighbor_count(int32_t n, const int64_t *off, const int32_t *nbr, const uint8_t *c,
                            int32_t *nc) {
  for (int32_t v = 0; v < n; ++v) {
    int32_t cnt = 0;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) cnt += c[nbr[e]] != 0;
    nc[v] = cnt;
  }
}

/* engine.cpp:121-160 (the newly-selected append is done by the caller) */
int orc_phase3_update(int32_t n, uint8_t *st, const uint8_t *c, const int32_t *nc, int64_t *sel,
                      int64_t *rem) {
  int64_t s = 0, r = 0;
  for (int32_t v = 0; v < n; ++v) {
    if (c[v]) {
      if (st[v] != 0) return 3; /* logic_error, engine.cpp:152-153 */
      st[v] = 1;
      ++s;
    } else if (st[v] == 0 && nc[v] > 0) {
      st[v] = 2;
      ++r;
    }
  }
  *sel = s;
  *rem = r;
  return 0;
}

/* engine.cpp:231-295 (fixed priorities) and engine.cpp:301-352 (fresh). */
int orc_luby_rounds(int32_t n, const int64_t *off, const int32_t *nbr, const uint32_t *p,
                    int fresh, uint64_t seed, const int64_t *tile_col_count, int T,
                    uint8_t *state_out, orc_round *rounds, int max_rounds) {
  if (n == 0) return 0; /* engine.cpp:240 */
  uint8_t *st = (uint8_t *)calloc((size_t)n, 1);
  uint8_t *c = (uint8_t *)malloc((size_t)n);
  uint64_t *mx = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  int32_t *nc = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  uint32_t *pf = fresh ? (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n) : NULL;
  int32_t nseg = T > 0 ? (n + T - 1) / T : 0;
  uint8_t *segflag = tile_col_count ? (uint8_t *)malloc((size_t)nseg + 1) : NULL;
  int64_t total_tiles = 0;
  if (tile_col_count)
    for (int32_t b = 0; b < nseg; ++b) total_tiles += tile_col_count[b];

  int64_t alive = n;
  int it = 0;
  int status = 0;
  while (alive > 0) {
    ++it;
    if (it > n || it > max_rounds) { status = -1; break; } /* engine.cpp:248-249 */
    const uint32_t *pr = p;
    if (fresh) { /* engine.cpp:324-325 */
      orc_h1_random(n, orc_combine_seed(seed, (uint64_t)it), pf);
      pr = pf;
    }
    orc_compute_max_np(n, off, nbr, pr, st, mx);
    /* engine.cpp:105-119 generate_candidates */
    orc_round *R = &rounds[it - 1];
    memset(R, 0, sizeof(*R));
    for (int32_t v = 0; v < n; ++v) {
      c[v] = (st[v] == 0 && key_of(pr, v) > mx[v]) ? 1 : 0;
      if (st[v] == 0) {
        int64_t d = off[v + 1] - off[v];
        R->alive_start++;
        R->nnz_alive += d;
        if (c[v]) R->nnz_cand += d;
        else { R->noncand++; R->nnz_noncand += d; }
      }
    }
    orc_csr_neighbor_count(n, off, nbr, c, nc);
    if (tile_col_count) { /* spmv.cpp:37-46 skip rule, counted per block column */
      memset(segflag, 0, (size_t)nseg);
      for (int32_t v = 0; v < n; ++v)
        if (c[v]) segflag[v / T] = 1;
      int64_t ev = 0;
      for (int32_t b = 0; b < nseg; ++b)
        if (segflag[b]) ev += tile_col_count[b];
      R->tiles_eval = ev;
      R->tiles_skip = total_tiles - ev;
    }
    int64_t s = 0, r = 0;
    if (orc_phase3_update(n, st, c, nc, &s, &r)) { status = -3; break; }
    alive -= s + r;
    R->sel = s;
    R->rem = r;
    R->alive = alive;
  }
  if (state_out) memcpy(state_out, st, (size_t)n);
  free(st); free(c); free(mx); free(nc); free(pf); free(segflag);
  return status ? status : it;
}

/* engine.cpp:162-229 */
int orc_h3_resolution(int32_t n, const int64_t *off, const int32_t *nbr, const uint32_t *p,
                      const uint8_t *states, uint8_t *c) {
  uint8_t *pend = (uint8_t *)malloc((size_t)n + 1);
  uint8_t *win = (uint8_t *)malloc((size_t)n + 1);
  int64_t remaining = 0;
  for (int32_t v = 0; v < n; ++v) {
    c[v] = 0;
    pend[v] = states[v] == 0;
    remaining += pend[v];
  }
  int inner = 0;
  while (remaining > 0) {
    ++inner;
    for (int32_t v = 0; v < n; ++v) {
      win[v] = 0;
      if (!pend[v]) continue;
      uint64_t k = key_of(p, v);
      int dom = 1;
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int32_t u = nbr[e];
        if (pend[u] && key_of(p, u) >= k) { dom = 0; break; }
      }
      win[v] = (uint8_t)dom;
    }
    int64_t dropped = 0;
    for (int32_t v = 0; v < n; ++v) {
      if (!pend[v]) continue;
      if (win[v]) { c[v] = 1; pend[v] = 0; ++dropped; continue; }
      for (int64_t e = off[v]; e < off[v + 1]; ++e)
        if (win[nbr[e]]) { pend[v] = 0; ++dropped; break; }
    }
    if (dropped == 0) { inner = -1; break; } /* engine.cpp:224-225 */
    remaining -= dropped;
  }
  free(pend);
  free(win);
  return inner;
}

/* ------------------------------------------------------------- radix sort */

static void radix_sort_u64(uint64_t *a, int64_t n, int bits) {
  if (n < 2) return;
  uint64_t *buf = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  uint64_t *src = a, *dst = buf;
  int64_t cnt[2048];
  for (int shift = 0; shift < bits; shift += 11) {
    memset(cnt, 0, sizeof(cnt));
    for (int64_t i = 0; i < n; ++i) cnt[(src[i] >> shift) & 2047]++;
    int64_t s = 0;
    for (int d = 0; d < 2048; ++d) { int64_t c = cnt[d]; cnt[d] = s; s += c; }
    for (int64_t i = 0; i < n; ++i) dst[cnt[(src[i] >> shift) & 2047]++] = src[i];
    uint64_t *t = src; src = dst; dst = t;
  }
  if (src != a) memcpy(a, src, sizeof(uint64_t) * (size_t)n);
  free(buf);
}

/* tests/support/oracles.cpp:76-92 */
int64_t orc_greedy_mis(int32_t n, const int64_t *off, const int32_t *nbr, const uint32_t *p,
                       uint8_t *member) {
  /* sort (p, id) keys descending: sort ~key ascending.  Keys need 64 bits. */
  uint64_t *k = (uint64_t *)malloc(sizeof(uint64_t) * ((size_t)n + 1));
  for (int32_t v = 0; v < n; ++v) k[v] = ~key_of(p, v);
  radix_sort_u64(k, n, 64);
  uint8_t *blocked = (uint8_t *)calloc((size_t)n + 1, 1);
  int64_t cnt = 0;
  if (n > 0) memset(member, 0, (size_t)n);
  for (int32_t i = 0; i < n; ++i) {
    int32_t v = (int32_t)((uint32_t)(~k[i]) - 1u);
    if (blocked[v]) continue;
    member[v] = 1;
    ++cnt;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) blocked[nbr[e]] = 1;
  }
  free(k);
  free(blocked);
  return cnt;
}

/* ----------------------------------------------------------------- tiling */

static int cmp_i32(const void *a, const void *b) {
  int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
  return (x > y) - (x < y);
}

/* tiling.cpp:44-84 -- distinct block columns per block row, ascending, with
 * the T row words ORed per tile.  A last-seen marker per block column keeps
 * it O(nnz + tiles log tiles). */
int64_t orc_tile_graph(int32_t n, const int64_t *off, const int32_t *nbr, int T,
                       int32_t *tile_row, int32_t *tile_col, uint64_t *row_bits,
                       int64_t *bro) {
  if (T < 1 || T > 64) return -1; /* tiling.cpp:17-21 */
  int32_t nb = (n + T - 1) / T;
  int32_t *seen = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nb + 1));
  int32_t *slot = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nb + 1));
  int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nb + 1));
  for (int32_t b = 0; b < nb; ++b) seen[b] = -1;
  int64_t total = 0;
  if (bro) bro[0] = 0;
  for (int32_t br = 0; br < nb; ++br) {
    int32_t lo = br * T, hi = lo + T < n ? lo + T : n;
    int32_t ncols = 0;
    for (int32_t v = lo; v < hi; ++v)
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int32_t bc = nbr[e] / T;
        if (seen[bc] != br) { seen[bc] = br; cols[ncols++] = bc; }
      }
    if (row_bits) {
      qsort(cols, (size_t)ncols, sizeof(int32_t), cmp_i32);
      for (int32_t i = 0; i < ncols; ++i) {
        slot[cols[i]] = i;
        tile_row[total + i] = br;
        tile_col[total + i] = cols[i];
      }
      memset(row_bits + total * T, 0, sizeof(uint64_t) * (size_t)ncols * (size_t)T);
      for (int32_t v = lo; v < hi; ++v)
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
          int32_t u = nbr[e];
          row_bits[(total + slot[u / T]) * T + (v - lo)] |= 1ULL << (u % T);
        }
    }
    total += ncols;
    if (bro) bro[br + 1] = total;
  }
  free(seen); free(slot); free(cols);
  return total;
}

int64_t orc_tile_row_counts(int32_t n, const int64_t *off, const int32_t *nbr, int T,
                            int64_t *rowtiles) {
  if (T < 1 || T > 64) return -1;
  int32_t nb = (n + T - 1) / T;
  int32_t *seen = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nb + 1));
  for (int32_t b = 0; b < nb; ++b) seen[b] = -1;
  int64_t total = 0;
  for (int32_t br = 0; br < nb; ++br) {
    int32_t lo = br * T, hi = lo + T < n ? lo + T : n;
    int64_t cnt = 0;
    for (int32_t v = lo; v < hi; ++v)
      for (int64_t e = off[v]; e < off[v + 1]; ++e) {
        int32_t bc = nbr[e] / T;
        if (seen[bc] != br) { seen[bc] = br; ++cnt; }
      }
    rowtiles[br] = cnt;
    total += cnt;
  }
  free(seen);
  return total;
}

/* tiling.cpp:86-101 */
void orc_pack_segments(int32_t n, const uint8_t *values, int T, uint64_t *seg) {
  int32_t ns = (n + T - 1) / T;
  for (int32_t s = 0; s < ns; ++s) seg[s] = 0;
  for (int32_t k = 0; k < n; ++k)
    if (values[k]) seg[k / T] |= 1ULL << (k % T);
}

/* spmv.cpp:12-16 + spmv.cpp:18-59 */
int orc_tiled_spmv(int32_t n, int T, int64_t tile_count, const int32_t *tile_col,
                   const uint64_t *row_bits, const int64_t *bro, const uint64_t *seg,
                   int32_t *nc, int64_t *evaluated, int64_t *skipped) {
  (void)tile_count;
  int32_t nb = (n + T - 1) / T;
  int64_t ev = 0, sk = 0;
  for (int32_t br = 0; br < nb; ++br) {
    int32_t acc[64] = {0};
    for (int64_t t = bro[br]; t < bro[br + 1]; ++t) {
      uint64_t s = seg[tile_col[t]];
      if (s == 0) { ++sk; continue; }
      ++ev;
      for (int i = 0; i < T; ++i) acc[i] += __builtin_popcountll(row_bits[t * T + i] & s);
    }
    for (int i = 0; i < T && br * T + i < n; ++i) nc[br * T + i] = acc[i];
  }
  *evaluated = ev;
  *skipped = sk;
  return 0;
}

/* ------------------------------------------------------------- generators */

static orc_graph *graph_alloc(int32_t n, int64_t nnz) {
  orc_graph *g = (orc_graph *)calloc(1, sizeof(orc_graph));
  g->n = n;
  g->nnz = nnz;
  g->off = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  g->nbr = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nnz + 1));
  return g;
}

void orc_graph_free(orc_graph *g) {
  if (!g) return;
  free(g->off);
  free(g->nbr);
  free(g);
}

/* graph.cpp:14-41 -- drop loops, add reverse edges, sort, dedupe */
orc_graph *orc_graph_from_edges(int32_t n, int64_t m, const int32_t *eu, const int32_t *ev) {
  if (n < 0) return NULL;
  uint64_t *k = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
  int64_t cnt = 0;
  for (int64_t i = 0; i < m; ++i) {
    int32_t u = eu[i], v = ev[i];
    if (u < 0 || u >= n || v < 0 || v >= n) { free(k); return NULL; }
    if (u == v) continue;
    k[cnt++] = ((uint64_t)(uint32_t)u << 32) | (uint32_t)v;
    k[cnt++] = ((uint64_t)(uint32_t)v << 32) | (uint32_t)u;
  }
  radix_sort_u64(k, cnt, 64);
  int64_t w = 0;
  for (int64_t i = 0; i < cnt; ++i)
    if (w == 0 || k[i] != k[w - 1]) k[w++] = k[i];
  orc_graph *g = graph_alloc(n, w);
  for (int64_t i = 0; i < w; ++i) {
    g->off[(k[i] >> 32) + 1]++;
    g->nbr[i] = (int32_t)(uint32_t)k[i];
  }
  for (int32_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
  free(k);
  return g;
}

/* generate.cpp:15-26: the i-th draw of SplitMix64(seed) is vertex_hash(i, seed) */
typedef struct { uint64_t state; } orc_rng;
static inline uint64_t rng_next(orc_rng *r) {
  r->state += GOLDEN;
  return orc_mix64(r->state);
}

/* generate.cpp:30-61 */
orc_graph *orc_gnp(int32_t n, double p, uint64_t seed) {
  if (n < 0) return NULL;
  if (p <= 0.0 || n < 2) return orc_graph_from_edges(n, 0, NULL, NULL);
  if (p >= 1.0) {
    int64_t m = (int64_t)n * (n - 1) / 2, i = 0;
    int32_t *eu = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    int32_t *ev = (int32_t *)malloc(sizeof(int32_t) * (size_t)m);
    for (int32_t u = 0; u < n; ++u)
      for (int32_t v = u + 1; v < n; ++v) { eu[i] = u; ev[i] = v; ++i; }
    orc_graph *g = orc_graph_from_edges(n, m, eu, ev);
    free(eu); free(ev);
    return g;
  }
  orc_rng rng = {orc_mix64(seed)};
  const double log_q = log1p(-p);
  const int64_t total = (int64_t)n * (n - 1) / 2;
  int64_t cap = 1024, m = 0;
  int32_t *eu = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
  int32_t *ev = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
  int64_t idx = -1, row = 0, row_start = 0, row_len = n - 1;
  for (;;) {
    double u = orc_hash_to_unit(rng_next(&rng));
    int64_t gap = (int64_t)floor(log1p(-u) / log_q);
    idx += 1 + gap;
    if (idx >= total) break;
    while (idx - row_start >= row_len) { row_start += row_len; ++row; --row_len; }
    if (m == cap) {
      cap *= 2;
      eu = (int32_t *)realloc(eu, sizeof(int32_t) * (size_t)cap);
      ev = (int32_t *)realloc(ev, sizeof(int32_t) * (size_t)cap);
    }
    eu[m] = (int32_t)row;
    ev[m] = (int32_t)(row + 1 + (idx - row_start));
    ++m;
  }
  orc_graph *g = orc_graph_from_edges(n, m, eu, ev);
  free(eu); free(ev);
  return g;
}

/* generate.cpp:63-66 */
orc_graph *orc_gnp_avg_degree(int32_t n, double avg_degree, uint64_t seed) {
  double p = n > 1 ? avg_degree / (double)(n - 1) : 0.0;
  return orc_gnp(n, p, seed);
}

/* generate.cpp:68-98 */
orc_graph *orc_rmat(int scale, int ef, uint64_t seed) {
  if (scale < 1 || scale > 30 || ef < 1) return NULL;
  int32_t n = (int32_t)1 << scale;
  int64_t samples = (int64_t)ef * n;
  int32_t *eu = (int32_t *)malloc(sizeof(int32_t) * (size_t)samples);
  int32_t *ev = (int32_t *)malloc(sizeof(int32_t) * (size_t)samples);
  orc_rng rng = {orc_mix64(seed)};
  for (int64_t e = 0; e < samples; ++e) {
    int32_t u = 0, v = 0;
    for (int l = 0; l < scale; ++l) {
      double r = orc_hash_to_unit(rng_next(&rng));
      u <<= 1;
      v <<= 1;
      if (r < 0.57) {
      } else if (r < 0.76) {
        v |= 1;
      } else if (r < 0.95) {
        u |= 1;
      } else {
        u |= 1;
        v |= 1;
      }
    }
    eu[e] = u;
    ev[e] = v;
  }
  orc_graph *g = orc_graph_from_edges(n, samples, eu, ev);
  free(eu); free(ev);
  return g;
}

/* New definition (no reference generator): side x side 4-neighbour mesh,
 * id = i*side + j. */
orc_graph *orc_grid(int32_t side) {
  int64_t n = (int64_t)side * side;
  int64_t nnz = side > 1 ? 4LL * side * (side - 1) : 0;
  orc_graph *g = graph_alloc((int32_t)n, nnz);
  int64_t w = 0;
  for (int32_t i = 0; i < side; ++i)
    for (int32_t j = 0; j < side; ++j) {
      int32_t v = i * side + j;
      if (i > 0) g->nbr[w++] = v - side;
      if (j > 0) g->nbr[w++] = v - 1;
      if (j + 1 < side) g->nbr[w++] = v + 1;
      if (i + 1 < side) g->nbr[w++] = v + side;
      g->off[v + 1] = w;
    }
  return g;
}

/* New definition: integer random geometric graph.  Point v is
 * (vertex_hash(2v, seed) >> 32, vertex_hash(2v+1, seed) >> 32) on the 2^32
 * lattice; u ~ v iff dx^2 + dy^2 <= R^2 exactly in u64, with
 * R = floor(sqrt(avg/(pi n)) * 2^32) computed once on the host. */
uint64_t orc_rgg_radius(int32_t n, double avg_degree) {
  if (n <= 0 || avg_degree <= 0.0) return 0;
  double r = sqrt(avg_degree / (3.14159265358979323846 * (double)n));
  double R = floor(r * 4294967296.0);
  if (R > 4294967295.0) R = 4294967295.0;
  return (uint64_t)R;
}

static int cmp_i32_asc(const void *a, const void *b) { return cmp_i32(a, b); }

orc_graph *orc_rgg(int32_t n, double avg_degree, uint64_t seed) {
  uint64_t R = orc_rgg_radius(n, avg_degree);
  if (n <= 0 || R == 0) return orc_graph_from_edges(n < 0 ? 0 : n, 0, NULL, NULL);
  uint32_t *x = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  uint32_t *y = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  for (int32_t v = 0; v < n; ++v) {
    x[v] = (uint32_t)(orc_vertex_hash(2ULL * (uint64_t)v, seed) >> 32);
    y[v] = (uint32_t)(orc_vertex_hash(2ULL * (uint64_t)v + 1, seed) >> 32);
  }
  uint64_t C = (4294967295ULL / R) + 1; /* cells per side, cell = coord / R */
  uint64_t ncell = C * C;
  int64_t *cs = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
  for (int32_t v = 0; v < n; ++v) cs[(x[v] / R) * C + (y[v] / R) + 1]++;
  for (uint64_t c = 0; c < ncell; ++c) cs[c + 1] += cs[c];
  int32_t *pts = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)ncell);
  memcpy(fill, cs, sizeof(int64_t) * (size_t)ncell);
  for (int32_t v = 0; v < n; ++v) pts[fill[(x[v] / R) * C + (y[v] / R)]++] = v;
  free(fill);
  uint64_t R2 = R * R;
  orc_graph *g = NULL;
  for (int pass = 0; pass < 2; ++pass) {
    int64_t w = 0;
    for (int32_t v = 0; v < n; ++v) {
      int64_t cx = x[v] / R, cy = y[v] / R;
      int64_t start = w;
      for (int64_t ax = cx - 1; ax <= cx + 1; ++ax) {
        if (ax < 0 || ax >= (int64_t)C) continue;
        for (int64_t ay = cy - 1; ay <= cy + 1; ++ay) {
          if (ay < 0 || ay >= (int64_t)C) continue;
          uint64_t c = (uint64_t)ax * C + (uint64_t)ay;
          for (int64_t q = cs[c]; q < cs[c + 1]; ++q) {
            int32_t u = pts[q];
            if (u == v) continue;
            uint64_t dx = x[u] > x[v] ? x[u] - x[v] : x[v] - x[u];
            uint64_t dy = y[u] > y[v] ? y[u] - y[v] : y[v] - y[u];
            if (dx > R || dy > R) continue;
            if (dx * dx + dy * dy <= R2) {
              if (pass == 1) g->nbr[w] = u;
              ++w;
            }
          }
        }
      }
      if (pass == 1) {
        qsort(g->nbr + start, (size_t)(w - start), sizeof(int32_t), cmp_i32_asc);
        g->off[v + 1] = w;
      }
    }
    if (pass == 0) g = graph_alloc(n, w);
  }
  free(x); free(y); free(cs); free(pts);
  return g;
}

/* generate.cpp:128-136 */
orc_graph *orc_petersen(void) {
  int32_t eu[15], ev[15];
  int k = 0;
  for (int32_t v = 0; v < 5; ++v) {
    eu[k] = v; ev[k] = (v + 1) % 5; ++k;
    eu[k] = 5 + v; ev[k] = 5 + (v + 2) % 5; ++k;
    eu[k] = v; ev[k] = 5 + v; ++k;
  }
  return orc_graph_from_edges(10, 15, eu, ev);
}

uint64_t orc_checksum_bytes(const void *data, int64_t len) {
  /* FNV-1a over 8-byte words (tail bytes folded individually) */
  const unsigned char *b = (const unsigned char *)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  int64_t i = 0;
  for (; i + 8 <= len; i += 8) {
    uint64_t w;
    memcpy(&w, b + i, 8);
    h ^= w;
    h *= 0x100000001b3ULL;
  }
  for (; i < len; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ------------------------------------------------------------ validation */

/* validate.cpp:45-56 check_independence: the first v (ascending) in the set
 * with a neighbour u in the set gives the witness (min, max).  Returns 1
 * independent, 0 not (witness in *wu, *wv), -1 an id outside [0, n). */
int orc_check_independence(int32_t n, const int64_t *off, const int32_t *nbr, const int32_t *set,
                           int64_t cnt, int32_t *wu, int32_t *wv) {
  uint8_t *in = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
  for (int64_t i = 0; i < cnt; ++i) {
    if (set[i] < 0 || set[i] >= n) {
      free(in);
      return -1;
    }
    in[set[i]] = 1;
  }
  for (int32_t v = 0; v < n; ++v) {
    if (!in[v]) continue;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      const int32_t u = nbr[e];
      if (in[u]) {
        *wu = u < v ? u : v;
        *wv = u < v ? v : u;
        free(in);
        return 0;
      }
    }
  }
  free(in);
  return 1;
}

/* validate.cpp:58-75 check_maximality (independent input): the first v not
 * in the set without a neighbour in the set is addable.  Returns 1 maximal,
 * 0 not (*addable), -1 bad id, -2 the set is not independent. */
int orc_check_maximality(int32_t n, const int64_t *off, const int32_t *nbr, const int32_t *set,
                         int64_t cnt, int32_t *addable) {
  int32_t a, b;
  const int ind = orc_check_independence(n, off, nbr, set, cnt, &a, &b);
  if (ind < 0) return -1;
  if (ind == 0) return -2;
  uint8_t *in = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
  for (int64_t i = 0; i < cnt; ++i) in[set[i]] = 1;
  for (int32_t v = 0; v < n; ++v) {
    if (in[v]) continue;
    int blocked = 0;
    for (int64_t e = off[v]; e < off[v + 1] && !blocked; ++e) blocked = in[nbr[e]];
    if (!blocked) {
      *addable = v;
      free(in);
      return 0;
    }
  }
  free(in);
  return 1;
}
