/*
 * tcmis_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference TC-MIS path (/root/reference/proj).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  Parity of the restatement itself is pinned against the
 * reference library compiled from its own sources (oracle/_ref, see
 * oracle/Makefile) and against the golden vectors in SURVEY.md 8(c) and
 * tests/golden/.
 */
#ifndef TCMIS_ORACLE_H
#define TCMIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* A CSR graph owned by the oracle (graph.hpp:18-39 layout). */
typedef struct orc_graph {
  int32_t n;
  int64_t nnz; /* = 2m directed entries */
  int64_t *off;
  int32_t *nbr;
} orc_graph;

typedef struct orc_round {
  int64_t sel, rem, alive, tiles_eval, tiles_skip;
  /* trajectory terms for the algorithmic-byte model */
  int64_t alive_start, nnz_alive, noncand, nnz_noncand, nnz_cand;
} orc_round;

/* priorities.cpp:15-31 */
uint64_t orc_mix64(uint64_t x);
uint64_t orc_vertex_hash(uint64_t v, uint64_t seed);
double orc_hash_to_unit(uint64_t h);
uint64_t orc_combine_seed(uint64_t seed, uint64_t round);
/* priorities.cpp:33-67; return 0 ok, 1 invalid argument */
int orc_h1_random(int32_t n, uint64_t seed, uint32_t *p);
uint32_t orc_h2_priority_value(double avg, int32_t deg, double eps, int scale_bits);
int orc_h2_degree_aware(int32_t n, const int64_t *off, uint64_t seed,
                        int scale_bits, uint32_t *p);

/* Luby rounds with fixed priorities (engine.cpp:86-160, 231-295) or redrawn
 * priorities (fresh=1, engine.cpp:317-348).  rowtiles (may be NULL) gives the
 * per-block-row tile count of the T-tiling for the tile counters.  state_out
 * receives the final VertexState per vertex (1 = InMIS, 2 = Removed).
 * Returns the number of rounds, or -1 when max_rounds is exceeded. */
int orc_luby_rounds(int32_t n, const int64_t *off, const int32_t *nbr,
                    const uint32_t *p, int fresh, uint64_t seed,
                    const int64_t *tile_col_count, int T, uint8_t *state_out,
                    orc_round *rounds, int max_rounds);

/* engine.cpp:162-229 run_h3_resolution over the alive set given by states
 * (0 = alive); writes c[v] in {0,1}.  Returns the number of inner rounds. */
int orc_h3_resolution(int32_t n, const int64_t *off, const int32_t *nbr,
                      const uint32_t *p, const uint8_t *states, uint8_t *c);

/* tests/support/oracles.cpp:76-92 -- lexicographically-first MIS under the
 * (p, id) key order.  Writes member flags; returns |MIS|. */
int64_t orc_greedy_mis(int32_t n, const int64_t *off, const int32_t *nbr,
                       const uint32_t *p, uint8_t *member);

/* engine.cpp:86-103 compute_max_np, engine.cpp:121-160 phase3_update
 * (returns 0 ok, 3 logic error), spmv.cpp:61-73 csr neighbor count. */
void orc_compute_max_np(int32_t n, const int64_t *off, const int32_t *nbr,
                        const uint32_t *p, const uint8_t *states, uint64_t *out);
int orc_phase3_update(int32_t n, uint8_t *states, const uint8_t *c,
                      const int32_t *nc, int64_t *sel, int64_t *rem);
void orc_csr_neighbor_count(int32_t n, const int64_t *off, const int32_t *nbr,
                            const uint8_t *c, int32_t *nc);

/* tiling.cpp:44-84 tile_graph.  Two calls: with row_bits == NULL only the
 * tile count is returned; otherwise tile_row/tile_col/row_bits (T words per
 * tile) and block_row_offsets (nb+1) are filled.  Returns tile count, or -1
 * for an invalid tile_dim. */
int64_t orc_tile_graph(int32_t n, const int64_t *off, const int32_t *nbr,
                       int T, int32_t *tile_row, int32_t *tile_col,
                       uint64_t *row_bits, int64_t *block_row_offsets);
/* Per-block-row distinct block-column count (== tiles per block row). */
int64_t orc_tile_row_counts(int32_t n, const int64_t *off, const int32_t *nbr,
                            int T, int64_t *rowtiles);
/* tiling.cpp:86-101 pack_vector segment bits (nseg words) */
void orc_pack_segments(int32_t n, const uint8_t *values, int T, uint64_t *seg);
/* spmv.cpp:18-59 tiled_spmv with skip; returns 0 ok */
int orc_tiled_spmv(int32_t n, int T, int64_t tile_count, const int32_t *tile_col,
                   const uint64_t *row_bits, const int64_t *block_row_offsets,
                   const uint64_t *seg, int32_t *nc, int64_t *evaluated,
                   int64_t *skipped);

/* Generators.  graph.cpp:14-41 normalisation; generate.cpp:30-98 G(n,p) and
 * R-MAT; grid and RGG are new definitions. */
orc_graph *orc_graph_from_edges(int32_t n, int64_t m, const int32_t *eu,
                                const int32_t *ev);
orc_graph *orc_gnp(int32_t n, double p, uint64_t seed);
orc_graph *orc_gnp_avg_degree(int32_t n, double avg_degree, uint64_t seed);
orc_graph *orc_rmat(int scale, int edge_factor, uint64_t seed);
orc_graph *orc_grid(int32_t side);
orc_graph *orc_rgg(int32_t n, double avg_degree, uint64_t seed);
uint64_t orc_rgg_radius(int32_t n, double avg_degree);
orc_graph *orc_petersen(void);
void orc_graph_free(orc_graph *g);

/* FNV-style checksum used by the golden fixtures. */
uint64_t orc_checksum_bytes(const void *data, int64_t len);

#ifdef __cplusplus
}
#endif
int orc_check_independence(int32_t n, const int64_t *off, const int32_t *nbr, const int32_t *set,
                           int64_t cnt, int32_t *wu, int32_t *wv);
int orc_check_maximality(int32_t n, const int64_t *off, const int32_t *nbr, const int32_t *set,
                         int64_t cnt, int32_t *addable);

#endif
