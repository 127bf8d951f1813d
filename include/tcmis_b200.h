/*
 * tcmis_b200.h -- C-ABI of the B200-native TC-MIS engine (sm_100a).
 *
 * This is the drop-in boundary for the reference's MIS call.  Every entry
 * point names the reference interface it replaces (paths relative to
 * /root/reference/proj).  Signatures carry only plain pointers, sizes and PODs;
 * errors are status codes plus tcmis_last_error(), which the C++ layer
 * (include/tcmis/*.hpp, libtcmis.so) maps back onto the reference's exception
 * types (SURVEY 8(b) "Errors").
 *
 * Threading: a context owns one device and one CUDA stream; calls on one
 * context are not re-entrant ("one coordinator per engine call").
 * There is no CPU fallback: every compute entry point launches sm_100a kernels
 * and fails with TCMIS_E_CUDA when no device is usable.
 */
#ifndef TCMIS_B200_H
#define TCMIS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCMIS_ABI_VERSION 1

/* Status codes; C++ mapping in brackets. */
typedef enum tcmis_status {
  TCMIS_OK = 0,
  TCMIS_E_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  TCMIS_E_RUNTIME = 2,          /* std::runtime_error (iteration cap, engine.cpp:248-249) */
  TCMIS_E_LOGIC = 3,            /* std::logic_error (engine.cpp:152-153) */
  TCMIS_E_CUDA = 4,             /* std::runtime_error: CUDA / no device */
  TCMIS_E_OUT_OF_RANGE = 5      /* std::out_of_range (graph.cpp:23-24) */
} tcmis_status;

/* engine.hpp:19 `enum class Heuristic { H1, H2, H3, LubyFresh, LubyPerm }` */
typedef enum tcmis_heuristic {
  TCMIS_H1 = 0,
  TCMIS_H2 = 1,
  TCMIS_H3 = 2,
  TCMIS_LUBY_FRESH = 3,
  TCMIS_LUBY_PERM = 4
} tcmis_heuristic;

/* engine.hpp:17 `enum class VertexState : uint8_t { Alive, InMIS, Removed }` */
enum { TCMIS_ALIVE = 0, TCMIS_IN_MIS = 1, TCMIS_REMOVED = 2 };

/* Neighbour-exclusion (Phase 2) kernel variants; see DESIGN.md "K4". */
typedef enum tcmis_exclusion {
  TCMIS_EXCL_AUTO = 0,     /* the variant ncu says wins (currently PUSH)      */
  TCMIS_EXCL_PUSH = 1,     /* candidates scatter Removed to their neighbours  */
  TCMIS_EXCL_CSR_PULL = 2, /* alive non-candidates look for a candidate nbr   */
  TCMIS_EXCL_TILE_BITS = 3,/* T x T bit tiles AND candidate segments (CUDA cores) */
  TCMIS_EXCL_TILE_MMA = 4  /* T=16 tiles x candidate vector on tensor cores (mma.sync s8) */
} tcmis_exclusion;

/* engine.hpp:24-34 IterationStats (timers are device-event times). */
typedef struct tcmis_iter_stats {
  int32_t iteration;
  int32_t reserved;
  int64_t candidates_selected;
  int64_t vertices_removed;
  int64_t alive_remaining;
  int64_t tiles_evaluated;
  int64_t tiles_skipped;
  double phase1_ms;
  double phase2_ms;
  double phase3_ms;
} tcmis_iter_stats;

/* engine.hpp:59-64 iteration_observer: called once per iteration, before the
 * state update, with host copies of the candidate flags and states. */
typedef void (*tcmis_observer_fn)(void *user, int32_t iteration, const uint8_t *candidates,
                                  const uint8_t *states, int32_t n);

/* engine.hpp:53-65 EngineConfig */
typedef struct tcmis_config {
  int32_t heuristic;  /* tcmis_heuristic, default TCMIS_H3 (engine.hpp:54) */
  int32_t tile_dim;   /* 1..64, default 16 */
  uint64_t seed;      /* default 1 */
  int32_t scale_bits; /* 8..30, default 20 (priorities.hpp:24-26) */
  int32_t workers;    /* accepted and ignored: the CUDA grid replaces parallel.cpp */
  int32_t exclusion;  /* tcmis_exclusion */
  uint32_t flags;     /* TCMIS_F_* */
  tcmis_observer_fn observer;
  void *observer_user;
} tcmis_config;

#define TCMIS_F_TIMING 0x1u     /* record per-phase device times in the stats */
#define TCMIS_F_HOST_LOOP 0x2u  /* drive rounds from the host (no CUDA-graph while loop) */
/* tcmis_solve_partitioned: mis_out / state_out cover this rank's rows only
 * (its share of a distributed result) instead of all n vertices */
#define TCMIS_F_OWN_RANGE 0x4u
/* Phase 1 as a tile x bit-vector product: the oriented adjacency A-up (u in
 * N(v) with key(u) > key(v)) in the compact T = 16 tile store times
 * the round's alive bitmap (csrc/tile_cand.cu), with the tile-form exclusion
 * (TCMIS_EXCL_TILE_MMA stays MMA, anything else becomes TILE_BITS).  A-up
 * depends on the priorities: it is built on first use per (heuristic, seed,
 * scale_bits) and cached on the graph (tcmis_graph_tile_cand_prepare builds
 * it ahead).  Not for luby-fresh (its keys change every round). */
#define TCMIS_F_TILE_CAND 0x8u
/* with TCMIS_F_TILE_CAND: the A-up tile x alive product on the tensor cores
 * (tcgen05.mma kind::i8, accumulator in TMEM; csrc/tile_umma.cuh) */
#define TCMIS_F_TILE_UMMA 0x10u
/* test hook: start the solve from a control block that disagrees with the
 * vertex states; the device's round invariant check must then fail the solve
 * with TCMIS_E_LOGIC (the reference's logic_error, engine.cpp:152-153) */
#define TCMIS_F_DEBUG_CORRUPT 0x100u

/* Fill *cfg with the reference defaults (EngineConfig{}). */
void tcmis_config_init(tcmis_config *cfg);

typedef struct tcmis_ctx tcmis_ctx;
typedef struct tcmis_graph tcmis_graph;

const char *tcmis_last_error(void);
int32_t tcmis_abi_version(void);

/* Context: device + stream + scratch.  Replaces parallel.cpp:12-62
 * (resolve_workers / parallel_for / parallel_chunks). */
int tcmis_ctx_create(int32_t device, tcmis_ctx **out);
void tcmis_ctx_destroy(tcmis_ctx *ctx);
/* The CUDA stream (cudaStream_t) every launch of this context goes to. */
void *tcmis_ctx_stream(tcmis_ctx *ctx);
int tcmis_ctx_synchronize(tcmis_ctx *ctx);
/* Kernels this context launched since creation (driver evidence counter). */
int64_t tcmis_ctx_launches(tcmis_ctx *ctx);

/* Per-kernel device times of the last solve run with TCMIS_F_TIMING (CUDA
 * events around every launch on the context stream).  Returns the number of
 * entries (copies at most cap). */
typedef struct tcmis_kernel_time {
  char name[32];
  int32_t round;
  float ms;
} tcmis_kernel_time;
int32_t tcmis_ctx_timeline(tcmis_ctx *ctx, tcmis_kernel_time *out, int32_t cap);

/* Device-resident CSR graph (graph.hpp:18-39 Graph: n, offsets[n+1] int64,
 * neighbors[2m] int32, normalised).  upload copies host arrays (H2D on the
 * context stream); wrap_device borrows device arrays the caller keeps alive. */
int tcmis_graph_upload(tcmis_ctx *ctx, int32_t n, const int64_t *offsets,
                       const int32_t *neighbors, tcmis_graph **out);
/* upload + tcmis_graph_tile(tile_dim) in one call, the tile count overlapping
 * the upload: neighbour ids go up in chunks of block rows while the light
 * block rows of the chunks already resident are counted on a side stream
 * (the drop-in path of run_mis / run_tc_mis(g, cfg), engine.cpp:297-299).
 * *tile_count (may be NULL) = TiledAdjacency::tile_count(). */
int tcmis_graph_upload_tiled(tcmis_ctx *ctx, int32_t n, const int64_t *offsets,
                             const int32_t *neighbors, int32_t tile_dim, tcmis_graph **out,
                             int64_t *tile_count);
int tcmis_graph_wrap_device(tcmis_ctx *ctx, int32_t n, int64_t nnz, const int64_t *d_offsets,
                            const int32_t *d_neighbors, tcmis_graph **out);
void tcmis_graph_destroy(tcmis_graph *g);
int32_t tcmis_graph_n(const tcmis_graph *g);
int64_t tcmis_graph_nnz(const tcmis_graph *g);
/* Device pointers of the CSR (for callers that launch around the engine). */
const int64_t *tcmis_graph_device_offsets(const tcmis_graph *g);
const int32_t *tcmis_graph_device_neighbors(const tcmis_graph *g);
/* Copy the CSR back to host buffers (n+1 / nnz entries). */
int tcmis_graph_download(tcmis_graph *g, int64_t *offsets, int32_t *neighbors);

/* K1 CSR->tile converter (tiling.cpp:44-84 tile_graph).  tcmis_graph_tile
 * derives, on the device, the T x T tiling the tile counters of run_tc_mis are
 * defined on (tiles per block row; spmv.cpp:37-46), and caches it on the
 * graph.  *tile_count receives TiledAdjacency::tile_count(). */
int tcmis_graph_tile(tcmis_graph *g, int32_t tile_dim, int64_t *tile_count);
/* Same, from a TiledAdjacency the caller already holds (the prebuilt-tiles
 * overload engine.hpp:111-112): block_row_offsets has n_block_rows+1 entries,
 * tile_col tile_count entries.  The tile counters of the solve are taken on
 * exactly this tile set (tiles per block column, spmv.cpp:37-46), whatever
 * tiling produced it; a column outside [0, n_block_rows) is rejected. */
int tcmis_graph_set_tiling(tcmis_graph *g, int32_t tile_dim, const int64_t *block_row_offsets,
                           int32_t n_block_rows, const int32_t *tile_col, int64_t tile_count);
/* Full tile materialisation in the reference layout (tile_row, tile_col,
 * T u64 row words per tile, block_row_offsets[nb+1]); host buffers sized from
 * tcmis_graph_tile()'s count. */
int tcmis_graph_export_tiles(tcmis_graph *g, int32_t tile_dim, int32_t *tile_row,
                             int32_t *tile_col, uint64_t *row_bits, int64_t *block_row_offsets);
/* An internal vertex order for the solve kernels (csrc/order.cu): the graph
 * keeps the caller's CSR and ids and adds a relabeled copy the round kernels
 * run on, for locality of their neighbour gathers.  Results, statistics and
 * every other entry point stay in the caller's ids and are bit-identical to
 * the unordered solve (keys, hash priorities and tile counters are taken on
 * the caller's ids).  TCMIS_ORDER_NONE drops the copy; SPATIAL needs a graph
 * from tcmis_gen_rgg; GIVEN takes order[n] (host), order[i] = the caller's id
 * of solve id i, a permutation of [0, n).  Not for row partitions.  Solves
 * with an iteration observer or a tile exclusion form use the caller's CSR. */
enum { TCMIS_ORDER_NONE = 0, TCMIS_ORDER_DEGREE = 1, TCMIS_ORDER_SPATIAL = 2,
       TCMIS_ORDER_GIVEN = 3 };
int tcmis_graph_reorder(tcmis_graph *g, int32_t mode, const int32_t *order);
/* A new graph whose ids ARE the order's solve ids (the relabeled CSR as an
 * ordinary graph, e.g. an RGG with spatially ordered ids). */
int tcmis_graph_permuted(tcmis_graph *g, tcmis_graph **out);

/* The compact device tile store the tile-form exclusion kernels read
 * (tile_dim 8 or 16; same tile set and order as tile_graph, tiling.cpp:44-84):
 * builds it if needed and reports its tile count; with non-null buffers also
 * copies block_row_offsets[nb+1], tile_col[tiles] and the payload (T rows of
 * T bits per tile: u16 rows for T = 16, u8 rows for T = 8) to the host. */
int tcmis_graph_tile_store(tcmis_graph *g, int32_t tile_dim, int64_t *tile_count,
                           int64_t *block_row_offsets, int32_t *tile_col, void *payload);

/* Build (or find cached) the A-up tile store TCMIS_F_TILE_CAND solves with
 * cfg's priorities use; *build_ms = device time of the orientation + tiling
 * (0 when cached), *tiles = its tile count. */
int tcmis_graph_tile_cand_prepare(tcmis_graph *g, const tcmis_config *cfg, double *build_ms,
                                  int64_t *tiles);

/* validate.cpp:45-75 check_independence + check_maximality on the device, in
 * one pass, with the reference's witnesses: *independent (else the violating
 * edge (u, v), u < v, of the smallest offending vertex) and *maximal (else
 * the smallest addable vertex; meaningful only for an independent set).  An id
 * outside [0, n) -> TCMIS_E_INVALID_ARGUMENT (validate.cpp:12-22). */
int tcmis_validate(tcmis_graph *g, const int32_t *set, int64_t count, int32_t *independent,
                   int32_t *violating_u, int32_t *violating_v, int32_t *maximal,
                   int32_t *addable_vertex);

/* priorities.cpp:33-67 (h1_random / h2_degree_aware) on the device; p_out is
 * a host buffer of n entries. */
int tcmis_priorities(tcmis_graph *g, int32_t heuristic, uint64_t seed, int32_t scale_bits,
                     uint32_t *p_out);

/* The MIS call: engine.cpp:354-365 run_mis / engine.cpp:231-299 run_tc_mis.
 * Heuristics H1/H2/H3 and both Luby modes.  Outputs (each may be NULL):
 *   state_out[n]  final VertexState per vertex (host)
 *   mis_out[n]    ascending MIS vertex ids (host), *mis_count = |MIS|
 *   stats[max_stats] per-iteration stats, *n_iterations = iterations.size()
 * For H1/H2/H3 tcmis_graph_tile() (or set_tiling) for cfg->tile_dim must have
 * run; otherwise the tiling is derived on the fly. */
int tcmis_solve(tcmis_graph *g, const tcmis_config *cfg, uint8_t *state_out, int32_t *mis_out,
                int64_t *mis_count, tcmis_iter_stats *stats, int32_t max_stats,
                int32_t *n_iterations);

/* Device-resident variant for benchmarking and multi-call pipelines: leaves
 * the results on the device.  *d_mis receives a device pointer (owned by the
 * graph, valid until the next solve) to the ascending MIS ids; *d_state the
 * device VertexState array.  Stats are copied to the host. */
int tcmis_solve_device(tcmis_graph *g, const tcmis_config *cfg, const int32_t **d_mis,
                       int64_t *mis_count, const uint8_t **d_state, tcmis_iter_stats *stats,
                       int32_t max_stats, int32_t *n_iterations);

/* Row-partitioned multi-GPU solve (host driver in
 * paper_2605_29604_b200/distributed.py).  Rank r uploads its rows [lo, hi)
 * with the full offsets (n+1, for global degrees) and the neighbour lists of
 * its rows (full_offsets[hi] - full_offsets[lo] ids).  Per round:
 *   tcmis_dist_select  -> own candidates as bitmap slice d_bits (bit v - lo)
 *   (host all-gathers the slices, rank r's at word r * maxw)
 *   tcmis_dist_apply(what = 0) -> remote candidates marked
 *   tcmis_dist_update  -> own removals as bitmap slice; d_counts[5] (DEVICE
 *                         memory) = this rank's (selected, removed, alive,
 *                         tiles_eval, tiles_skip)
 *   (host all-gathers, all-reduces the counts on the device)
 *   tcmis_dist_apply(what = 1) -> remote removals applied
 * until the all-reduced alive count is 0; tcmis_dist_state copies the own
 * range's VertexStates.  rank_lo has world + 1 entries (rank_lo[world] = n).
 * Every call is stream-ordered on the context stream without a host sync, so
 * NCCL collectives enqueued on that stream (tcmis_ctx_stream) interleave. */
int tcmis_graph_upload_partition(tcmis_ctx *ctx, int32_t n, int32_t lo, int32_t hi,
                                 const int64_t *full_offsets, const int32_t *row_neighbors,
                                 tcmis_graph **out);
/* The same partition cut from a device-resident full graph (device to device). */
int tcmis_graph_partition(tcmis_graph *full, int32_t lo, int32_t hi, tcmis_graph **out);
int tcmis_dist_begin(tcmis_graph *g, const tcmis_config *cfg);
int tcmis_dist_select(tcmis_graph *g, uint32_t *d_bits, int32_t words);
int tcmis_dist_apply(tcmis_graph *g, const uint32_t *d_gathered, const int32_t *rank_lo,
                     int32_t world, int32_t maxw, int32_t me, int32_t what);
int tcmis_dist_update(tcmis_graph *g, uint32_t *d_bits, int32_t words, int64_t *d_counts);
int tcmis_dist_state(tcmis_graph *g, uint8_t *own_state);
/* h3 on a partition: after the rounds, this rank's share of the collapsed
 * iteration's tiles_evaluated and its tile total (sum over ranks on the host). */
int tcmis_dist_h3_tiles(tcmis_graph *g, int64_t *tiles_evaluated, int64_t *tile_total);

/* The native partitioned solve (csrc/partitioned.cu): the whole
 * solve of one rank in one call, every round driven from C++ with the
 * exchange below -- bitmap slices in the first rounds, id lists once the
 * all-reduced alive count bounds a round's decisions below a slice -- and, for
 * a capturable exchange (NCCL), each round one CUDA graph launch with the host
 * one round ahead of the counters it reads.  The reference has no multi-GPU
 * path; this partitions its run_tc_mis loop (engine.cpp:247-291) so that the
 * MIS, the iteration count and every per-iteration statistic equal the
 * single-GPU solve for any world size.  `part` holds this rank's rows
 * (tcmis_graph_upload_partition / tcmis_graph_partition); rank_lo[world + 1]
 * as for tcmis_dist_apply.  Outputs (each may be NULL but n_iterations):
 * state_out[n] the final VertexState of ALL n vertices, mis_out[n] the
 * ascending ids of the whole MIS (every rank holds the replicated state at
 * the end; with TCMIS_F_OWN_RANGE both cover this rank's rows only), stats as tcmis_solve (counters summed over the ranks; phase
 * times are this rank's).  Every rank must call it with the same arguments
 * (collectives); a rank's error leaves its peers blocked in the exchange. */
typedef struct tcmis_exchange tcmis_exchange;
/* ncclGetUniqueId (128 bytes) for rank 0 to broadcast; NCCL (libnccl.so.2) is
 * bound at run time -- the copy the process already loaded first, else the
 * loader's (TCMIS_NCCL_LIB overrides) -- so the library has no link-time
 * NCCL dependency. */
int tcmis_nccl_unique_id(uint8_t id[128]);
/* a communicator of its own (ncclCommInitRank on the context's device) */
int tcmis_exchange_nccl(tcmis_ctx *ctx, int32_t world, int32_t rank, const uint8_t id[128],
                        tcmis_exchange **out);
/* an ncclComm_t the caller owns and keeps alive (created by the same libnccl) */
int tcmis_exchange_nccl_comm(void *nccl_comm, tcmis_exchange **out);
/* world ranks of ONE process, one host thread each (one context per rank, on
 * any devices): all-gathers are copies through UVA / peer access.  out[world]. */
int tcmis_exchange_local_group(int32_t world, tcmis_exchange **out);
void tcmis_exchange_destroy(tcmis_exchange *x);
/* in-process group: release the peers of a rank that failed before (or
 * outside) tcmis_solve_partitioned from the exchange; a failing solve does
 * this itself.  No-op for NCCL. */
void tcmis_exchange_abort(tcmis_exchange *x);
int32_t tcmis_exchange_world(const tcmis_exchange *x);
int32_t tcmis_exchange_rank(const tcmis_exchange *x);
int tcmis_solve_partitioned(tcmis_graph *part, tcmis_exchange *x, const int32_t *rank_lo,
                            int32_t world, const tcmis_config *cfg, uint8_t *state_out,
                            int32_t *mis_out, int64_t *mis_count, tcmis_iter_stats *stats,
                            int32_t max_stats, int32_t *n_iterations);

/* Host-side profile of the last tcmis_solve_partitioned on `part`: out[0]
 * rounds, out[1] total host time spent enqueueing rounds (graph launches or
 * direct launches + exchange calls), out[2] total time the host waited for
 * round counters, out[3] wall time of the round loop (all us), out[4] rounds
 * enqueued with id lists, out[5] rounds run by the single-device tail (the
 * alive subgraph gathered on every rank once it fits k_tail). */
int tcmis_partitioned_profile(const tcmis_graph *part, double out[6]);

/* h1_random (priorities.cpp:33-41) without a graph: n priorities on the
 * device of the context, copied to p_out[n]. */
int tcmis_h1_random(tcmis_ctx *ctx, int32_t n, uint64_t seed, uint32_t *p_out);

/* run_h3_resolution (engine.cpp:162-229): the greedy MIS of the alive subset
 * of `states` under the priorities p, computed by the engine's rounds on the
 * device; c_out[v] = 1 for the selected vertices. */
int tcmis_h3_resolution(tcmis_graph *g, const uint32_t *p, const uint8_t *states,
                        uint8_t *c_out);

/* tiled_spmv (spmv.cpp:18-59) over a TiledAdjacency in the reference layout
 * (host arrays, uploaded per call): nc = A * c with tile skipping, plus the
 * tiles_evaluated / tiles_skipped counters.  exclusion selects the kernel:
 * TCMIS_EXCL_TILE_BITS (popcount of row & segment on CUDA cores) or
 * TCMIS_EXCL_TILE_MMA (T = 16 only: tiles x segment on the tensor cores via
 * mma.sync m16n8k16 s8). */
int tcmis_tiled_spmv_tiles(tcmis_ctx *ctx, int32_t n, int32_t tile_dim, int64_t tile_count,
                           const int32_t *tile_col, const uint64_t *row_bits,
                           const int64_t *block_row_offsets, const uint64_t *segment_bits,
                           int32_t exclusion, int32_t *nc_out, int64_t *tiles_evaluated,
                           int64_t *tiles_skipped);

/* Phase-level helpers on the device (engine.hpp:71-106, spmv.hpp:15-42);
 * host buffers in, host buffers out, for parity tests of single phases. */
int tcmis_compute_max_np(tcmis_graph *g, const uint32_t *p, const uint8_t *states,
                         uint64_t *max_np_out);
int tcmis_neighbor_count(tcmis_graph *g, const uint8_t *candidates, int32_t *nc_out);
int tcmis_tiled_spmv(tcmis_graph *g, int32_t tile_dim, const uint8_t *candidates,
                     int32_t exclusion, int32_t *nc_out, int64_t *tiles_evaluated,
                     int64_t *tiles_skipped);

/* Synthetic graph generators on the device (generate.cpp:30-98 and the new
 * grid / RGG definitions of DESIGN.md); the result is a device-resident
 * normalised graph (graph.cpp:14-41 semantics). */
int tcmis_gen_rmat(tcmis_ctx *ctx, int32_t scale, int32_t edge_factor, uint64_t seed,
                   tcmis_graph **out);
int tcmis_gen_grid(tcmis_ctx *ctx, int32_t side, tcmis_graph **out);
/* graph.cpp:14-41 graph_from_edges on the device: the m edges
 * (u[i], v[i]) symmetrised, self-loops dropped, duplicates merged, rows
 * sorted; an endpoint outside [0, n) -> TCMIS_E_OUT_OF_RANGE. */
int tcmis_graph_from_edges(tcmis_ctx *ctx, int32_t n, int64_t m, const int32_t *u,
                           const int32_t *v, tcmis_graph **out);
int tcmis_gen_rgg(tcmis_ctx *ctx, int32_t n, uint64_t radius, uint64_t seed,
                  tcmis_graph **out);
/* gnp_graph_avg_degree (generate.cpp:30-66) on the device: the serial
 * SplitMix64 stream in counter form, the pair-index increments prefix-summed
 * (replaces the reference's serial generator; bit-identical graph). */
int tcmis_gen_gnp(tcmis_ctx *ctx, int32_t n, double avg_degree, uint64_t seed,
                  tcmis_graph **out);
/* The same G(n,p) on the host (the serial definition), returned as malloc'ed
 * CSR arrays the caller frees with tcmis_free(). */
int tcmis_gen_gnp_host(int32_t n, double avg_degree, uint64_t seed, int64_t **offsets,
                       int32_t **neighbors, int64_t *nnz);
void tcmis_free(void *p);
/* Radius of the RGG definition: floor(sqrt(avg/(pi n)) * 2^32). */
uint64_t tcmis_rgg_radius(int32_t n, double avg_degree);

#ifdef __cplusplus
}
#endif
#endif /* TCMIS_B200_H */
