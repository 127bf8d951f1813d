// capi.cu -- the extern "C" boundary (include/tcmis_b200.h).
//
// Every entry point validates like the reference (exception type -> status
// code), owns no hidden global state beyond the thread-local error string, and
// launches only sm_100a kernels from this library.  There is deliberately no
// CPU fallback: without a usable CUDA device every compute call fails with
// TCMIS_E_CUDA.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <string>
#include <vector>

#include "internal.cuh"

#define TCMIS_API extern "C" __attribute__((visibility("default")))

namespace tcmis_b200 {

static thread_local std::string g_last_error;
thread_local cudaStream_t t_alloc_stream = nullptr;

int set_error(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char *what) {
  g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return TCMIS_E_CUDA;
}

int solve_impl(tcmis_graph *g, const tcmis_config *cfg, tcmis_iter_stats *stats,
               int32_t max_stats, int32_t *n_iter, int64_t *mis_count_out);
int priorities_impl(tcmis_graph *g, int heuristic, uint64_t seed, int scale_bits,
                    uint32_t *p_out);
int max_np_impl(tcmis_graph *g, const uint32_t *p, const uint8_t *states, uint64_t *out);
int neighbor_count_impl(tcmis_graph *g, const uint8_t *c, int32_t *nc, int T, int64_t *ev,
                        int64_t *sk);
int gen_rmat(tcmis_ctx *ctx, int32_t scale, int32_t ef, uint64_t seed, tcmis_graph **out);
int gen_grid(tcmis_ctx *ctx, int32_t side, tcmis_graph **out);
int gen_from_edges(tcmis_ctx *ctx, int32_t n, int64_t m, const int32_t *u, const int32_t *v,
                   tcmis_graph **out);
int gen_rgg(tcmis_ctx *ctx, int32_t n, uint64_t R, uint64_t seed, tcmis_graph **out);
int gen_gnp(tcmis_ctx *ctx, int32_t n, double avg_degree, uint64_t seed, tcmis_graph **out);
int gen_gnp_host(int32_t n, double avg_degree, uint64_t seed, int64_t **offsets,
                 int32_t **neighbors, int64_t *nnz_out);
int h1_impl(tcmis_ctx *ctx, int32_t n, uint64_t seed, uint32_t *p_out);
int partition_device(tcmis_graph *full, int32_t lo, int32_t hi, tcmis_graph **out);
int validate_impl(tcmis_graph *g, const int32_t *set, int64_t cnt, int32_t *independent,
                  int32_t *wu, int32_t *wv, int32_t *maximal, int32_t *addable);
int upload_partition(tcmis_ctx *ctx, int32_t n, int32_t lo, int32_t hi, const int64_t *full,
                     const int32_t *rows, tcmis_graph **out);
int dist_begin(tcmis_graph *g, const tcmis_config *cfg);
int dist_select(tcmis_graph *g, uint32_t *d_bits, int32_t words);
int dist_apply(tcmis_graph *g, const uint32_t *d_gathered, const int32_t *h_rank_lo,
               int32_t world, int32_t maxw, int32_t me, int32_t what);
int dist_update(tcmis_graph *g, uint32_t *d_bits, int32_t words, int64_t *counts);
int dist_state_out(tcmis_graph *g, uint8_t *own_state);
int dist_h3_tiles(tcmis_graph *g, int64_t *ev, int64_t *total);
int h3_resolution_impl(tcmis_graph *g, const uint32_t *p, const uint8_t *states, uint8_t *c);
int tiled_spmv_tiles_impl(tcmis_ctx *ctx, int32_t n, int32_t T, int64_t tiles,
                          const int32_t *tile_col, const uint64_t *row_bits, const int64_t *bro,
                          const uint64_t *seg, int32_t exclusion, int32_t *nc, int64_t *ev,
                          int64_t *sk);

int wrap_owned(tcmis_ctx *ctx, int32_t n, int64_t nnz, int64_t *d_off, int32_t *d_nbr,
               tcmis_graph **out) {
  auto *g = new tcmis_graph();
  g->ctx = ctx;
  g->n = n;
  g->nnz = nnz;
  g->d_off = d_off;
  g->d_nbr = d_nbr;
  g->owns = true;
  *out = g;
  return 0;
}

}  // namespace tcmis_b200

using namespace tcmis_b200;

// every entry point: the context's device, and its stream for the
// stream-ordered allocations of this call (internal.cuh dev_alloc)
#define ENTER(c)                                   \
  do {                                             \
    TCMIS_CUDA(cudaSetDevice((c)->device));        \
    t_alloc_stream = (c)->stream;                  \
  } while (0)

#define NEED(cond, msg) \
  if (!(cond)) return set_error(TCMIS_E_INVALID_ARGUMENT, msg)

TCMIS_API const char *tcmis_last_error(void) { return g_last_error.c_str(); }
TCMIS_API int32_t tcmis_abi_version(void) { return TCMIS_ABI_VERSION; }

TCMIS_API void tcmis_config_init(tcmis_config *c) {
  std::memset(c, 0, sizeof(*c));
  c->heuristic = TCMIS_H3;  // engine.hpp:54
  c->tile_dim = 16;
  c->seed = 1;
  c->scale_bits = 20;
  c->workers = 0;
  c->exclusion = TCMIS_EXCL_AUTO;
}

TCMIS_API int tcmis_ctx_create(int32_t device, tcmis_ctx **out) {
  NEED(out, "null output handle");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_error(TCMIS_E_CUDA, "no CUDA device available (the B200 engine has no CPU path)");
  NEED(device >= 0 && device < count, "device index out of range");
  TCMIS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  TCMIS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return set_error(TCMIS_E_CUDA, std::string("device ") + prop.name +
                                       " is not sm_100-class; this build targets sm_100a only");
  auto *ctx = new tcmis_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return cuda_error(e, "cudaStreamCreate");
  }
  for (auto &ev : ctx->ev) cudaEventCreate(&ev);
  // keep freed blocks in the device pool (dev_alloc / dev_free): repeated
  // upload -> solve -> destroy cycles then never return to the driver
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = ctx;
  return 0;
}

TCMIS_API void tcmis_ctx_destroy(tcmis_ctx *ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  t_alloc_stream = ctx->stream;
  free_staging(ctx);
  free_workspace(ctx->spare);
  cudaStreamSynchronize(ctx->stream);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  for (auto &ev : ctx->ev) cudaEventDestroy(ev);
  for (auto &ev : ctx->event_pool) cudaEventDestroy(ev);
  cudaStreamDestroy(ctx->stream);
  if (ctx->side) {
    cudaStreamDestroy(ctx->side);
    for (cudaEvent_t e : ctx->side_ev) cudaEventDestroy(e);
  }
  delete ctx;
}

TCMIS_API void *tcmis_ctx_stream(tcmis_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }
TCMIS_API int64_t tcmis_ctx_launches(tcmis_ctx *ctx) { return ctx ? ctx->launches : 0; }
TCMIS_API int32_t tcmis_ctx_timeline(tcmis_ctx *ctx, tcmis_kernel_time *out, int32_t cap) {
  if (!ctx) return 0;
  const int32_t n = (int32_t)ctx->timeline.size();
  for (int32_t i = 0; i < n && i < cap && out; ++i) out[i] = ctx->timeline[i];
  return n;
}
TCMIS_API int tcmis_ctx_synchronize(tcmis_ctx *ctx) {
  NEED(ctx, "null context");
  TCMIS_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

TCMIS_API int tcmis_graph_upload_tiled(tcmis_ctx *ctx, int32_t n, const int64_t *offsets,
                                       const int32_t *neighbors, int32_t tile_dim,
                                       tcmis_graph **out, int64_t *tile_count) {
  TCMIS_RANGE("tcmis_graph_upload_tiled");
  NEED(ctx && out, "null handle");
  NEED(n >= 0, "vertex count must be non-negative");
  NEED(n == 0 || offsets, "null offsets");
  *out = nullptr;
  const int64_t nnz = offsets ? offsets[n] : 0;
  NEED(nnz >= 0, "negative edge count");
  NEED(nnz == 0 || neighbors, "null neighbors");
  ENTER(ctx);
  tcmis_graph *g = nullptr;
  if (int rc = upload_tiled(ctx, n, offsets, neighbors, tile_dim, &g)) {
    if (g) tcmis_graph_destroy(g);
    return rc;
  }
  *out = g;
  if (tile_count) *tile_count = g->tile_total;
  return 0;
}

TCMIS_API int tcmis_graph_upload(tcmis_ctx *ctx, int32_t n, const int64_t *offsets,
                                 const int32_t *neighbors, tcmis_graph **out) {
  TCMIS_RANGE("tcmis_graph_upload");
  NEED(ctx && out, "null handle");
  NEED(n >= 0, "vertex count must be non-negative");
  NEED(n == 0 || offsets, "null offsets");
  *out = nullptr;
  const int64_t nnz = offsets ? offsets[n] : 0;
  NEED(nnz >= 0, "negative edge count");
  NEED(nnz == 0 || neighbors, "null neighbors");
  ENTER(ctx);
  int64_t *d_off = nullptr;
  int32_t *d_nbr = nullptr;
  if (int rc = dev_alloc(&d_off, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_nbr, (size_t)nnz)) {
    dev_free(d_off);
    return rc;
  }
  int rc = 0;
  if (offsets) rc = h2d(ctx, d_off, offsets, 8ull * (n + 1), ctx->stream);
  else if (cudaMemsetAsync(d_off, 0, 8, ctx->stream) != cudaSuccess)
    rc = cuda_error(cudaGetLastError(), "graph upload");
  if (!rc && nnz) rc = h2d(ctx, d_nbr, neighbors, 4ull * nnz, ctx->stream);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (!rc && e != cudaSuccess) rc = cuda_error(e, "graph upload");
  if (rc) {
    dev_free(d_off);
    dev_free(d_nbr);
    return rc;
  }
  return wrap_owned(ctx, n, nnz, d_off, d_nbr, out);
}

TCMIS_API int tcmis_graph_wrap_device(tcmis_ctx *ctx, int32_t n, int64_t nnz,
                                      const int64_t *d_offsets, const int32_t *d_neighbors,
                                      tcmis_graph **out) {
  NEED(ctx && out && d_offsets, "null handle");
  NEED(n >= 0 && nnz >= 0, "negative size");
  auto *g = new tcmis_graph();
  g->ctx = ctx;
  g->n = n;
  g->nnz = nnz;
  g->d_off = const_cast<int64_t *>(d_offsets);
  g->d_nbr = const_cast<int32_t *>(d_neighbors);
  g->owns = false;
  *out = g;
  return 0;
}

TCMIS_API void tcmis_graph_destroy(tcmis_graph *g) {
  if (!g) return;
  cudaSetDevice(g->ctx->device);
  t_alloc_stream = g->ctx->stream;  // frees are stream-ordered behind its work
  if (g->owns) {
    dev_free(g->d_off);
    dev_free(g->d_nbr);
  }
  dev_free(g->d_rowtiles);
  dev_free(g->d_nz);
  dev_free(g->d_off_full);
  free_dist(g);
  free_partitioned(g);
  free_order(g);
  free_up_store(g);
  dev_free(g->d_spatial);
  free_tile_store(g);
  Workspace &sp = g->ctx->spare;
  if (g->ws.ctrl && g->ws.n_cap >= sp.n_cap) {
    free_workspace(sp);
    sp = g->ws;
    g->ws = Workspace{};
  } else {
    free_workspace(g->ws);
  }
  delete g;
}

TCMIS_API int32_t tcmis_graph_n(const tcmis_graph *g) { return g ? g->n : 0; }
TCMIS_API int64_t tcmis_graph_nnz(const tcmis_graph *g) { return g ? g->nnz : 0; }
TCMIS_API const int64_t *tcmis_graph_device_offsets(const tcmis_graph *g) {
  return g ? g->d_off : nullptr;
}
TCMIS_API const int32_t *tcmis_graph_device_neighbors(const tcmis_graph *g) {
  return g ? g->d_nbr : nullptr;
}

TCMIS_API int tcmis_graph_download(tcmis_graph *g, int64_t *offsets, int32_t *neighbors) {
  NEED(g && offsets, "null handle");
  cudaStream_t st = g->ctx->stream;
  TCMIS_CUDA(cudaMemcpyAsync(offsets, g->d_off, 8ull * (g->n + 1), cudaMemcpyDeviceToHost, st));
  if (g->nnz && neighbors)
    TCMIS_CUDA(cudaMemcpyAsync(neighbors, g->d_nbr, 4ull * g->nnz, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

TCMIS_API int tcmis_graph_tile(tcmis_graph *g, int32_t tile_dim, int64_t *tile_count) {
  TCMIS_RANGE("tcmis_graph_tile");
  NEED(g, "null graph");
  ENTER(g->ctx);
  if (g->tile_T != tile_dim)
    if (int rc = build_tile_counts(g, tile_dim)) return rc;
  if (tile_count) *tile_count = g->tile_total;
  return 0;
}

TCMIS_API int tcmis_graph_set_tiling(tcmis_graph *g, int32_t T, const int64_t *bro,
                                     int32_t nb, const int32_t *tile_col, int64_t tile_count) {
  TCMIS_RANGE("tcmis_graph_set_tiling");
  NEED(g, "null graph");
  ENTER(g->ctx);
  if (T < 1 || T > 64)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tile_dim must be in [1, 64], got " + std::to_string(T));
  NEED(nb == (int32_t)(((int64_t)g->n + T - 1) / T), "tiled adjacency built for a different graph");
  NEED(nb == 0 || bro, "null block_row_offsets");
  NEED(tile_count == 0 || tile_col, "null tile_col");
  NEED(nb == 0 || bro[nb] - bro[0] == tile_count, "block_row_offsets disagree with tile_count");
  // The counters of tiled_spmv (spmv.cpp:37-46) are defined on THIS tiling:
  // a tile is evaluated iff the segment of its block column holds a
  // candidate, so the device keeps tiles per block column, counted from the
  // caller's tile_col (any tile set, not only tile_graph(g)'s symmetric one).
  std::vector<int32_t> ct((size_t)nb + 1, 0);
  for (int64_t t = 0; t < tile_count; ++t) {
    const int32_t c = tile_col[t];
    if (c < 0 || c >= nb) return set_error(TCMIS_E_INVALID_ARGUMENT, "tile column out of range");
    ++ct[(size_t)c];
  }
  dev_free(g->d_rowtiles);
  g->d_rowtiles = nullptr;
  g->tile_T = 0;
  if (int rc = dev_alloc(&g->d_rowtiles, (size_t)nb + 1)) return rc;
  TCMIS_CUDA(cudaMemcpyAsync(g->d_rowtiles, ct.data(), 4ull * (nb + 1), cudaMemcpyHostToDevice,
                             g->ctx->stream));
  TCMIS_CUDA(cudaStreamSynchronize(g->ctx->stream));
  g->tile_nb = nb;
  g->tile_total = tile_count;
  g->tile_T = T;
  return 0;
}

TCMIS_API int tcmis_graph_export_tiles(tcmis_graph *g, int32_t T, int32_t *tile_row,
                                       int32_t *tile_col, uint64_t *row_bits, int64_t *bro) {
  TCMIS_RANGE("tcmis_graph_export_tiles");
  NEED(g && bro, "null handle");
  ENTER(g->ctx);
  return export_tiles(g, T, tile_row, tile_col, row_bits, bro);
}

TCMIS_API int tcmis_graph_tile_store(tcmis_graph *g, int32_t T, int64_t *tile_count,
                                     int64_t *bro, int32_t *tile_col, void *payload) {
  TCMIS_RANGE("tcmis_graph_tile_store");
  NEED(g, "null graph");
  ENTER(g->ctx);
  if (int rc = build_tile_store(g, T)) return rc;
  const int32_t nb = (int32_t)(((int64_t)g->n + T - 1) / T);
  int64_t tiles = 0;
  cudaStream_t st = g->ctx->stream;
  TCMIS_CUDA(cudaMemcpyAsync(&tiles, g->d_tbro + nb, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (tile_count) *tile_count = tiles;
  if (bro) TCMIS_CUDA(cudaMemcpyAsync(bro, g->d_tbro, 8ull * (nb + 1), cudaMemcpyDeviceToHost, st));
  if (tile_col && tiles)
    TCMIS_CUDA(cudaMemcpyAsync(tile_col, g->d_tcol, 4ull * tiles, cudaMemcpyDeviceToHost, st));
  if (payload && tiles)
    TCMIS_CUDA(cudaMemcpyAsync(payload, g->d_tbits, (size_t)tiles * T * (T / 8),
                               cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

TCMIS_API int tcmis_validate(tcmis_graph *g, const int32_t *set, int64_t count,
                             int32_t *independent, int32_t *violating_u, int32_t *violating_v,
                             int32_t *maximal, int32_t *addable_vertex) {
  TCMIS_RANGE("tcmis_validate");
  NEED(g && independent && violating_u && violating_v && maximal && addable_vertex,
       "null handle");
  NEED(count >= 0 && (count == 0 || set), "null set");
  ENTER(g->ctx);
  return validate_impl(g, set, count, independent, violating_u, violating_v, maximal,
                       addable_vertex);
}

TCMIS_API int tcmis_priorities(tcmis_graph *g, int32_t heuristic, uint64_t seed,
                               int32_t scale_bits, uint32_t *p_out) {
  TCMIS_RANGE("tcmis_priorities");
  NEED(g && p_out, "null handle");
  ENTER(g->ctx);
  return priorities_impl(g, heuristic, seed, scale_bits, p_out);
}

static int solve_common(tcmis_graph *g, const tcmis_config *cfg, tcmis_iter_stats *stats,
                        int32_t max_stats, int32_t *n_iterations, int64_t *mis_count) {
  NEED(g && cfg, "null handle");
  ENTER(g->ctx);
  int32_t it = 0;
  int64_t mc = 0;
  int rc = solve_impl(g, cfg, stats, max_stats, &it, &mc);
  if (n_iterations) *n_iterations = it;
  if (mis_count) *mis_count = mc;
  return rc;
}

TCMIS_API int tcmis_solve(tcmis_graph *g, const tcmis_config *cfg, uint8_t *state_out,
                          int32_t *mis_out, int64_t *mis_count, tcmis_iter_stats *stats,
                          int32_t max_stats, int32_t *n_iterations) {
  TCMIS_RANGE("tcmis_solve");
  int64_t mc = 0;
  if (int rc = solve_common(g, cfg, stats, max_stats, n_iterations, &mc)) return rc;
  if (mis_count) *mis_count = mc;
  if (g->n == 0) return 0;
  cudaStream_t st = g->ctx->stream;
  if (state_out) {
    if (int rc = states_in_caller_order(g)) return rc;
    if (int rc = d2h(g->ctx, state_out, g->ws.relabeled ? g->ws.state_o : g->ws.state,
                     (size_t)g->n, st))
      return rc;
  }
  if (mis_out && mc)
    if (int rc = d2h(g->ctx, mis_out, g->ws.mis, 4ull * mc, st)) return rc;
  TCMIS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

TCMIS_API int tcmis_solve_device(tcmis_graph *g, const tcmis_config *cfg, const int32_t **d_mis,
                                 int64_t *mis_count, const uint8_t **d_state,
                                 tcmis_iter_stats *stats, int32_t max_stats,
                                 int32_t *n_iterations) {
  TCMIS_RANGE("tcmis_solve_device");
  if (int rc = solve_common(g, cfg, stats, max_stats, n_iterations, mis_count)) return rc;
  if (d_mis) *d_mis = g->ws.mis;
  if (d_state) {
    if (int rc = states_in_caller_order(g)) return rc;
    *d_state = g->ws.relabeled ? g->ws.state_o : g->ws.state;
  }
  return 0;
}

TCMIS_API int tcmis_graph_tile_cand_prepare(tcmis_graph *g, const tcmis_config *cfg,
                                            double *build_ms, int64_t *tiles) {
  TCMIS_RANGE("tcmis_graph_tile_cand_prepare");
  NEED(g && cfg, "null handle");
  if (cfg->heuristic < TCMIS_H1 || cfg->heuristic > TCMIS_LUBY_PERM ||
      cfg->heuristic == TCMIS_LUBY_FRESH)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "the A-up store needs fixed priorities");
  if (cfg->heuristic != TCMIS_H1 && (cfg->scale_bits < 8 || cfg->scale_bits > 30))
    return set_error(TCMIS_E_INVALID_ARGUMENT, "scale_bits must be in [8, 30]");
  ENTER(g->ctx);
  const int64_t key[3] = {cfg->heuristic, (int64_t)cfg->seed, cfg->scale_bits};
  double ms = 0;
  if (g->n > 0)
    if (int rc = tile_cand_prepare(g, cfg->heuristic, cfg->seed, cfg->scale_bits, key, &ms))
      return rc;
  if (build_ms) *build_ms = ms;
  if (tiles) *tiles = g->up_tiles;
  return 0;
}

TCMIS_API int tcmis_graph_permuted(tcmis_graph *g, tcmis_graph **out) {
  TCMIS_RANGE("tcmis_graph_permuted");
  NEED(g && out, "null handle");
  NEED(g->d_perm || g->n == 0, "tcmis_graph_reorder first");
  ENTER(g->ctx);
  int64_t *off = nullptr;
  int32_t *nbr = nullptr;
  if (int rc = dev_alloc(&off, (size_t)g->n + 1)) return rc;
  if (int rc = dev_alloc(&nbr, (size_t)std::max<int64_t>(g->nnz, 1))) return rc;
  cudaStream_t st = g->ctx->stream;
  if (g->n) {
    TCMIS_CUDA(cudaMemcpyAsync(off, g->d_roff, 8ull * (g->n + 1), cudaMemcpyDeviceToDevice, st));
    if (g->nnz)
      TCMIS_CUDA(cudaMemcpyAsync(nbr, g->d_rnbr, 4ull * g->nnz, cudaMemcpyDeviceToDevice, st));
  } else {
    TCMIS_CUDA(cudaMemsetAsync(off, 0, 8, st));
  }
  // rows ascending (graph.hpp:21 Graph invariant): reorder_impl sorted the
  // rows of <= kSortedMax entries, the longer ones here
  if (g->nnz && g->n)
    if (int rc = sort_rows(g->ctx, g->n, off, nbr, 2)) return rc;
  TCMIS_CUDA(cudaStreamSynchronize(st));
  return wrap_owned(g->ctx, g->n, g->nnz, off, nbr, out);
}

TCMIS_API int tcmis_graph_reorder(tcmis_graph *g, int32_t mode, const int32_t *order) {
  TCMIS_RANGE("tcmis_graph_reorder");
  NEED(g, "null handle");
  ENTER(g->ctx);
  return reorder_impl(g, mode, order);
}

TCMIS_API int tcmis_graph_upload_partition(tcmis_ctx *ctx, int32_t n, int32_t lo, int32_t hi,
                                           const int64_t *full_offsets,
                                           const int32_t *row_neighbors, tcmis_graph **out) {
  TCMIS_RANGE("tcmis_graph_upload_partition");
  NEED(ctx && out && full_offsets, "null handle");
  NEED(n >= 0, "vertex count must be non-negative");
  ENTER(ctx);
  return upload_partition(ctx, n, lo, hi, full_offsets, row_neighbors, out);
}

TCMIS_API int tcmis_graph_partition(tcmis_graph *full, int32_t lo, int32_t hi,
                                    tcmis_graph **out) {
  TCMIS_RANGE("tcmis_graph_partition");
  NEED(full && out, "null handle");
  ENTER(full->ctx);
  return partition_device(full, lo, hi, out);
}

TCMIS_API int tcmis_dist_begin(tcmis_graph *g, const tcmis_config *cfg) {
  NEED(g && cfg, "null handle");
  ENTER(g->ctx);
  return dist_begin(g, cfg);
}

TCMIS_API int tcmis_dist_select(tcmis_graph *g, uint32_t *d_bits, int32_t words) {
  NEED(g && d_bits, "null handle");
  ENTER(g->ctx);
  return dist_select(g, d_bits, words);
}

TCMIS_API int tcmis_dist_apply(tcmis_graph *g, const uint32_t *d_gathered,
                               const int32_t *rank_lo, int32_t world, int32_t maxw, int32_t me,
                               int32_t what) {
  NEED(g && d_gathered && rank_lo, "null handle");
  NEED(world >= 1 && me >= 0 && me < world && maxw >= 0, "bad rank layout");
  ENTER(g->ctx);
  return dist_apply(g, d_gathered, rank_lo, world, maxw, me, what);
}

TCMIS_API int tcmis_dist_update(tcmis_graph *g, uint32_t *d_bits, int32_t words,
                                int64_t *counts) {
  NEED(g && d_bits && counts, "null handle");  // counts: device int64[5]
  ENTER(g->ctx);
  return dist_update(g, d_bits, words, counts);
}

TCMIS_API int tcmis_dist_state(tcmis_graph *g, uint8_t *own_state) {
  NEED(g, "null handle");
  ENTER(g->ctx);
  return dist_state_out(g, own_state);
}

TCMIS_API int tcmis_dist_h3_tiles(tcmis_graph *g, int64_t *tiles_evaluated,
                                  int64_t *tile_total) {
  NEED(g && tiles_evaluated && tile_total, "null handle");
  ENTER(g->ctx);
  return dist_h3_tiles(g, tiles_evaluated, tile_total);
}

TCMIS_API int tcmis_h1_random(tcmis_ctx *ctx, int32_t n, uint64_t seed, uint32_t *p_out) {
  NEED(ctx && (n < 1 || p_out), "null handle");
  ENTER(ctx);
  return h1_impl(ctx, n, seed, p_out);
}

TCMIS_API int tcmis_h3_resolution(tcmis_graph *g, const uint32_t *p, const uint8_t *states,
                                  uint8_t *c_out) {
  TCMIS_RANGE("tcmis_h3_resolution");
  NEED(g && (g->n == 0 || (p && states && c_out)), "null handle");
  ENTER(g->ctx);
  return h3_resolution_impl(g, p, states, c_out);
}

TCMIS_API int tcmis_tiled_spmv_tiles(tcmis_ctx *ctx, int32_t n, int32_t T, int64_t tiles,
                                     const int32_t *tile_col, const uint64_t *row_bits,
                                     const int64_t *bro, const uint64_t *seg, int32_t exclusion,
                                     int32_t *nc, int64_t *ev, int64_t *sk) {
  TCMIS_RANGE("tcmis_tiled_spmv_tiles");
  NEED(ctx && ev && sk, "null handle");
  NEED(n == 0 || (bro && seg && nc), "null buffers");
  NEED(tiles == 0 || (tile_col && row_bits), "null tile buffers");
  ENTER(ctx);
  return tiled_spmv_tiles_impl(ctx, n, T, tiles, tile_col, row_bits, bro, seg, exclusion, nc, ev,
                               sk);
}

TCMIS_API int tcmis_compute_max_np(tcmis_graph *g, const uint32_t *p, const uint8_t *states,
                                   uint64_t *out) {
  NEED(g && p && states && out, "null handle");
  ENTER(g->ctx);
  return max_np_impl(g, p, states, out);
}

TCMIS_API int tcmis_neighbor_count(tcmis_graph *g, const uint8_t *c, int32_t *nc) {
  NEED(g && c && nc, "null handle");
  ENTER(g->ctx);
  return neighbor_count_impl(g, c, nc, 0, nullptr, nullptr);
}

TCMIS_API int tcmis_tiled_spmv(tcmis_graph *g, int32_t T, const uint8_t *c, int32_t exclusion,
                               int32_t *nc, int64_t *ev, int64_t *sk) {
  NEED(g && c && nc && ev && sk, "null handle");
  if (T < 1 || T > 64)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tile_dim must be in [1, 64], got " + std::to_string(T));
  (void)exclusion;
  ENTER(g->ctx);
  return neighbor_count_impl(g, c, nc, T, ev, sk);
}

TCMIS_API int tcmis_gen_rmat(tcmis_ctx *ctx, int32_t scale, int32_t ef, uint64_t seed,
                             tcmis_graph **out) {
  TCMIS_RANGE("tcmis_gen_rmat");
  NEED(ctx && out, "null handle");
  ENTER(ctx);
  return gen_rmat(ctx, scale, ef, seed, out);
}

TCMIS_API int tcmis_graph_from_edges(tcmis_ctx *ctx, int32_t n, int64_t m, const int32_t *u,
                                     const int32_t *v, tcmis_graph **out) {
  TCMIS_RANGE("tcmis_graph_from_edges");
  NEED(ctx && out && (m == 0 || (u && v)), "null handle");
  ENTER(ctx);
  return gen_from_edges(ctx, n, m, u, v, out);
}

TCMIS_API int tcmis_gen_grid(tcmis_ctx *ctx, int32_t side, tcmis_graph **out) {
  TCMIS_RANGE("tcmis_gen_grid");
  NEED(ctx && out, "null handle");
  ENTER(ctx);
  return gen_grid(ctx, side, out);
}

TCMIS_API int tcmis_gen_rgg(tcmis_ctx *ctx, int32_t n, uint64_t radius, uint64_t seed,
                            tcmis_graph **out) {
  TCMIS_RANGE("tcmis_gen_rgg");
  NEED(ctx && out, "null handle");
  ENTER(ctx);
  return gen_rgg(ctx, n, radius, seed, out);
}

TCMIS_API int tcmis_gen_gnp(tcmis_ctx *ctx, int32_t n, double avg_degree, uint64_t seed,
                            tcmis_graph **out) {
  TCMIS_RANGE("tcmis_gen_gnp");
  NEED(ctx && out, "null handle");
  ENTER(ctx);
  return gen_gnp(ctx, n, avg_degree, seed, out);
}

TCMIS_API int tcmis_gen_gnp_host(int32_t n, double avg, uint64_t seed, int64_t **offsets,
                                 int32_t **neighbors, int64_t *nnz) {
  NEED(offsets && neighbors && nnz, "null output");
  return gen_gnp_host(n, avg, seed, offsets, neighbors, nnz);
}

TCMIS_API void tcmis_free(void *p) { std::free(p); }

TCMIS_API uint64_t tcmis_rgg_radius(int32_t n, double avg) {
  if (n <= 0 || avg <= 0.0) return 0;
  const double r = std::sqrt(avg / (3.14159265358979323846 * (double)n));
  double R = std::floor(r * 4294967296.0);
  if (R > 4294967295.0) R = 4294967295.0;
  return (uint64_t)R;
}
