// dist.cu -- the per-rank device side of the row-partitioned multi-GPU solve.
//
// rank r owns the contiguous rows [lo_r, hi_r) (edge-balanced,
// boundaries aligned to a multiple of 64 and of the tile dimension) and holds
// them as a "partial CSR": offsets for all n vertices (rows outside the range
// are empty) and only its own neighbour lists, with global column ids.  Keys,
// states and decision flags are replicated for all n vertices.  One round is
//
//   select (own worklist)  -> publish own candidates as a bitmap slice
//   NCCL all-gather        -> every rank marks the remote candidates (next = 1)
//   pull exclusion + update (own check list) -> publish own removals
//   NCCL all-gather        -> every rank marks the remote removals (state Removed)
//   NCCL all-reduce of the round counters (host, distributed.py)
//
// i.e. exactly the reference's bulk-synchronous round (engine.cpp:247-291),
// so the MIS and every per-round statistic equal the single-GPU ones.  The
// kernels are the single-GPU ones; only the publish/apply steps are new.
// The host side (partitioning, collectives, termination) is
// paper_2605_29604_b200/distributed.py.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

int wrap_owned(tcmis_ctx *ctx, int32_t n, int64_t nnz, int64_t *d_off, int32_t *d_nbr,
               tcmis_graph **out);
int solve_prepare(tcmis_graph *g, const tcmis_config *cfg, RoundArgs &a, int64_t own_isolated);
int seg_total(tcmis_graph *g, int64_t *ev);

namespace {

// partial offsets: rows outside [lo, hi) are empty
__global__ void k_partial_offsets(int32_t n, int32_t lo, int32_t hi,
                                  const int64_t *__restrict__ full, int64_t *__restrict__ part) {
  const int64_t base = full[lo];
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = v < lo ? lo : (v > hi ? hi : v);
    part[v] = full[c] - base;
  }
}

// remote decisions from the gathered slices: rank r's slice starts at word
// r * maxw and holds bit (v - lo_r) of v in [lo_r, hi_r)
__global__ void k_apply_bits(const uint32_t *__restrict__ gathered,
                             const int32_t *__restrict__ rank_lo, int32_t world, int32_t maxw,
                             int32_t me, int what, uint8_t *__restrict__ next,
                             uint8_t *__restrict__ state, uint16_t *__restrict__ q) {
  const int64_t total = (int64_t)world * maxw;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(w / maxw);
    if (r == me) continue;
    uint32_t bits = gathered[w];
    const int64_t first = rank_lo[r] + (w - (int64_t)r * maxw) * 32;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t v = first + b;
      if (v >= rank_lo[r + 1]) break;
      if (what == 0) {  // remote candidate of this round
        next[v] = 1;
        state[v] = TCMIS_IN_MIS;
      } else {  // remote removal: invisible from now on
        state[v] = TCMIS_REMOVED;
        q[v] = 0;
      }
    }
  }
}

}  // namespace

int upload_partition(tcmis_ctx *ctx, int32_t n, int32_t lo, int32_t hi, const int64_t *full,
                     const int32_t *rows, tcmis_graph **out) {
  if (lo < 0 || hi < lo || hi > n)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "partition range outside [0, n]");
  cudaStream_t st = ctx->stream;
  const int64_t nnz = full[hi] - full[lo];
  int64_t *d_full = nullptr, *d_part = nullptr;
  int32_t *d_nbr = nullptr;
  if (int rc = dev_alloc(&d_full, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_part, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_nbr, (size_t)nnz)) return rc;
  if (int rc = h2d(ctx, d_full, full, 8ull * (n + 1), st)) return rc;
  if (nnz)
    if (int rc = h2d(ctx, d_nbr, rows, 4ull * nnz, st)) return rc;
  k_partial_offsets<<<grid_for(ctx, (int64_t)n + 1, 256, 16), 256, 0, st>>>(n, lo, hi, d_full,
                                                                            d_part);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (int rc = wrap_owned(ctx, n, nnz, d_part, d_nbr, out)) return rc;
  (*out)->d_off_full = d_full;
  (*out)->nnz_global = full[n];
  (*out)->part_lo = lo;
  (*out)->part_hi = hi;
  return 0;
}

struct DistState {
  RoundArgs a;
  bool active = false;
  int32_t round = 0;                 // rounds updated so far (all run in the round kernels)
  std::vector<int32_t> h_rank_lo;    // cached copy of the last rank layout ...
  int32_t *d_rank_lo = nullptr;      // ... and its device mirror (uploaded once)
};

// owned by the graph (created on first use, freed by tcmis_graph_destroy)
static DistState &dist_state(tcmis_graph *g) {
  if (!g->dist) g->dist = new DistState{};
  return *g->dist;
}

void free_dist(tcmis_graph *g) {
  if (!g->dist) return;
  dev_free(g->dist->d_rank_lo);
  delete g->dist;
  g->dist = nullptr;
}

int dist_begin(tcmis_graph *g, const tcmis_config *cfg) {
  if (g->part_hi < 0)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "graph is not a row partition");
  if (cfg->heuristic == TCMIS_LUBY_FRESH)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "luby-fresh redraws every alive key per round; the partitioned solve "
                     "runs the fixed-priority heuristics (h1, h2, h3, luby-perm)");
  DistState &d = dist_state(g);
  // own isolated vertices are round-1 candidates settled by k_priorities
  const int64_t own = (int64_t)g->part_hi - g->part_lo;
  if (int rc = ensure_workspace(g)) return rc;
  const int64_t own_nz = g->nz_count;  // non-empty rows of the partial CSR = own non-isolated
  if (int rc = solve_prepare(g, cfg, d.a, own - own_nz)) return rc;
  d.a.pull = 1;  // a push would have to reach remote rows
  d.a.tail_thr = 0;
  d.a.pub_lo = g->part_lo;
  d.active = true;
  d.round = 0;
  return 0;
}

int dist_select(tcmis_graph *g, uint32_t *d_bits, int32_t words) {
  DistState &d = dist_state(g);
  if (!d.active) return set_error(TCMIS_E_LOGIC, "tcmis_dist_begin first");
  TCMIS_CUDA(cudaMemsetAsync(d_bits, 0, 4ull * words, g->ctx->stream));
  d.a.pub_cand = d_bits;
  d.a.pub_dead = nullptr;
  return launch_select(g, d.a);
}

// Stream-ordered, no host synchronisation: the host driver enqueues
// select -> all-gather -> apply -> update -> all-gather -> apply -> all-reduce
// on the engine stream and reads one counter vector per round.
int dist_apply(tcmis_graph *g, const uint32_t *d_gathered, const int32_t *h_rank_lo,
               int32_t world, int32_t maxw, int32_t me, int32_t what) {
  tcmis_ctx *ctx = g->ctx;
  DistState &d = dist_state(g);
  if (d.h_rank_lo.size() != (size_t)world + 1 ||
      !std::equal(d.h_rank_lo.begin(), d.h_rank_lo.end(), h_rank_lo)) {
    dev_free(d.d_rank_lo);
    d.d_rank_lo = nullptr;
    if (int rc = dev_alloc(&d.d_rank_lo, (size_t)world + 1)) return rc;
    d.h_rank_lo.assign(h_rank_lo, h_rank_lo + world + 1);
    TCMIS_CUDA(cudaMemcpyAsync(d.d_rank_lo, d.h_rank_lo.data(), 4ull * (world + 1),
                               cudaMemcpyHostToDevice, ctx->stream));
    TCMIS_CUDA(cudaStreamSynchronize(ctx->stream));  // h_rank_lo storage may change
  }
  k_apply_bits<<<grid_for(ctx, (int64_t)world * maxw, 256, 8), 256, 0, ctx->stream>>>(
      d_gathered, d.d_rank_lo, world, maxw, me, what, g->ws.next, g->ws.state, g->ws.q);
  TCMIS_LAUNCHED(ctx);
  return 0;
}

// d_counts: DEVICE int64[5] = this rank's (selected, removed, alive,
// tiles_evaluated, tiles_skipped) of the round, copied stream-ordered from
// the DevRound k_round_end publishes (its first 5 x u64, in that order).
int dist_update(tcmis_graph *g, uint32_t *d_bits, int32_t words, int64_t *d_counts) {
  static_assert(offsetof(DevRound, skip) == 4 * sizeof(int64_t), "DevRound layout");
  DistState &d = dist_state(g);
  if (!d.active) return set_error(TCMIS_E_LOGIC, "tcmis_dist_begin first");
  cudaStream_t st = g->ctx->stream;
  TCMIS_CUDA(cudaMemsetAsync(d_bits, 0, 4ull * words, st));
  d.a.pub_cand = nullptr;
  d.a.pub_dead = d_bits;
  if (int rc = launch_update(g, d.a, 0, 0)) return rc;
  Workspace &ws = g->ws;
  const int32_t round = ++d.round;
  TCMIS_CUDA(cudaMemcpyAsync(d_counts, ws.rounds + (round - 1) % ws.round_cap,
                             5 * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  return 0;
}

// h3 (one collapsed iteration): tiles of the own block columns holding any
// MIS vertex, and the own tile total
int dist_h3_tiles(tcmis_graph *g, int64_t *ev, int64_t *total) {
  if (int rc = seg_total(g, ev)) return rc;
  *total = g->tile_total;
  return 0;
}

// A rank's partition built from a device-resident full graph (e.g. the
// device generators): offsets copied, own rows' neighbour lists sliced, both
// device to device.
int partition_device(tcmis_graph *full, int32_t lo, int32_t hi, tcmis_graph **out) {
  tcmis_ctx *ctx = full->ctx;
  const int32_t n = full->n;
  if (lo < 0 || hi < lo || hi > n)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "partition range outside [0, n]");
  cudaStream_t st = ctx->stream;
  int64_t ends[2] = {0, 0};
  TCMIS_CUDA(cudaMemcpyAsync(&ends[0], full->d_off + lo, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaMemcpyAsync(&ends[1], full->d_off + hi, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  const int64_t nnz = ends[1] - ends[0];
  int64_t *d_full = nullptr, *d_part = nullptr;
  int32_t *d_nbr = nullptr;
  if (int rc = dev_alloc(&d_full, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_part, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_nbr, (size_t)nnz)) return rc;
  TCMIS_CUDA(cudaMemcpyAsync(d_full, full->d_off, 8ull * (n + 1), cudaMemcpyDeviceToDevice, st));
  if (nnz)
    TCMIS_CUDA(cudaMemcpyAsync(d_nbr, full->d_nbr + ends[0], 4ull * nnz, cudaMemcpyDeviceToDevice,
                               st));
  k_partial_offsets<<<grid_for(ctx, (int64_t)n + 1, 256, 16), 256, 0, st>>>(n, lo, hi, d_full,
                                                                            d_part);
  TCMIS_LAUNCHED(ctx);
  int64_t total = 0;
  TCMIS_CUDA(cudaMemcpyAsync(&total, full->d_off + n, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (int rc = wrap_owned(ctx, n, nnz, d_part, d_nbr, out)) return rc;
  (*out)->d_off_full = d_full;
  (*out)->nnz_global = total;
  (*out)->part_lo = lo;
  (*out)->part_hi = hi;
  return 0;
}

int dist_state_out(tcmis_graph *g, uint8_t *own_state) {
  const int64_t own = (int64_t)g->part_hi - g->part_lo;
  if (own > 0)
    TCMIS_CUDA(cudaMemcpy(own_state, g->ws.state + g->part_lo, (size_t)own,
                          cudaMemcpyDeviceToHost));
  dist_state(g).active = false;
  return 0;
}

}  // namespace tcmis_b200
