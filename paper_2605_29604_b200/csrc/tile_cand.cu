// tile_cand.cu -- Phase 1 (candidate detection) as a tile x bit-vector
// product: the oriented adjacency A-up over the compact T = 16 tile store
// (SURVEY 7 "Phase 1 as a true SpMV").
//
// Priorities are fixed for the whole solve (engine.cpp:242), so "u is a
// neighbour of v with a larger key" is a static relation: A-up[v][u] = 1 iff
// u in N(v) and key(u) > key(v) (priorities.hpp:61-64).  It holds exactly m of
// the 2m entries, and
//
//     C = alive AND NOT (A-up * alive > 0)
//
// is compute_max_np + generate_candidates (engine.cpp:86-119) bit for bit.
// With A-up in the compact tile store, a round's Phase 1 is the tile kernel
// k_tile_excl_bits over (A-up tiles, alive bitmap) -- the very product the
// tile-form exclusion runs over (A tiles, candidate bitmap) -- plus one pass
// that turns "not blocked" into candidates.  No priority gathers at all in the
// rounds: only 16-bit alive segments.
//
// The catch is that A-up depends on the priorities, i.e. on (heuristic, seed,
// scale_bits): orienting the CSR and tiling it is one pass over all 2m
// entries with a key comparison each (as much work as a Phase 1 without early
// exit) plus the tiling, paid per priority configuration.  The store is
// cached on the graph for repeated solves with the same configuration.
// Measured keep/drop: profiles/r02/phase1_tiles.md.
#include <cub/cub.cuh>

#include "internal.cuh"
#include "common.cuh"

namespace tcmis_b200 {

int build_tile_store(tcmis_graph *g, int T);  // tiles.cu
int wrap_owned(tcmis_ctx *ctx, int32_t n, int64_t nnz, int64_t *d_off, int32_t *d_nbr,
               tcmis_graph **out);

namespace {

__device__ __forceinline__ bool higher(const uint32_t *__restrict__ p, int32_t u, int32_t v) {
  const uint32_t pu = __ldg(&p[u]), pv = __ldg(&p[v]);
  return pu != pv ? pu > pv : u > v;  // key = (p << 32) | (id + 1)
}

// warp per row: the number of higher-key neighbours (pass 0) or the row of
// A-up itself, in the CSR's entry order (pass 1)
template <bool kFill>
__global__ void k_orient(int32_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                         const uint32_t *__restrict__ p, int64_t *__restrict__ uoff,
                         int32_t *__restrict__ unbr) {
  const int lane = threadIdx.x & 31;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t s = off[v], e = off[v + 1];
    int64_t base = kFill ? uoff[v] : 0;
    int64_t cnt = 0;
    for (int64_t k0 = s; k0 < e; k0 += 32) {
      const int64_t k = k0 + lane;
      const int32_t u = k < e ? __ldg(&nbr[k]) : -1;
      const bool keep = u >= 0 && higher(p, u, (int32_t)v);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (kFill && keep) unbr[base + __popc(m & ((1u << lane) - 1u))] = u;
      base += __popc(m);
      cnt += __popc(m);
    }
    if (!kFill && lane == 0) uoff[v] = cnt;
  }
}

}  // namespace

void free_up_store(tcmis_graph *g) {
  dev_free(g->d_up_trow);
  dev_free(g->d_up_tcol);
  dev_free(g->d_up_tbits);
  g->d_up_trow = g->d_up_tcol = nullptr;
  g->d_up_tbits = nullptr;
  g->up_tiles = 0;
  g->up_key[0] = -1;
}

// The A-up tile store of the priorities p (device, n entries) under the
// configuration key (heuristic, seed, scale_bits); a no-op when cached.
int build_up_store(tcmis_graph *g, const uint32_t *p, const int64_t key[3], double *build_ms) {
  if (g->d_up_trow && g->up_key[0] == key[0] && g->up_key[1] == key[1] && g->up_key[2] == key[2])
    return 0;
  free_up_store(g);
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int32_t n = g->n;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (build_ms) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
  }
  int64_t *uoff = nullptr;
  int32_t *unbr = nullptr;
  if (int rc = dev_alloc(&uoff, (size_t)n + 1)) return rc;
  k_orient<false><<<grid_for(ctx, 32ll * n, 256, 16), 256, 0, st>>>(n, g->d_off, g->d_nbr, p,
                                                                    uoff, nullptr);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaMemsetAsync(uoff + n, 0, 8, st));
  {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, uoff, uoff, (int64_t)n + 1, st);
    void *tmp = nullptr;
    if (int rc = dev_alloc((char **)&tmp, bytes)) return rc;
    TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, uoff, uoff, (int64_t)n + 1, st));
    ctx->launches++;
    dev_free(tmp);
  }
  int64_t m_up = 0;
  TCMIS_CUDA(cudaMemcpyAsync(&m_up, uoff + n, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (int rc = dev_alloc(&unbr, (size_t)std::max<int64_t>(m_up, 1))) return rc;
  k_orient<true><<<grid_for(ctx, 32ll * n, 256, 16), 256, 0, st>>>(n, g->d_off, g->d_nbr, p, uoff,
                                                                   unbr);
  TCMIS_LAUNCHED(ctx);
  // the tiling of the oriented CSR (tiles.cu build_tile_store) on a
  // temporary handle whose store is then taken over
  tcmis_graph *tmp = nullptr;
  if (int rc = wrap_owned(ctx, n, m_up, uoff, unbr, &tmp)) return rc;
  int rc = build_tile_store(tmp, 16);
  if (!rc) {
    g->d_up_trow = tmp->d_trow;
    g->d_up_tcol = tmp->d_tcol;
    g->d_up_tbits = static_cast<uint16_t *>(tmp->d_tbits);
    g->up_tiles = tmp->store_tiles;
    tmp->d_trow = tmp->d_tcol = nullptr;
    tmp->d_tbits = nullptr;
    g->up_key[0] = key[0];
    g->up_key[1] = key[1];
    g->up_key[2] = key[2];
  }
  dev_free(tmp->d_tbro);
  dev_free(tmp->d_trow);
  dev_free(tmp->d_tcol);
  dev_free(tmp->d_tbits);
  dev_free(uoff);
  dev_free(unbr);
  delete tmp;
  if (build_ms) {
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    *build_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  return rc;
}

}  // namespace tcmis_b200
