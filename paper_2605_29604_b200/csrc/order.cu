// order.cu -- an internal vertex order for the solve kernels (locality).
//
// The round kernels gather q / state / next of every neighbour they visit, so
// their speed is set by how many distinct L2 sectors those gathers touch.  A
// graph whose ids scatter its neighbourhoods over the id space (RGG in draw
// order: 1.00 nonzero per 16x16 tile; R-MAT: hubs spread over the ids with
// few one-bits, half the ids isolated) wastes most of every sector it reads.
// tcmis_graph_reorder keeps the caller's CSR and ids and adds a relabeled
// copy of the CSR (solve id i = the caller's vertex perm[i]):
//
//   TCMIS_ORDER_DEGREE   by degree, descending, ties by id (stable): R-MAT's
//                        hubs -- the most gathered vertices -- share sectors,
//                        and the isolated vertices leave the gathered range;
//   TCMIS_ORDER_SPATIAL  tcmis_gen_rgg's points by Morton code of their grid
//                        cell: a vertex's neighbours sit in the same or the
//                        adjacent cells, i.e. at nearby solve ids;
//   TCMIS_ORDER_GIVEN    a permutation the caller supplies.
//
// Nothing about the MIS changes: keys are (p[v], v) of the caller's ids
// (priorities.hpp:61-64) -- the kernels compare q / p and, on a p tie, the
// caller's ids through perm (common.cuh orig_id) --, hash priorities hash the
// caller's id, the tile counters flag the caller's block columns, and the
// result is mapped back (k_unpermute + an ordered compaction).  The rounds
// therefore equal the reference's bit for bit; tests/test_gpu_parity.py
// checks relabeled against direct solves.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

namespace {

__global__ void k_degree_keys(int32_t n, const int64_t *__restrict__ off,
                              uint32_t *__restrict__ key, int32_t *__restrict__ id) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = off[v + 1] - off[v];
    key[v] = ~(uint32_t)(d > 0xffffffffLL ? 0xffffffffLL : d);  // ascending key = descending degree
    id[v] = (int32_t)v;
  }
}

// inv[perm[i]] = i; a value outside [0, n) or seen twice flags `bad`
__global__ void k_invert(int32_t n, const int32_t *__restrict__ perm, int32_t *__restrict__ inv,
                         int *__restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[i];
    if (v < 0 || v >= n) {
      *bad = 1;
      continue;
    }
    if (atomicExch(&inv[v], (int32_t)i) != -1) *bad = 1;
  }
}

__global__ void k_relabel_degrees(int32_t n, const int32_t *__restrict__ perm,
                                  const int64_t *__restrict__ off, int64_t *__restrict__ roff) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = perm[i];
    roff[i] = off[v + 1] - off[v];
  }
}

// warp per solve row: the caller's row perm[i], every id mapped through inv
// (the row keeps the caller's entry order)
__global__ void k_relabel_rows(int32_t n, const int32_t *__restrict__ perm,
                               const int32_t *__restrict__ inv, const int64_t *__restrict__ off,
                               const int32_t *__restrict__ nbr, const int64_t *__restrict__ roff,
                               int32_t *__restrict__ rnbr) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t v = perm[i];
    const int64_t s = off[v], e = off[v + 1], d = roff[i];
    for (int64_t k = s + lane; k < e; k += 32) rnbr[d + (k - s)] = __ldg(&inv[__ldg(&nbr[k])]);
  }
}

struct HasEdgesR {
  const int64_t *off;
  __device__ __forceinline__ bool operator()(int32_t v) const { return off[v + 1] > off[v]; }
};

}  // namespace

void free_order(tcmis_graph *g) {
  dev_free(g->d_perm);
  dev_free(g->d_inv);
  dev_free(g->d_roff);
  dev_free(g->d_rnbr);
  dev_free(g->d_rnz);
  g->d_perm = nullptr;
  g->d_inv = nullptr;
  g->d_roff = nullptr;
  g->d_rnbr = nullptr;
  g->d_rnz = nullptr;
  g->rnz_count = 0;
  g->order_mode = TCMIS_ORDER_NONE;
}

namespace {
int scan_in_place(tcmis_ctx *ctx, int64_t *d, int64_t count) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, d, d, count, ctx->stream);
  void *tmp = nullptr;
  if (int rc = dev_alloc((char **)&tmp, bytes)) return rc;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, bytes, d, d, count, ctx->stream);
  ctx->launches++;
  dev_free(tmp);
  return e == cudaSuccess ? 0 : cuda_error(e, "relabeled offsets");
}
}  // namespace

int reorder_impl(tcmis_graph *g, int32_t mode, const int32_t *order) {
  if (mode == TCMIS_ORDER_NONE) {
    free_order(g);
    return 0;
  }
  if (mode != TCMIS_ORDER_DEGREE && mode != TCMIS_ORDER_SPATIAL && mode != TCMIS_ORDER_GIVEN)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "unknown vertex order");
  if (g->part_hi >= 0)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "a row partition keeps the caller's ids");
  if (mode == TCMIS_ORDER_SPATIAL && !g->d_spatial)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "TCMIS_ORDER_SPATIAL needs a graph from tcmis_gen_rgg (its point order)");
  if (mode == TCMIS_ORDER_GIVEN && !order && g->n > 0)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "TCMIS_ORDER_GIVEN needs the order");
  free_order(g);
  const int32_t n = g->n;
  if (n == 0) {
    g->order_mode = mode;
    return 0;
  }
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  int32_t *perm = nullptr, *inv = nullptr;
  int *bad = nullptr;
  int rc = dev_alloc(&perm, (size_t)n);
  if (!rc) rc = dev_alloc(&inv, (size_t)n);
  if (!rc) rc = dev_alloc(&bad, 1);
  if (!rc && mode == TCMIS_ORDER_DEGREE) {
    uint32_t *key = nullptr, *key2 = nullptr;
    int32_t *id = nullptr;
    rc = dev_alloc(&key, (size_t)n);
    if (!rc) rc = dev_alloc(&key2, (size_t)n);
    if (!rc) rc = dev_alloc(&id, (size_t)n);
    if (!rc) {
      k_degree_keys<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, g->d_off, key, id);
      ctx->launches++;
      size_t bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, bytes, key, key2, id, perm, n, 0, 32, st);
      void *tmp = nullptr;
      rc = dev_alloc((char **)&tmp, bytes);
      if (!rc) {
        cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, bytes, key, key2, id, perm, n, 0, 32, st);
        if (e != cudaSuccess) rc = cuda_error(e, "degree order");
        ctx->launches++;
      }
      dev_free(tmp);
    }
    dev_free(key);
    dev_free(key2);
    dev_free(id);
  } else if (!rc && mode == TCMIS_ORDER_SPATIAL) {
    cudaError_t e = cudaMemcpyAsync(perm, g->d_spatial, 4ull * n, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) rc = cuda_error(e, "spatial order");
  } else if (!rc) {
    rc = h2d(ctx, perm, order, 4ull * n, st);
  }
  if (!rc) {
    cudaMemsetAsync(inv, 0xff, 4ull * n, st);
    cudaMemsetAsync(bad, 0, sizeof(int), st);
    k_invert<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, perm, inv, bad);
    ctx->launches++;
    int h_bad = 0;
    cudaMemcpyAsync(&h_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "vertex order");
    else if (h_bad) rc = set_error(TCMIS_E_INVALID_ARGUMENT, "the order is not a permutation of [0, n)");
  }
  int64_t *roff = nullptr;
  int32_t *rnbr = nullptr, *rnz = nullptr;
  if (!rc) rc = dev_alloc(&roff, (size_t)n + 1);
  if (!rc) rc = dev_alloc(&rnbr, (size_t)std::max<int64_t>(g->nnz, 1));
  if (!rc) rc = dev_alloc(&rnz, (size_t)n);
  if (!rc) {
    k_relabel_degrees<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, perm, g->d_off, roff);
    ctx->launches++;
    cudaMemsetAsync(roff + n, 0, 8, st);
    rc = scan_in_place(ctx, roff, (int64_t)n + 1);
  }
  if (!rc) {
    k_relabel_rows<<<grid_for(ctx, 32ll * n, 256, 16), 256, 0, st>>>(n, perm, inv, g->d_off,
                                                                     g->d_nbr, roff, rnbr);
    ctx->launches++;
    thrust::counting_iterator<int32_t> ids(0);
    size_t bytes = 0;
    int64_t *d_cnt = nullptr;
    rc = dev_alloc(&d_cnt, 1);
    cub::DeviceSelect::If(nullptr, bytes, ids, rnz, d_cnt, n, HasEdgesR{roff}, st);
    void *tmp = nullptr;
    if (!rc) rc = dev_alloc((char **)&tmp, bytes);
    if (!rc) {
      cub::DeviceSelect::If(tmp, bytes, ids, rnz, d_cnt, n, HasEdgesR{roff}, st);
      ctx->launches++;
      int64_t cnt = 0;
      cudaMemcpyAsync(&cnt, d_cnt, 8, cudaMemcpyDeviceToHost, st);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = cuda_error(e, "relabeled CSR");
      g->rnz_count = (int32_t)cnt;
    }
    dev_free(tmp);
    dev_free(d_cnt);
  }
  dev_free(bad);
  if (rc) {
    dev_free(inv);
    dev_free(perm);
    dev_free(roff);
    dev_free(rnbr);
    dev_free(rnz);
    return rc;
  }
  g->d_perm = perm;
  g->d_inv = inv;
  g->d_roff = roff;
  g->d_rnbr = rnbr;
  g->d_rnz = rnz;
  g->order_mode = mode;
  return 0;
}

}  // namespace tcmis_b200
