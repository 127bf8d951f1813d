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
//   TCMIS_ORDER_DEGREE   by degree, descending, ties by id (stable; for a
//                        tcmis_gen_rgg graph ties in its points' spatial
//                        order): R-MAT's hubs -- the most gathered vertices
//                        -- share sectors, the isolated vertices leave the
//                        gathered range, and the degree classes carry the
//                        H2 key bounds (solver.cu k_class_bounds);
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

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

namespace {

// the sort's input sequence: the caller's ids, or (tcmis_gen_rgg graphs) its
// points in spatial order, so that the stable sort keeps each degree class
// in that order and the gathers keep their locality within a class
__global__ void k_degree_keys(int32_t n, const int64_t *__restrict__ off,
                              const int32_t *__restrict__ seq, uint32_t *__restrict__ key,
                              int32_t *__restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = seq ? seq[i] : (int32_t)i;
    const int64_t d = off[v + 1] - off[v];
    key[i] = ~(uint32_t)(d > 0xffffffffLL ? 0xffffffffLL : d);  // ascending key = descending degree
    id[i] = v;
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
// (then sorted per row, reorder_impl)
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

// the first solve id of every degree class (ids sorted by descending degree)
struct ClassHead {
  const int64_t *off;
  __device__ __forceinline__ bool operator()(int32_t i) const {
    return i == 0 || off[i + 1] - off[i] != off[i] - off[i - 1];
  }
};

// ---- the rows of the relabeled CSR sorted ascending, in place.  Rows are
// binned by length into tiers (k_bin_rows: counts, then lists), and each tier
// is a merge sort sized to within 2x of its rows: logical warps of 8 threads
// x 4 keys (rows of <= 32 entries, most of them), warps of 32 x 2..16 (<=
// 512), blocks of 128 / 256 threads x 8..16 (<= 4096).  Rows longer than
// kSortedMax are hubs; the solve does not need them sorted (their class
// bounds carry lo = 0, k_class_bounds) and tcmis_graph_permuted sorts them
// with one device-wide radix pass over (row, id) keys.  (One cub
// DeviceSegmentedSort over all rows took 225 ms at R-MAT s26: a block per
// segment serialises the hubs.)
struct IdLess {
  __device__ __forceinline__ bool operator()(int32_t a, int32_t b) const { return a < b; }
};

constexpr int kTiers = 9;  // <=32, 64, 128, 256, 512, 1024, 2048, 4096, longer
__device__ __forceinline__ int row_tier(int64_t len) {
  if (len <= 32) return 0;
  if (len > kSortedMax) return kTiers - 1;
  return 64 - __clzll(len - 1) - 5;  // ceil(log2 len) - 5
}

// pass 0: per-tier counts; pass 1: the lists (cursor[t] starts at the tier's
// offset)
template <bool kFill>
__global__ void k_bin_rows(int32_t n, const int64_t *__restrict__ off, int32_t *__restrict__ cursor,
                           int32_t *__restrict__ list) {
  __shared__ int32_t s_cnt[kTiers], s_base[kTiers];
  if (threadIdx.x < kTiers) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const int64_t len = v < n ? off[v + 1] - off[v] : 0;
    const int t = len >= 2 ? row_tier(len) : -1;
    int slot = 0;
    if (t >= 0) slot = atomicAdd(&s_cnt[t], 1);
    if (kFill) {
      __syncthreads();
      if (threadIdx.x < kTiers) {
        s_base[threadIdx.x] = s_cnt[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], s_cnt[threadIdx.x]) : 0;
        s_cnt[threadIdx.x] = 0;
      }
      __syncthreads();
      if (t >= 0) list[s_base[t] + slot] = (int32_t)v;
      __syncthreads();
    }
  }
  if (!kFill) {
    __syncthreads();
    if (threadIdx.x < kTiers && s_cnt[threadIdx.x]) atomicAdd(&cursor[threadIdx.x], s_cnt[threadIdx.x]);
  }
}

template <int kThreads, int kItems>
__global__ void __launch_bounds__(256) k_sort_rows_warp(const int32_t *__restrict__ rows, int32_t cnt,
                                                        const int64_t *__restrict__ off,
                                                        int32_t *__restrict__ nbr) {
  using Sort = cub::WarpMergeSort<int32_t, kItems, kThreads>;
  constexpr int kWarps = 256 / kThreads;
  __shared__ typename Sort::TempStorage tmp[kWarps];
  const int w = threadIdx.x / kThreads, t = threadIdx.x % kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kWarps + w; i < cnt; i += (int64_t)gridDim.x * kWarps) {
    const int32_t v = rows[i];
    const int64_t s = off[v], len = off[v + 1] - s;
    int32_t k[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int idx = t * kItems + j;
      k[j] = idx < len ? nbr[s + idx] : 0x7fffffff;
    }
    Sort(tmp[w]).Sort(k, IdLess(), (int)len, 0x7fffffff);
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int idx = t * kItems + j;
      if (idx < len) nbr[s + idx] = k[j];
    }
  }
}

template <int kThreads, int kItems>
__global__ void __launch_bounds__(kThreads) k_sort_rows_block(const int32_t *__restrict__ rows,
                                                              int32_t cnt,
                                                              const int64_t *__restrict__ off,
                                                              int32_t *__restrict__ nbr) {
  using Sort = cub::BlockMergeSort<int32_t, kThreads, kItems>;
  __shared__ typename Sort::TempStorage tmp;
  for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int32_t v = rows[i];
    const int64_t s = off[v], len = off[v + 1] - s;
    int32_t k[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int idx = threadIdx.x * kItems + j;
      k[j] = idx < len ? nbr[s + idx] : 0x7fffffff;
    }
    Sort(tmp).Sort(k, IdLess(), (int)len, 0x7fffffff);
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int idx = threadIdx.x * kItems + j;
      if (idx < len) nbr[s + idx] = k[j];
    }
    __syncthreads();  // tmp is reused by the next row
  }
}

__global__ void k_long_rows_len(int32_t cnt, const int32_t *__restrict__ rows,
                                const int64_t *__restrict__ off, int64_t *__restrict__ boff) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
    boff[i] = off[rows[i] + 1] - off[rows[i]];
}

// the listed rows to one buffer of (list index << 32 | id) keys and back
template <bool kOut>
__global__ void k_long_rows_copy(int32_t cnt, const int32_t *__restrict__ rows,
                                 const int64_t *__restrict__ off, const int64_t *__restrict__ boff,
                                 int32_t *__restrict__ nbr, uint64_t *__restrict__ buf) {
  for (int32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int64_t s = off[rows[i]], len = off[rows[i] + 1] - s, b = boff[i];
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
      if (kOut) buf[b + k] = ((uint64_t)i << 32) | (uint32_t)nbr[s + k];
      else nbr[s + k] = (int32_t)(uint32_t)buf[b + k];
    }
  }
}

// round 1's settling data (select.cuh r1_max / r1_cls): per solve id the
// largest neighbour id -- the row's last entry when the row is sorted, a
// block reduction for the hub rows, which are the ids [0, H) of the degree
// order -- and the degree class
__global__ void k_row_max(int32_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                          int32_t *__restrict__ rmax, int32_t *__restrict__ hub_end) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = off[v], e = off[v + 1];
    rmax[v] = e == s ? -1 : (e - s <= kSortedMax ? nbr[e - 1] : -2);
    // the first id whose row is sorted (degrees descend)
    if (e - s <= kSortedMax && (v == 0 || off[v] - off[v - 1] > kSortedMax)) *hub_end = (int32_t)v;
  }
}
__global__ void k_hub_max(const int32_t *__restrict__ hub_end, const int64_t *__restrict__ off,
                          const int32_t *__restrict__ nbr, int32_t *__restrict__ rmax) {
  __shared__ int32_t s_m[32];
  const int32_t h = *hub_end;
  for (int32_t v = blockIdx.x; v < h; v += gridDim.x) {
    int32_t m = -1;
    for (int64_t k = off[v] + threadIdx.x; k < off[v + 1]; k += blockDim.x) m = max(m, nbr[k]);
    m = __reduce_max_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
      m = threadIdx.x < (int)(blockDim.x >> 5) ? s_m[threadIdx.x] : -1;
      m = __reduce_max_sync(0xffffffffu, m);
      if (threadIdx.x == 0) rmax[v] = m;
    }
    __syncthreads();
  }
}
__global__ void k_class_degree(int32_t ncls, const int32_t *__restrict__ cls,
                               const int64_t *__restrict__ off, int32_t *__restrict__ deg) {
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncls; c += gridDim.x * blockDim.x)
    deg[c] = (int32_t)(off[cls[c] + 1] - off[cls[c]]);
}
__global__ void k_vertex_class(int32_t n, int32_t ncls, const int32_t *__restrict__ cls,
                               uint16_t *__restrict__ vcls) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = 0, b = ncls - 1;  // last class starting at or before v
    while (a < b) {
      const int32_t m = (a + b + 1) >> 1;
      if (__ldg(&cls[m]) <= v) a = m; else b = m - 1;
    }
    vcls[v] = (uint16_t)a;
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
  dev_free(g->d_cls_start);
  dev_free(g->d_cb);
  dev_free(g->d_cbc);
  dev_free(g->d_rmax);
  dev_free(g->d_vcls);
  dev_free(g->d_cls_deg);
  g->d_cls_deg = nullptr;
  g->d_cbc = nullptr;
  g->d_rmax = nullptr;
  g->d_vcls = nullptr;
  g->d_cls_start = nullptr;
  g->d_cb = nullptr;
  g->n_cls = 0;
  g->cb_scale_bits = -1;
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

// TCMIS_ORDER_TRACE: the stages' wall times on stderr (synchronised)
struct StageClock {
  bool on = std::getenv("TCMIS_ORDER_TRACE") != nullptr;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char *what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tcmis order] %s %.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

int sort_long_rows(tcmis_ctx *ctx, const int32_t *rows, int32_t h_cnt, const int64_t *off,
                   int32_t *nbr) {
  cudaStream_t st = ctx->stream;
  int64_t *boff = nullptr;
  uint64_t *buf = nullptr, *buf2 = nullptr;
  int rc = dev_alloc(&boff, (size_t)h_cnt + 1);
  if (!rc) {
    k_long_rows_len<<<grid_for(ctx, h_cnt, 256, 4), 256, 0, st>>>(h_cnt, rows, off, boff);
    cudaMemsetAsync(boff + h_cnt, 0, 8, st);
    ctx->launches++;
    rc = scan_in_place(ctx, boff, (int64_t)h_cnt + 1);
  }
  int64_t total = 0;
  if (!rc) {
    cudaMemcpyAsync(&total, boff + h_cnt, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "row sort");
  }
  if (!rc) rc = dev_alloc(&buf, (size_t)total);
  if (!rc) rc = dev_alloc(&buf2, (size_t)total);
  if (!rc) {
    const int grid = std::min(h_cnt, ctx->num_sms * 8);
    k_long_rows_copy<true><<<grid, 256, 0, st>>>(h_cnt, rows, off, boff, nbr, buf);
    // key bits: the id (< 2^31) and the list index above bit 32
    const int end_bit = 32 + (32 - __builtin_clz((unsigned)std::max(h_cnt, 2)));
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, buf, buf2, total, 0, end_bit, st);
    void *tmp = nullptr;
    rc = dev_alloc((char **)&tmp, bytes);
    if (!rc) {
      cudaError_t e = cub::DeviceRadixSort::SortKeys(tmp, bytes, buf, buf2, total, 0, end_bit, st);
      if (e != cudaSuccess) rc = cuda_error(e, "row sort");
    }
    if (!rc) k_long_rows_copy<false><<<grid, 256, 0, st>>>(h_cnt, rows, off, boff, nbr, buf2);
    ctx->launches += 3;
    cudaError_t e = cudaStreamSynchronize(st);  // before the buffers go
    if (!rc && e != cudaSuccess) rc = cuda_error(e, "row sort");
    dev_free(tmp);
  }
  dev_free(boff);
  dev_free(buf);
  dev_free(buf2);
  return rc;
}

}  // namespace

// the rows of (off, nbr) ascending: which & 1 the rows of <= kSortedMax
// entries, which & 2 the longer ones (the solve leaves those in any order)
int sort_rows(tcmis_ctx *ctx, int32_t n, const int64_t *off, int32_t *nbr, int which) {
  cudaStream_t st = ctx->stream;
  StageClock clk{};
  clk.st = st;
  int32_t *cursor = nullptr, *list = nullptr;
  int rc = dev_alloc(&cursor, kTiers);
  if (!rc) rc = dev_alloc(&list, (size_t)std::max(n, 1));
  int32_t cnt[kTiers] = {}, first[kTiers] = {};
  if (!rc) {
    const int grid = grid_for(ctx, n, 256, 8);
    cudaMemsetAsync(cursor, 0, 4 * kTiers, st);
    k_bin_rows<false><<<grid, 256, 0, st>>>(n, off, cursor, list);
    cudaMemcpyAsync(cnt, cursor, 4 * kTiers, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "row sort");
    for (int t = 1; t < kTiers; ++t) first[t] = first[t - 1] + cnt[t - 1];
    if (!rc) {
      cudaMemcpyAsync(cursor, first, 4 * kTiers, cudaMemcpyHostToDevice, st);
      k_bin_rows<true><<<grid, 256, 0, st>>>(n, off, cursor, list);
      ctx->launches += 2;
    }
  }
  clk.mark("sort: bins");
  if (!rc && (which & 1)) {
    const int g = ctx->num_sms * 16;
    auto L = [&](int t) { return list + first[t]; };
    if (cnt[0]) k_sort_rows_warp<8, 4><<<g, 256, 0, st>>>(L(0), cnt[0], off, nbr);
    if (cnt[1]) k_sort_rows_warp<32, 2><<<g, 256, 0, st>>>(L(1), cnt[1], off, nbr);
    if (cnt[2]) k_sort_rows_warp<32, 4><<<g, 256, 0, st>>>(L(2), cnt[2], off, nbr);
    if (cnt[3]) k_sort_rows_warp<32, 8><<<g, 256, 0, st>>>(L(3), cnt[3], off, nbr);
    if (cnt[4]) k_sort_rows_warp<32, 16><<<g, 256, 0, st>>>(L(4), cnt[4], off, nbr);
    if (cnt[5]) k_sort_rows_block<128, 8><<<g, 128, 0, st>>>(L(5), cnt[5], off, nbr);
    if (cnt[6]) k_sort_rows_block<128, 16><<<g, 128, 0, st>>>(L(6), cnt[6], off, nbr);
    if (cnt[7]) k_sort_rows_block<256, 16><<<g, 256, 0, st>>>(L(7), cnt[7], off, nbr);
    ctx->launches += 8;
    clk.mark("sort: rows <= 4096");
  }
  if (!rc && (which & 2) && cnt[8]) rc = sort_long_rows(ctx, list + first[8], cnt[8], off, nbr);
  clk.mark("sort: longer rows");
  cudaError_t e = cudaStreamSynchronize(st);  // before the list goes
  if (!rc && e != cudaSuccess) rc = cuda_error(e, "row sort");
  dev_free(cursor);
  dev_free(list);
  return rc;
}

namespace {
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
  StageClock clk{};
  clk.st = st;
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
      k_degree_keys<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, g->d_off, g->d_spatial, key,
                                                                id);
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
  clk.mark("order");
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
    clk.mark("inverse + relabeled offsets");
    k_relabel_rows<<<grid_for(ctx, 32ll * n, 256, 16), 256, 0, st>>>(n, perm, inv, g->d_off,
                                                                     g->d_nbr, roff, rnbr);
    ctx->launches++;
    clk.mark("relabeled rows");
    // rows ascending in solve ids: the select / pull scans run from a row's
    // end, i.e. (degree order) from the lowest-degree, highest-priority
    // neighbours, and with the class bounds they stop at the first entry
    // below the vertex's lower bound (select.cuh)
    if (!rc && g->nnz > 0) rc = sort_rows(ctx, n, roff, rnbr, 1);
  }
  clk.mark("row sort");
  int32_t *cls = nullptr;
  if (!rc && mode == TCMIS_ORDER_DEGREE) {
    thrust::counting_iterator<int32_t> ids(0);
    size_t bytes = 0;
    int64_t *d_cnt = nullptr;
    rc = dev_alloc(&d_cnt, 1);
    if (!rc) rc = dev_alloc(&cls, (size_t)n + 1);
    cub::DeviceSelect::If(nullptr, bytes, ids, cls, d_cnt, n, ClassHead{roff}, st);
    void *tmp = nullptr;
    if (!rc) rc = dev_alloc((char **)&tmp, bytes);
    if (!rc) {
      cub::DeviceSelect::If(tmp, bytes, ids, cls, d_cnt, n, ClassHead{roff}, st);
      ctx->launches++;
      int64_t cnt = 0;
      cudaMemcpyAsync(&cnt, d_cnt, 8, cudaMemcpyDeviceToHost, st);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = cuda_error(e, "degree classes");
      g->n_cls = (int32_t)cnt;
      if (!rc) {  // the end sentinel cls[n_cls] = n
        e = cudaMemcpyAsync(cls + cnt, &n, 4, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_error(e, "degree classes");
      }
    }
    dev_free(tmp);
    dev_free(d_cnt);
  }
  if (!rc) {
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
  // round 1's settling data (degree order, classes fit a u16)
  int32_t *rmax = nullptr, *cls_deg = nullptr;
  uint16_t *vcls = nullptr;
  if (!rc && mode == TCMIS_ORDER_DEGREE && g->n_cls > 0 && g->n_cls <= 65535) {
    int32_t *hub_end = nullptr;
    rc = dev_alloc(&rmax, (size_t)n);
    if (!rc) rc = dev_alloc(&vcls, (size_t)n);
    if (!rc) rc = dev_alloc(&hub_end, 1);
    if (!rc) rc = dev_alloc(&cls_deg, (size_t)g->n_cls);
    if (!rc) {
      // every row a hub (no sorted row to find): H = n
      cudaMemcpyAsync(hub_end, &n, 4, cudaMemcpyHostToDevice, st);
      k_row_max<<<grid_for(ctx, n, 256, 8), 256, 0, st>>>(n, roff, rnbr, rmax, hub_end);
      k_hub_max<<<ctx->num_sms * 4, 256, 0, st>>>(hub_end, roff, rnbr, rmax);
      k_vertex_class<<<grid_for(ctx, n, 256, 8), 256, 0, st>>>(n, g->n_cls, cls, vcls);
      k_class_degree<<<grid_for(ctx, g->n_cls, 256, 4), 256, 0, st>>>(g->n_cls, cls, roff, cls_deg);
      ctx->launches += 4;
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = cuda_error(e, "round-1 settling data");
    }
    dev_free(hub_end);
  }
  clk.mark("classes + non-isolated list");
  dev_free(bad);
  if (rc) {
    dev_free(cls_deg);
    dev_free(rmax);
    dev_free(vcls);
    dev_free(cls);
    g->n_cls = 0;
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
  g->d_cls_start = cls;
  g->d_rmax = rmax;
  g->d_cls_deg = cls_deg;
  g->d_vcls = vcls;
  g->order_mode = mode;
  return 0;
}

}  // namespace tcmis_b200
