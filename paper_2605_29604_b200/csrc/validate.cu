// validate.cu -- SURVEY 8(f2): the reference's result checks on the device.
//
// check_independence / check_maximality (validate.cpp:45-75) are O(n + m)
// serial scans on the host in the reference; every bench solve can afford
// them here.  One kernel answers both, with the reference's witnesses:
//   * independence: the smallest v in the set with a neighbour in the set;
//     its first such neighbour u in row order (rows are sorted; u > v, else
//     u would be a smaller violating vertex) -> (min, max) = (v, u);
//   * maximality: the smallest v outside the set with no neighbour in it.
// A warp scans a row (early exit), packs (v, u) into one 64-bit key and
// atomicMin's it, so the minimum over v is exact whatever the schedule.
#include <cuda_runtime.h>

#include <climits>

#include "internal.cuh"

namespace tcmis_b200 {

namespace {

__global__ void k_membership(const int32_t *__restrict__ set, int64_t cnt, int32_t n,
                             uint8_t *__restrict__ in, int *__restrict__ bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = set[i];
    if (v < 0 || v >= n) atomicExch(bad, 1);  // membership(), validate.cpp:12-22
    else in[v] = 1;
  }
}

__global__ void k_check_set(int32_t n, const int64_t *__restrict__ off,
                            const int32_t *__restrict__ nbr, const uint8_t *__restrict__ in,
                            unsigned long long *__restrict__ viol,
                            unsigned long long *__restrict__ addable) {
  const int lane = threadIdx.x & 31;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const bool member = in[v] != 0;
    const int64_t s = off[v], e = off[v + 1];
    // first neighbour in the set, in row order
    long long first = LLONG_MAX;
    for (int64_t base = s; base < e && first == LLONG_MAX; base += 128) {
      bool hit[4];
      int64_t idx[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        idx[j] = base + lane + 32 * j;
        hit[j] = idx[j] < e && in[__ldg(&nbr[idx[j]])];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned m = __ballot_sync(0xffffffffu, hit[j]);
        if (m && first == LLONG_MAX) first = base + 32 * j + (__ffs(m) - 1);
      }
    }
    if (lane == 0) {
      if (member && first != LLONG_MAX) {
        const uint32_t u = (uint32_t)__ldg(&nbr[first]);
        atomicMin(viol, ((unsigned long long)v << 32) | u);
      } else if (!member && first == LLONG_MAX) {
        atomicMin(addable, (unsigned long long)v);
      }
    }
  }
}

}  // namespace

int validate_impl(tcmis_graph *g, const int32_t *set, int64_t cnt, int32_t *independent,
                  int32_t *wu, int32_t *wv, int32_t *maximal, int32_t *addable) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int32_t n = g->n;
  uint8_t *in = nullptr;
  int32_t *d_set = nullptr;
  unsigned long long *d_res = nullptr;  // [0] violation key, [1] addable, [2] bad id
  if (int rc = dev_alloc(&in, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_set, (size_t)cnt + 1)) return rc;
  if (int rc = dev_alloc(&d_res, 3)) return rc;
  unsigned long long h[3] = {ULLONG_MAX, ULLONG_MAX, 0};
  int rc = 0;
  cudaError_t e = cudaMemsetAsync(in, 0, (size_t)n + 1, st);
  if (e == cudaSuccess && cnt)
    e = cudaMemcpyAsync(d_set, set, 4ull * cnt, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_res, h, sizeof(h), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && cnt) {
    k_membership<<<grid_for(ctx, cnt, 256, 8), 256, 0, st>>>(
        d_set, cnt, n, in, reinterpret_cast<int *>(d_res + 2));
    ctx->launches++;
  }
  if (e == cudaSuccess && n) {
    k_check_set<<<grid_for(ctx, 32ll * n, 256, 8), 256, 0, st>>>(n, g->d_off, g->d_nbr, in,
                                                                  d_res, d_res + 1);
    ctx->launches++;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d_res, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  dev_free(in);
  dev_free(d_set);
  dev_free(d_res);
  if (e != cudaSuccess) return cuda_error(e, "validate");
  if ((int)h[2]) return set_error(TCMIS_E_INVALID_ARGUMENT, "set contains a vertex id outside [0, n)");
  *independent = h[0] == ULLONG_MAX ? 1 : 0;
  if (!*independent) {
    *wu = (int32_t)(h[0] >> 32);
    *wv = (int32_t)(h[0] & 0xffffffffu);
  }
  *maximal = h[1] == ULLONG_MAX ? 1 : 0;
  if (!*maximal) *addable = (int32_t)h[1];
  return rc;
}

}  // namespace tcmis_b200
