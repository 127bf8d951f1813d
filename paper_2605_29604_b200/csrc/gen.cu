// gen.cu -- synthetic graphs for the BASELINE configs, built on the device.
//
// R-MAT (generate.cpp:68-98) is re-derived counter-based: SplitMix64 draw i
// of seed s is vertex_hash(i, s) (generate.cpp:15-26 + priorities.cpp:21-23),
// so sample e, level l uses draw e*scale + l and every sample is independent.
// Normalisation (graph.cpp:14-41: drop loops, add reverse edges, sort, dedupe)
// is a radix sort + unique over (u << scale | v) keys.  The result is bit-
// identical to tcmis::rmat_graph (pinned by tests/test_gpu_parity.py::test_gpu_rmat_bit_identical).
//
// Grid and RGG have no reference generator; their definitions are DESIGN.md's
// (and oracle/tcmis_oracle.c's).  G(n,p) consumes one draw per edge, so its
// stream is counter-form too: the pair-index increments are independent and a
// prefix sum places them (gen_gnp; tests/test_gpu_parity.py
// test_gpu_gnp_bit_identical).  The serial host form stays as tcmis_gen_gnp_host.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

int wrap_owned(tcmis_ctx *ctx, int32_t n, int64_t nnz, int64_t *d_off, int32_t *d_nbr,
               tcmis_graph **out);

namespace {

__global__ void k_rmat_keys(int scale, int64_t samples, uint64_t mseed,
                            unsigned long long *__restrict__ keys) {
  const uint64_t loop_key = (1ull << (2 * scale)) - 1;  // (n-1, n-1): never a real edge
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < samples;
       e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t u = 0, v = 0;
    const uint64_t first = (uint64_t)e * (uint64_t)scale;
    for (int l = 0; l < scale; ++l) {
      const double r = (double)(vertex_hash_m(first + l, mseed) >> 11) * 0x1.0p-53;
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
    if (u == v) {
      keys[2 * e] = loop_key;
      keys[2 * e + 1] = loop_key;
    } else {
      keys[2 * e] = ((uint64_t)u << scale) | v;
      keys[2 * e + 1] = ((uint64_t)v << scale) | u;
    }
  }
}

// sorted unique keys -> CSR (row starts found at the key where the row changes)
__global__ void k_keys_to_csr(int scale, int32_t n, int64_t m,
                              const unsigned long long *__restrict__ keys,
                              int64_t *__restrict__ off, int32_t *__restrict__ nbr) {
  const uint64_t mask = (1ull << scale) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i < m ? (int64_t)(keys[i] >> scale) : n;
    const int64_t prev = i > 0 ? (int64_t)(keys[i - 1] >> scale) : -1;
    for (int64_t r = prev + 1; r <= row; ++r) off[r] = i;
    if (i < m) nbr[i] = (int32_t)(keys[i] & mask);
  }
}

__global__ void k_grid_deg(int32_t side, int64_t *__restrict__ deg) {
  const int64_t n = (int64_t)side * side;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (v == n) {
      deg[v] = 0;
      continue;
    }
    const int32_t i = (int32_t)(v / side), j = (int32_t)(v % side);
    deg[v] = (i > 0) + (j > 0) + (j + 1 < side) + (i + 1 < side);
  }
}

__global__ void k_grid_fill(int32_t side, const int64_t *__restrict__ off,
                            int32_t *__restrict__ nbr) {
  const int64_t n = (int64_t)side * side;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t i = (int32_t)(v / side), j = (int32_t)(v % side);
    int64_t w = off[v];
    if (i > 0) nbr[w++] = (int32_t)(v - side);
    if (j > 0) nbr[w++] = (int32_t)(v - 1);
    if (j + 1 < side) nbr[w++] = (int32_t)(v + 1);
    if (i + 1 < side) nbr[w++] = (int32_t)(v + side);
  }
}

// ----------------------------------------------------------------- RGG

__global__ void k_rgg_points(int32_t n, uint64_t mseed, uint64_t R, uint64_t C,
                             uint32_t *__restrict__ x, uint32_t *__restrict__ y,
                             unsigned long long *__restrict__ cell, int32_t *__restrict__ ids) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t xv = (uint32_t)(vertex_hash_m(2ull * v, mseed) >> 32);
    const uint32_t yv = (uint32_t)(vertex_hash_m(2ull * v + 1, mseed) >> 32);
    x[v] = xv;
    y[v] = yv;
    cell[v] = (xv / R) * C + (yv / R);
    ids[v] = (int32_t)v;
  }
}

// Morton (Z-order) code of a point's grid cell: the RGG's spatial vertex
// order (order.cu, TCMIS_ORDER_SPATIAL)
__device__ __forceinline__ uint64_t spread2(uint64_t v) {
  v &= 0xffffffffull;
  v = (v | (v << 16)) & 0x0000ffff0000ffffull;
  v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
  v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__global__ void k_rgg_morton(int32_t n, uint64_t R, const uint32_t *__restrict__ x,
                             const uint32_t *__restrict__ y, unsigned long long *__restrict__ key,
                             int32_t *__restrict__ ids) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = (spread2(x[v] / R) << 1) | spread2(y[v] / R);
    ids[v] = (int32_t)v;
  }
}

__global__ void k_cell_starts(int64_t ncell, int32_t n, const unsigned long long *__restrict__ cell,
                              int64_t *__restrict__ cs) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i < n ? (int64_t)cell[i] : ncell;
    const int64_t prev = i > 0 ? (int64_t)cell[i - 1] : -1;
    for (int64_t k = prev + 1; k <= c; ++k) cs[k] = i;
  }
}

template <bool fill>
__global__ void k_rgg_rows(int32_t n, uint64_t R, uint64_t C, const uint32_t *__restrict__ x,
                           const uint32_t *__restrict__ y, const int64_t *__restrict__ cs,
                           const int32_t *__restrict__ pts, int64_t *__restrict__ deg,
                           const int64_t *__restrict__ off, int32_t *__restrict__ nbr) {
  const uint64_t R2 = R * R;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t xv = x[v], yv = y[v];
    const int64_t cx = xv / R, cy = yv / R;
    int64_t w = fill ? off[v] : 0;
    const int64_t start = w;
    for (int64_t ax = cx - 1; ax <= cx + 1; ++ax) {
      if (ax < 0 || ax >= (int64_t)C) continue;
      for (int64_t ay = cy - 1; ay <= cy + 1; ++ay) {
        if (ay < 0 || ay >= (int64_t)C) continue;
        const int64_t c = ax * (int64_t)C + ay;
        for (int64_t q = cs[c]; q < cs[c + 1]; ++q) {
          const int32_t u = pts[q];
          if (u == v) continue;
          const uint64_t dx = x[u] > xv ? x[u] - xv : xv - x[u];
          const uint64_t dy = y[u] > yv ? y[u] - yv : yv - y[u];
          if (dx > R || dy > R) continue;
          if (dx * dx + dy * dy <= R2) {
            if (fill) nbr[w] = u;
            ++w;
          }
        }
      }
    }
    if (!fill) {
      deg[v] = w;
    } else {  // rows are short (mean ~3): insertion sort in place
      for (int64_t a = start + 1; a < w; ++a) {
        const int32_t t = nbr[a];
        int64_t b = a - 1;
        while (b >= start && nbr[b] > t) {
          nbr[b + 1] = nbr[b];
          --b;
        }
        nbr[b + 1] = t;
      }
    }
  }
}

template <typename T>
struct DevBuf {
  T *p = nullptr;
  ~DevBuf() { dev_free(p); }
  int alloc(size_t n) { return dev_alloc(&p, n); }
  T *release() {
    T *q = p;
    p = nullptr;
    return q;
  }
};

int exclusive_scan_i64(tcmis_ctx *ctx, int64_t *d, int64_t count) {
  size_t bytes = 0;
  TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, d, d, count, ctx->stream));
  DevBuf<char> tmp;
  if (int rc = tmp.alloc(bytes)) return rc;
  TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, d, d, count, ctx->stream));
  ctx->launches++;
  return 0;
}

}  // namespace

int gen_rmat(tcmis_ctx *ctx, int32_t scale, int32_t ef, uint64_t seed, tcmis_graph **out) {
  if (scale < 1 || scale > 30)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "rmat scale must be in [1, 30]");
  if (ef < 1) return set_error(TCMIS_E_INVALID_ARGUMENT, "edge_factor must be >= 1");
  cudaStream_t st = ctx->stream;
  const int32_t n = (int32_t)(1u << scale);
  const int64_t samples = (int64_t)ef * n;
  const int64_t nk = 2 * samples;
  DevBuf<unsigned long long> a, b;
  if (int rc = a.alloc((size_t)nk)) return rc;
  if (int rc = b.alloc((size_t)nk)) return rc;
  k_rmat_keys<<<grid_for(ctx, samples, 256, 16), 256, 0, st>>>(scale, samples, mix64(seed), a.p);
  TCMIS_LAUNCHED(ctx);
  {
    size_t bytes = 0;
    TCMIS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, a.p, b.p, nk, 0, 2 * scale, st));
    DevBuf<char> tmp;
    if (int rc = tmp.alloc(bytes)) return rc;
    TCMIS_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, a.p, b.p, nk, 0, 2 * scale, st));
    ctx->launches++;
  }
  DevBuf<int64_t> d_m;
  if (int rc = d_m.alloc(1)) return rc;
  {
    size_t bytes = 0;
    TCMIS_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, b.p, a.p, d_m.p, nk, st));
    DevBuf<char> tmp;
    if (int rc = tmp.alloc(bytes)) return rc;
    TCMIS_CUDA(cub::DeviceSelect::Unique(tmp.p, bytes, b.p, a.p, d_m.p, nk, st));
    ctx->launches++;
  }
  int64_t m = 0;
  TCMIS_CUDA(cudaMemcpyAsync(&m, d_m.p, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  // drop the loop sentinel (the largest possible key) if present
  if (m > 0) {
    unsigned long long last = 0;
    TCMIS_CUDA(cudaMemcpy(&last, a.p + (m - 1), 8, cudaMemcpyDeviceToHost));
    if (last == (1ull << (2 * scale)) - 1) --m;
  }
  DevBuf<int64_t> off;
  DevBuf<int32_t> nbr;
  if (int rc = off.alloc((size_t)n + 1)) return rc;
  if (int rc = nbr.alloc((size_t)m)) return rc;
  k_keys_to_csr<<<grid_for(ctx, m + 1, 256, 16), 256, 0, st>>>(scale, n, m, a.p, off.p, nbr.p);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaStreamSynchronize(st));
  int64_t *o = off.release();
  int32_t *q = nbr.release();
  return wrap_owned(ctx, n, m, o, q, out);
}

namespace {

// graph.cpp:14-41 graph_from_edges, step 1: both directions of every edge as
// a (u << bits | v) key; self-loops become the sentinel (all ones), which
// sorts last and is dropped after the unique pass
__global__ void k_edge_keys(int bits, int32_t n, int64_t m, const int32_t *__restrict__ eu,
                            const int32_t *__restrict__ ev,
                            unsigned long long *__restrict__ keys, int *__restrict__ bad) {
  const unsigned long long sentinel = (bits >= 32) ? ~0ull : ((1ull << (2 * bits)) - 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = eu[e], v = ev[e];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      atomicExch(bad, 1);
      keys[2 * e] = keys[2 * e + 1] = sentinel;
    } else if (u == v) {
      keys[2 * e] = keys[2 * e + 1] = sentinel;
    } else {
      keys[2 * e] = ((unsigned long long)u << bits) | (unsigned)v;
      keys[2 * e + 1] = ((unsigned long long)v << bits) | (unsigned)u;
    }
  }
}

}  // namespace

// graph_from_edges (graph.cpp:14-41: symmetrise, drop
// self-loops, dedup, CSR with sorted rows) on the device -- radix sort +
// unique over 2*ceil(log2 n)-bit keys, the same pipeline as the R-MAT
// generator.  An endpoint outside [0, n) -> std::out_of_range (graph.cpp:23-24).
// (d_u / d_v non-null: the edges are already on the device, h_u / h_v unused)
static int from_edges_impl(tcmis_ctx *ctx, int32_t n, int64_t m, const int32_t *h_u,
                           const int32_t *h_v, tcmis_graph **out, const int32_t *d_u,
                           const int32_t *d_v) {
  if (n < 0 || m < 0) return set_error(TCMIS_E_INVALID_ARGUMENT, "negative size");
  cudaStream_t st = ctx->stream;
  int bits = 1;
  while (bits < 31 && (1ll << bits) < (int64_t)n) ++bits;
  const int64_t nk = 2 * m;
  DevBuf<int32_t> du, dv;
  DevBuf<unsigned long long> a, b;
  DevBuf<int> bad;
  if (!d_u) {
    if (int rc = du.alloc((size_t)m)) return rc;
    if (int rc = dv.alloc((size_t)m)) return rc;
  }
  if (int rc = a.alloc((size_t)nk)) return rc;
  if (int rc = b.alloc((size_t)nk)) return rc;
  if (int rc = bad.alloc(1)) return rc;
  TCMIS_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  if (m) {
    if (!d_u) {
      TCMIS_CUDA(cudaMemcpyAsync(du.p, h_u, 4ull * m, cudaMemcpyHostToDevice, st));
      TCMIS_CUDA(cudaMemcpyAsync(dv.p, h_v, 4ull * m, cudaMemcpyHostToDevice, st));
    }
    k_edge_keys<<<grid_for(ctx, m, 256, 16), 256, 0, st>>>(bits, n, m, d_u ? d_u : du.p,
                                                         d_v ? d_v : dv.p, a.p, bad.p);
    TCMIS_LAUNCHED(ctx);
  }
  int h_bad = 0;
  TCMIS_CUDA(cudaMemcpyAsync(&h_bad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (h_bad) return set_error(TCMIS_E_OUT_OF_RANGE, "edge endpoint outside [0, n)");
  int64_t mm = 0;
  if (nk) {
    size_t bytes = 0;
    TCMIS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, a.p, b.p, nk, 0, 2 * bits, st));
    DevBuf<char> tmp;
    if (int rc = tmp.alloc(bytes)) return rc;
    TCMIS_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, a.p, b.p, nk, 0, 2 * bits, st));
    DevBuf<int64_t> d_m;
    if (int rc = d_m.alloc(1)) return rc;
    size_t ub = 0;
    TCMIS_CUDA(cub::DeviceSelect::Unique(nullptr, ub, b.p, a.p, d_m.p, nk, st));
    DevBuf<char> tmp2;
    if (int rc = tmp2.alloc(ub)) return rc;
    TCMIS_CUDA(cub::DeviceSelect::Unique(tmp2.p, ub, b.p, a.p, d_m.p, nk, st));
    ctx->launches += 2;
    TCMIS_CUDA(cudaMemcpyAsync(&mm, d_m.p, 8, cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    if (mm > 0) {
      unsigned long long last = 0;
      TCMIS_CUDA(cudaMemcpy(&last, a.p + (mm - 1), 8, cudaMemcpyDeviceToHost));
      const unsigned long long sentinel = (1ull << (2 * bits)) - 1;
      if (last == sentinel) --mm;
    }
  }
  DevBuf<int64_t> off;
  DevBuf<int32_t> nbr;
  if (int rc = off.alloc((size_t)n + 1)) return rc;
  if (int rc = nbr.alloc((size_t)mm)) return rc;
  k_keys_to_csr<<<grid_for(ctx, mm + 1, 256, 16), 256, 0, st>>>(bits, n, mm, a.p, off.p, nbr.p);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaStreamSynchronize(st));
  int64_t *o = off.release();
  int32_t *q = nbr.release();
  return wrap_owned(ctx, n, mm, o, q, out);
}

int gen_from_edges(tcmis_ctx *ctx, int32_t n, int64_t m, const int32_t *h_u, const int32_t *h_v,
                   tcmis_graph **out) {
  return from_edges_impl(ctx, n, m, h_u, h_v, out, nullptr, nullptr);
}

int gen_gnp_host(int32_t n, double avg_degree, uint64_t seed, int64_t **offsets,
                 int32_t **neighbors, int64_t *nnz_out);

int gen_grid(tcmis_ctx *ctx, int32_t side, tcmis_graph **out) {
  if (side < 0 || (int64_t)side * side > 0x7fffffffLL)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "grid side out of range");
  cudaStream_t st = ctx->stream;
  const int64_t n = (int64_t)side * side;
  const int64_t m = side > 1 ? 4ll * side * (side - 1) : 0;
  DevBuf<int64_t> off;
  DevBuf<int32_t> nbr;
  if (int rc = off.alloc((size_t)n + 1)) return rc;
  if (int rc = nbr.alloc((size_t)m)) return rc;
  k_grid_deg<<<grid_for(ctx, n + 1, 256, 16), 256, 0, st>>>(side, off.p);
  TCMIS_LAUNCHED(ctx);
  if (int rc = exclusive_scan_i64(ctx, off.p, n + 1)) return rc;
  k_grid_fill<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(side, off.p, nbr.p);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaStreamSynchronize(st));
  int64_t *o = off.release();
  int32_t *q = nbr.release();
  return wrap_owned(ctx, (int32_t)n, m, o, q, out);
}

int gen_rgg(tcmis_ctx *ctx, int32_t n, uint64_t R, uint64_t seed, tcmis_graph **out) {
  if (n < 0) return set_error(TCMIS_E_INVALID_ARGUMENT, "n must be non-negative");
  cudaStream_t st = ctx->stream;
  if (n == 0 || R == 0) {  // edgeless
    DevBuf<int64_t> off;
    if (int rc = off.alloc((size_t)n + 1)) return rc;
    TCMIS_CUDA(cudaMemsetAsync(off.p, 0, 8ull * (n + 1), st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    int32_t *q = nullptr;
    if (int rc = dev_alloc(&q, 1)) return rc;
    int64_t *o = off.release();
    return wrap_owned(ctx, n, 0, o, q, out);
  }
  const uint64_t C = 4294967295ull / R + 1;
  const uint64_t ncell = C * C;
  int cell_bits = 1;
  while (cell_bits < 64 && (1ull << cell_bits) <= ncell) ++cell_bits;
  DevBuf<uint32_t> x, y;
  DevBuf<unsigned long long> cell, cell2;
  DevBuf<int32_t> ids, pts;
  if (int rc = x.alloc(n)) return rc;
  if (int rc = y.alloc(n)) return rc;
  if (int rc = cell.alloc(n)) return rc;
  if (int rc = cell2.alloc(n)) return rc;
  if (int rc = ids.alloc(n)) return rc;
  if (int rc = pts.alloc(n)) return rc;
  k_rgg_points<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, mix64(seed), R, C, x.p, y.p, cell.p,
                                                           ids.p);
  TCMIS_LAUNCHED(ctx);
  {
    size_t bytes = 0;
    TCMIS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, cell.p, cell2.p, ids.p, pts.p,
                                               (int64_t)n, 0, cell_bits, st));
    DevBuf<char> tmp;
    if (int rc = tmp.alloc(bytes)) return rc;
    TCMIS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, cell.p, cell2.p, ids.p, pts.p,
                                               (int64_t)n, 0, cell_bits, st));
    ctx->launches++;
  }
  DevBuf<int64_t> cs;
  if (int rc = cs.alloc(ncell + 1)) return rc;
  k_cell_starts<<<grid_for(ctx, n + 1, 256, 16), 256, 0, st>>>((int64_t)ncell, n, cell2.p, cs.p);
  TCMIS_LAUNCHED(ctx);
  DevBuf<int64_t> off;
  if (int rc = off.alloc((size_t)n + 1)) return rc;
  TCMIS_CUDA(cudaMemsetAsync(off.p + n, 0, 8, st));
  k_rgg_rows<false><<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, R, C, x.p, y.p, cs.p, pts.p,
                                                               off.p, nullptr, nullptr);
  TCMIS_LAUNCHED(ctx);
  if (int rc = exclusive_scan_i64(ctx, off.p, (int64_t)n + 1)) return rc;
  int64_t m = 0;
  TCMIS_CUDA(cudaMemcpyAsync(&m, off.p + n, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  DevBuf<int32_t> nbr;
  if (int rc = nbr.alloc((size_t)m)) return rc;
  k_rgg_rows<true><<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, R, C, x.p, y.p, cs.p, pts.p,
                                                              nullptr, off.p, nbr.p);
  TCMIS_LAUNCHED(ctx);
  // the points in Z-order of their cells: the graph's spatial vertex order
  // (kept on the graph for tcmis_graph_reorder(TCMIS_ORDER_SPATIAL))
  DevBuf<int32_t> spatial;
  if (int rc = spatial.alloc(n)) return rc;
  {
    k_rgg_morton<<<grid_for(ctx, n, 256, 16), 256, 0, st>>>(n, R, x.p, y.p, cell.p, ids.p);
    TCMIS_LAUNCHED(ctx);
    int bits = 2;
    while (bits < 64 && (1ull << (bits / 2)) < C) bits += 2;
    size_t bytes = 0;
    TCMIS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, cell.p, cell2.p, ids.p, spatial.p,
                                               (int64_t)n, 0, bits, st));
    DevBuf<char> tmp;
    if (int rc = tmp.alloc(bytes)) return rc;
    TCMIS_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, cell.p, cell2.p, ids.p, spatial.p,
                                               (int64_t)n, 0, bits, st));
    ctx->launches++;
  }
  TCMIS_CUDA(cudaStreamSynchronize(st));
  int64_t *o = off.release();
  int32_t *q = nbr.release();
  if (int rc = wrap_owned(ctx, n, m, o, q, out)) return rc;
  (*out)->d_spatial = spatial.release();
  return 0;
}

// generate.cpp:30-66 on the host: the gap sequence is one serial RNG stream.
namespace {

// gnp_graph (generate.cpp:30-60) draw by draw: draw k of the SplitMix64 stream
// is mix64(mix64(seed) + (k + 1) golden) (counter form, as in the R-MAT
// kernel), and the pair index advances by 1 + floor(log1p(-u) / log1p(-p)),
// so the increments are independent and the pair indices are their prefix
// sum.  The increment is clamped to total + 1 (one such step already ends the
// stream), which keeps the sums in range for any p.
__global__ void k_gnp_steps(int64_t K, uint64_t mseed, double log_q, int64_t total,
                            int64_t *__restrict__ inc) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(vertex_hash_m((uint64_t)k, mseed) >> 11) * 0x1.0p-53;
    const double g = floor(log1p(-u) / log_q);
    inc[k] = g >= (double)total ? total + 1 : 1 + (int64_t)g;
  }
}

// first pair index of row r: pairs (i, j), i < j, in row-major order
__device__ __forceinline__ int64_t gnp_row_start(int64_t n, int64_t r) {
  return (int64_t)(((uint64_t)r * (uint64_t)(2 * n - r - 1)) >> 1);
}

// pair index -> (row, column), generate.cpp:50-57 (the while loop over rows)
// in closed form: a floating-point estimate of the row, corrected exactly
__global__ void k_gnp_pairs(int64_t E, int64_t n, const int64_t *__restrict__ idx1,
                            int32_t *__restrict__ eu, int32_t *__restrict__ ev) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < E;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t idx = idx1[k] - 1;  // the prefix sum starts the stream at -1
    const double b = (double)(2 * n - 1);
    int64_t r = (int64_t)floor((b - sqrt(b * b - 8.0 * (double)idx)) * 0.5);
    r = r < 0 ? 0 : (r > n - 2 ? n - 2 : r);
    while (r > 0 && gnp_row_start(n, r) > idx) --r;
    while (r < n - 2 && gnp_row_start(n, r + 1) <= idx) ++r;
    eu[k] = (int32_t)r;
    ev[k] = (int32_t)(r + 1 + (idx - gnp_row_start(n, r)));
  }
}

__global__ void k_count_below(int64_t K, const int64_t *__restrict__ idx1, int64_t total,
                              unsigned long long *__restrict__ cnt) {
  unsigned long long c = 0;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < K;
       k += (int64_t)gridDim.x * blockDim.x)
    c += idx1[k] - 1 < total ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, (unsigned)c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

}  // namespace

// gnp_graph_avg_degree (generate.cpp:62-65) on the device:
// bit-identical to the reference's serial stream (tests/test_gpu_parity.py).
// p >= 1 (the complete graph, a corner only tiny n reaches) is built on the
// host and uploaded.
int gen_gnp(tcmis_ctx *ctx, int32_t n, double avg_degree, uint64_t seed, tcmis_graph **out) {
  if (n < 0) return set_error(TCMIS_E_INVALID_ARGUMENT, "n must be non-negative");
  const double p = n > 1 ? avg_degree / (double)(n - 1) : 0.0;
  if (p <= 0.0 || n < 2) return gen_from_edges(ctx, n, 0, nullptr, nullptr, out);
  if (p >= 1.0) {
    int64_t *off = nullptr;
    int32_t *nbr = nullptr;
    int64_t nnz = 0;
    if (int rc = gen_gnp_host(n, avg_degree, seed, &off, &nbr, &nnz)) return rc;
    std::vector<int32_t> eu, ev;
    for (int32_t v = 0; v < n; ++v)
      for (int64_t e = off[v]; e < off[v + 1]; ++e)
        if (v < nbr[e]) {
          eu.push_back(v);
          ev.push_back(nbr[e]);
        }
    std::free(off);
    std::free(nbr);
    return gen_from_edges(ctx, n, (int64_t)eu.size(), eu.data(), ev.data(), out);
  }
  cudaStream_t st = ctx->stream;
  const double log_q = std::log1p(-p);  // the host's log1p, as the reference's
  const int64_t total = (int64_t)n * (n - 1) / 2;
  const double mean = p * (double)total;
  // draws: the expected edge count plus 8 standard deviations; more if that
  // did not reach the end of the pair range
  int64_t K = (int64_t)(mean + 8.0 * std::sqrt(mean) + 1024.0);
  const uint64_t mseed = mix64(seed);
  for (;;) {
    DevBuf<int64_t> inc, idx1;
    DevBuf<unsigned long long> cnt;
    if (int rc = inc.alloc((size_t)K)) return rc;
    if (int rc = idx1.alloc((size_t)K)) return rc;
    if (int rc = cnt.alloc(1)) return rc;
    k_gnp_steps<<<grid_for(ctx, K, 256, 16), 256, 0, st>>>(K, mseed, log_q, total, inc.p);
    TCMIS_LAUNCHED(ctx);
    size_t bytes = 0;
    TCMIS_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, inc.p, idx1.p, K, st));
    DevBuf<char> tmp;
    if (int rc = tmp.alloc(bytes)) return rc;
    TCMIS_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, inc.p, idx1.p, K, st));
    ctx->launches += 1;
    TCMIS_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
    k_count_below<<<grid_for(ctx, K, 256, 16), 256, 0, st>>>(K, idx1.p, total, cnt.p);
    TCMIS_LAUNCHED(ctx);
    unsigned long long E = 0;
    TCMIS_CUDA(cudaMemcpyAsync(&E, cnt.p, sizeof(E), cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    if ((int64_t)E == K) {  // the stream did not end within K draws
      K *= 2;
      continue;
    }
    DevBuf<int32_t> eu, ev;
    if (int rc = eu.alloc((size_t)E + 1)) return rc;
    if (int rc = ev.alloc((size_t)E + 1)) return rc;
    if (E)
      k_gnp_pairs<<<grid_for(ctx, (int64_t)E, 256, 16), 256, 0, st>>>((int64_t)E, n, idx1.p,
                                                                     eu.p, ev.p);
    TCMIS_LAUNCHED(ctx);
    return from_edges_impl(ctx, n, (int64_t)E, nullptr, nullptr, out, eu.p, ev.p);
  }
}

int gen_gnp_host(int32_t n, double avg_degree, uint64_t seed, int64_t **offsets,
                 int32_t **neighbors, int64_t *nnz_out) {
  if (n < 0) return set_error(TCMIS_E_INVALID_ARGUMENT, "n must be non-negative");
  const double p = n > 1 ? avg_degree / (double)(n - 1) : 0.0;
  std::vector<uint64_t> keys;  // directed (u << 32 | v)
  if (!(p <= 0.0 || n < 2)) {
    if (p >= 1.0) {
      for (int32_t u = 0; u < n; ++u)
        for (int32_t v = u + 1; v < n; ++v) {
          keys.push_back(((uint64_t)u << 32) | (uint32_t)v);
          keys.push_back(((uint64_t)v << 32) | (uint32_t)u);
        }
    } else {
      uint64_t state = mix64(seed);
      const double log_q = std::log1p(-p);
      const int64_t total = (int64_t)n * (n - 1) / 2;
      int64_t idx = -1, row = 0, row_start = 0, row_len = n - 1;
      for (;;) {
        state += kGolden;
        const double u = (double)(mix64(state) >> 11) * 0x1.0p-53;
        const int64_t gap = (int64_t)std::floor(std::log1p(-u) / log_q);
        idx += 1 + gap;
        if (idx >= total) break;
        while (idx - row_start >= row_len) {
          row_start += row_len;
          ++row;
          --row_len;
        }
        const uint32_t a = (uint32_t)row, b = (uint32_t)(row + 1 + (idx - row_start));
        keys.push_back(((uint64_t)a << 32) | b);
        keys.push_back(((uint64_t)b << 32) | a);
      }
    }
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  int64_t *off = (int64_t *)std::calloc((size_t)n + 1, sizeof(int64_t));
  int32_t *nbr = (int32_t *)std::malloc(sizeof(int32_t) * (keys.size() + 1));
  if (!off || !nbr) {
    std::free(off);
    std::free(nbr);
    return set_error(TCMIS_E_RUNTIME, "out of host memory");
  }
  for (size_t i = 0; i < keys.size(); ++i) {
    off[(keys[i] >> 32) + 1]++;
    nbr[i] = (int32_t)(uint32_t)keys[i];
  }
  for (int32_t v = 0; v < n; ++v) off[v + 1] += off[v];
  *offsets = off;
  *neighbors = nbr;
  *nnz_out = (int64_t)keys.size();
  return 0;
}

}  // namespace tcmis_b200
