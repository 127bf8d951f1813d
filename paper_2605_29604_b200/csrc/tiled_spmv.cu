// tiled_spmv.cu -- Phase 2 in the paper's tile form (K4b / K4c).
//
// Reference: tiled_spmv + tile_mma (spmv.cpp:12-59): for every block row, the
// T x T 0/1 tiles of that row are multiplied with the candidate segment of
// their block column, skipping tiles whose segment is all zero.  Two device
// kernels over a TiledAdjacency in the reference layout (tile_col[],
// row_bits[T per tile], block_row_offsets[]):
//
//  k_tiled_bits  CUDA cores: one warp per block row, lane i owns tile row i
//                (two rows per lane for T > 32); acc_i += popc(row_i & seg).
//                One coalesced T-word load per tile.
//  k_tiled_mma   tensor cores, T = 16: one warp per block row; every
//                non-skipped tile is one mma.sync.m16n8k16 s8 x s8 -> s32 with
//                the 16x16 bit tile expanded to s8 in registers as A and the
//                candidate segment as column 0 of B, accumulating over the
//                block row (the paper's Listing 1 WMMA, on
//                the native IMMA path; the b1 .and.popc form is emulated on
//                sm_100a).
//
// Both reproduce tile_mma exactly (integer arithmetic) and the reference's
// tiles_evaluated / tiles_skipped.  DESIGN.md "K4" records the measured
// comparison against the CSR forms of the engine.
#include <cuda_runtime.h>

#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

namespace {

__global__ void __launch_bounds__(256)
    k_tiled_bits(int32_t n, int T, int32_t nb, const int32_t *__restrict__ tile_col,
                 const uint64_t *__restrict__ row_bits, const int64_t *__restrict__ bro,
                 const uint64_t *__restrict__ seg, int32_t *__restrict__ nc,
                 unsigned long long *__restrict__ counters) {
  const int lane = threadIdx.x & 31;
  unsigned long long ev = 0, sk = 0;
  for (int64_t br = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; br < nb;
       br += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int acc0 = 0, acc1 = 0;
    for (int64_t t = bro[br]; t < bro[br + 1]; ++t) {
      const uint64_t sgm = seg[tile_col[t]];
      if (sgm == 0) {  // spmv.cpp:40-43
        ++sk;
        continue;
      }
      ++ev;
      if (lane < T) acc0 += __popcll(row_bits[t * T + lane] & sgm);
      if (lane + 32 < T) acc1 += __popcll(row_bits[t * T + lane + 32] & sgm);
    }
    const int64_t base = br * T;
    if (lane < T && base + lane < n) nc[base + lane] = acc0;
    if (lane + 32 < T && base + lane + 32 < n) nc[base + lane + 32] = acc1;
  }
  if (lane == 0) {  // every lane counted the same tiles
    atomicAdd(&counters[0], ev);
    atomicAdd(&counters[1], sk);
  }
}

// 4 bits -> 4 bytes of 0/1 (bit i -> byte i)
__device__ __forceinline__ uint32_t nib_to_s8(uint32_t x) {
  return (x & 1u) | ((x & 2u) << 7) | ((x & 4u) << 14) | ((x & 8u) << 21);
}

__global__ void __launch_bounds__(256)
    k_tiled_mma(int32_t n, int32_t nb, const int32_t *__restrict__ tile_col,
                const uint64_t *__restrict__ row_bits, const int64_t *__restrict__ bro,
                const uint64_t *__restrict__ seg, int32_t *__restrict__ nc,
                unsigned long long *__restrict__ counters) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 2, tig = lane & 3;
  unsigned long long ev = 0, sk = 0;
  for (int64_t br = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; br < nb;
       br += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int d0 = 0, d1 = 0, d2 = 0, d3 = 0;
    for (int64_t t = bro[br]; t < bro[br + 1]; ++t) {
      const uint64_t sgm = seg[tile_col[t]];
      if (sgm == 0) {
        ++sk;
        continue;
      }
      ++ev;
      // A fragment (row-major 16x16 s8): a0 = A[grp][tig*4 .. +3],
      // a1 = A[grp+8][tig*4 .. +3]
      const uint32_t r0 = (uint32_t)row_bits[t * 16 + grp];
      const uint32_t r1 = (uint32_t)row_bits[t * 16 + grp + 8];
      const uint32_t a0 = nib_to_s8((r0 >> (tig * 4)) & 0xFu);
      const uint32_t a1 = nib_to_s8((r1 >> (tig * 4)) & 0xFu);
      // B fragment (col-major 16x8 s8): b = B[tig*4 .. +3][grp]; the segment
      // is column 0
      const uint32_t b = grp == 0 ? nib_to_s8((uint32_t)(sgm >> (tig * 4)) & 0xFu) : 0u;
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.s32.s8.s8.s32 "
          "{%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};\n"
          : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3)
          : "r"(a0), "r"(a1), "r"(b));
    }
    // D[row][0]: row grp in d0 and row grp+8 in d2 of the lanes with tig == 0
    const int64_t base = br * 16;
    if (tig == 0) {
      if (base + grp < n) nc[base + grp] = d0;
      if (base + grp + 8 < n) nc[base + grp + 8] = d2;
    }
    (void)d1;
    (void)d3;
  }
  if (lane == 0) {
    atomicAdd(&counters[0], ev);
    atomicAdd(&counters[1], sk);
  }
}

template <typename T>
struct Dev {
  T *p = nullptr;
  ~Dev() { dev_free(p); }
};

}  // namespace

int tiled_spmv_tiles_impl(tcmis_ctx *ctx, int32_t n, int32_t T, int64_t tiles,
                          const int32_t *tile_col, const uint64_t *row_bits, const int64_t *bro,
                          const uint64_t *seg, int32_t exclusion, int32_t *nc, int64_t *ev,
                          int64_t *sk) {
  if (T < 1 || T > 64)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tile_dim must be in [1, 64], got " + std::to_string(T));
  if (exclusion == TCMIS_EXCL_TILE_MMA && T != 16)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "the tensor-core tile kernel needs tile_dim 16");
  const int32_t nb = (int32_t)(((int64_t)n + T - 1) / T);
  *ev = *sk = 0;
  if (n == 0) return 0;
  cudaStream_t st = ctx->stream;
  Dev<int32_t> d_col, d_nc;
  Dev<uint64_t> d_bits, d_seg;
  Dev<int64_t> d_bro;
  Dev<unsigned long long> d_cnt;
  if (int rc = dev_alloc(&d_col.p, (size_t)tiles)) return rc;
  if (int rc = dev_alloc(&d_bits.p, (size_t)tiles * T)) return rc;
  if (int rc = dev_alloc(&d_bro.p, (size_t)nb + 1)) return rc;
  if (int rc = dev_alloc(&d_seg.p, (size_t)nb)) return rc;
  if (int rc = dev_alloc(&d_nc.p, (size_t)n)) return rc;
  if (int rc = dev_alloc(&d_cnt.p, 2)) return rc;
  if (tiles) {
    TCMIS_CUDA(cudaMemcpyAsync(d_col.p, tile_col, 4ull * tiles, cudaMemcpyHostToDevice, st));
    TCMIS_CUDA(cudaMemcpyAsync(d_bits.p, row_bits, 8ull * tiles * T, cudaMemcpyHostToDevice, st));
  }
  TCMIS_CUDA(cudaMemcpyAsync(d_bro.p, bro, 8ull * (nb + 1), cudaMemcpyHostToDevice, st));
  TCMIS_CUDA(cudaMemcpyAsync(d_seg.p, seg, 8ull * nb, cudaMemcpyHostToDevice, st));
  TCMIS_CUDA(cudaMemsetAsync(d_cnt.p, 0, 16, st));
  const int grid = grid_for(ctx, 32ll * nb, 256, 8);
  if (exclusion == TCMIS_EXCL_TILE_MMA)
    k_tiled_mma<<<grid, 256, 0, st>>>(n, nb, d_col.p, d_bits.p, d_bro.p, d_seg.p, d_nc.p,
                                      d_cnt.p);
  else
    k_tiled_bits<<<grid, 256, 0, st>>>(n, T, nb, d_col.p, d_bits.p, d_bro.p, d_seg.p, d_nc.p,
                                       d_cnt.p);
  TCMIS_LAUNCHED(ctx);
  unsigned long long cnt[2] = {0, 0};
  TCMIS_CUDA(cudaMemcpyAsync(nc, d_nc.p, 4ull * n, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaMemcpyAsync(cnt, d_cnt.p, 16, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  *ev = (int64_t)cnt[0];
  *sk = (int64_t)cnt[1];
  return 0;
}

}  // namespace tcmis_b200
