// tile_umma.cuh -- the tile x bit-vector product of Phase 1 (A-up tiles x the
// alive bitmap, tile_cand.cu) on the 5th-generation tensor cores: tcgen05.mma
// kind::i8 with the accumulator in TMEM (TCMIS_F_TILE_UMMA).  The keep/drop
// experiment the north star asks for ("tile x status-vector products on
// tensor cores ... tcgen05 where tile density justifies it ... kept only if it
// beats the CUDA-core variant"); profiles/r02/phase1_tiles.md has the numbers.
//
// One MMA per 8 tiles: M = 128 rows = 8 tiles x 16 rows (A, K-major, the
// tile rows' bits expanded to 0/1 bytes in shared memory, K = 32 with the
// upper 16 columns zero), N = 16 columns of which column j holds tile j's
// alive segment (B, K-major, 0/1 bytes), D = A.B in TMEM as s32: row 16j + i,
// column j is "row i of tile j has an alive higher-key neighbour".  Only the
// 8 diagonal 16x1 blocks of the 128x16 product are used (1/16 of the MACs,
// and half of K is padding): a single bit-vector per tile leaves the tensor
// core nothing to reuse, which is the point the measurement makes.
//
// Per batch: all 128 threads expand their tile row into shared memory,
// fence.proxy.async, one elected thread issues tcgen05.mma and tcgen05.commit
// to an mbarrier, every warp waits on it (bounded: a trap instead of a hang)
// and reads its 32 TMEM lanes with tcgen05.ld.32x32b.x16.
#pragma once

#include "common.cuh"

namespace tcmis_b200 {

struct UmmaArgs {
  int64_t tiles;
  const int32_t *trow;
  const int32_t *tcol;
  const uint16_t *tbits;
  const uint32_t *xbits;  // the vector, bit per vertex
  uint32_t *hit;          // out: per block row, rows with a non-zero product
  const Ctrl *gate_ctrl;  // run only in a tile round (alive >= gate)
  int32_t gate;
};

__device__ __forceinline__ uint32_t umma_nib(uint32_t x) {  // 4 bits -> 4 bytes of 0/1
  x &= 0xfu;
  return (x & 1u) | ((x & 2u) << 7) | ((x & 4u) << 14) | ((x & 8u) << 21);
}
__device__ __forceinline__ uint4 umma_expand16(uint32_t b) {
  return make_uint4(umma_nib(b), umma_nib(b >> 4), umma_nib(b >> 8), umma_nib(b >> 12));
}

// shared-memory matrix descriptor, K-major, no swizzle (canonical layout
// ((8,m),(16B,2)) : ((16B,SBO),(1,LBO)), cute/atom/mma_traits_sm100.hpp)
__device__ __forceinline__ uint64_t umma_smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((lbo >> 4) & 0x3fffu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);  // version 1 (sm_100), layout 0
}

constexpr int kUmmaM = 128, kUmmaN = 16, kUmmaTiles = 8;
// instruction descriptor (cute::UMMA::InstrDescriptor): D s32, A / B unsigned
// 8-bit, both K-major, N >> 3, M >> 4
constexpr uint32_t kUmmaIdesc = (2u << 4) | ((uint32_t)(kUmmaN >> 3) << 17) |
                                ((uint32_t)(kUmmaM >> 4) << 24);

__global__ void __launch_bounds__(128) k_tile_umma(UmmaArgs a) {
  if (a.gate_ctrl && a.gate_ctrl->alive < a.gate) return;
  __shared__ __align__(1024) uint8_t sA[kUmmaM * 32];  // 16 row blocks x (2 K blocks of 128 B)
  __shared__ __align__(128) uint8_t sB[kUmmaN * 32];   // 2 N blocks x (2 K blocks of 128 B)
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t s_tmem;
  __shared__ int32_t s_row[kUmmaTiles];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (int)sizeof(sA) / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(sA)[i] = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < (int)sizeof(sB) / 16; i += blockDim.x)
    reinterpret_cast<uint4 *>(sB)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t mbar_addr = (uint32_t)__cvta_generic_to_shared(&mbar);
  if (warp == 0) {
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tmem);
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(dst));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar_addr));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  const uint64_t adesc = umma_smem_desc((uint32_t)__cvta_generic_to_shared(sA), 128, 256);
  const uint64_t bdesc = umma_smem_desc((uint32_t)__cvta_generic_to_shared(sB), 128, 256);
  uint32_t phase = 0;
  const uint4 *__restrict__ pay = reinterpret_cast<const uint4 *>(a.tbits);
  for (int64_t base = (int64_t)blockIdx.x * kUmmaTiles; base < a.tiles;
       base += (int64_t)gridDim.x * kUmmaTiles) {
    // A: thread m = row (m & 15) of tile (m >> 4); its 16 bits -> 16 bytes
    {
      const int64_t t = base + (tid >> 4);
      uint32_t bits = 0;
      if (t < a.tiles) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t *>(pay + 2 * t) + ((tid & 15) >> 1));
        bits = (w >> (16 * (tid & 1))) & 0xffffu;
      }
      *reinterpret_cast<uint4 *>(sA + (tid >> 3) * 256 + (tid & 7) * 16) = umma_expand16(bits);
    }
    // B: threads 0-7 = column j: tile j's alive segment
    if (tid < kUmmaTiles) {
      const int64_t t = base + tid;
      uint32_t seg = 0;
      int32_t row = -1;
      if (t < a.tiles) {
        const int32_t c = __ldg(&a.tcol[t]);
        seg = (__ldg(&a.xbits[c >> 1]) >> ((c & 1) * 16)) & 0xffffu;
        row = __ldg(&a.trow[t]);
      }
      *reinterpret_cast<uint4 *>(sB + tid * 16) = umma_expand16(seg);
      s_row[tid] = row;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.u32 p, 0, 0;\n"
          " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
          "l"(adesc), "l"(bdesc), "r"(kUmmaIdesc));
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              mbar_addr));
    }
    // wait for the MMA (bounded: a broken descriptor traps instead of hanging)
    {
      uint32_t done = 0;
      for (int64_t spin = 0; !done; ++spin) {
        asm volatile(
            "{\n .reg .pred q;\n mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2;\n"
            " selp.u32 %0, 1, 0, q;\n}"
            : "=r"(done)
            : "r"(mbar_addr), "r"(phase));
        if (spin > (1ll << 24)) asm volatile("trap;");
      }
      phase ^= 1u;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]),
          "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    // row m = tid of tile j = m >> 4 reads column j: warp w holds tiles 2w, 2w+1
    uint32_t dj = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w)
      if (warp == w) dj = lane < 16 ? d[2 * w] : d[2 * w + 1];
    const unsigned bal = __ballot_sync(0xffffffffu, dj != 0u);
    if ((lane & 15) == 0) {
      const int j = tid >> 4;
      const uint32_t mask = (bal >> (lane & 16)) & 0xffffu;
      if (mask && s_row[j] >= 0) atomicOr(&a.hit[s_row[j]], mask);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // the next batch rewrites sA / sB / s_row
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

}  // namespace tcmis_b200
