// tile_excl.cuh -- Phase 2 (neighbour exclusion) over the compact T = 16 tile
// store, in the engine's round: the paper's tile form.
//
// Reference: tiled_spmv (spmv.cpp:18-59) computes nc = A * c block row by
// block row over the non-empty T x T tiles, skipping a tile whose candidate
// segment is zero (spmv.cpp:40-43); phase3_update removes an alive
// non-candidate with nc > 0 (engine.cpp:144-147).  Only "nc > 0" matters, so
// both kernels produce, per block row b, the 16-bit mask hit[b] of rows with a
// candidate neighbour; k_update (Phase 3) removes the alive rows in it.
//
// Work layout: flat over the tile array (tile-parallel), because tiles per
// block row range from ~5 (grid) to ~10^5 (R-MAT hub rows): a warp per block
// row -- the first version, and the paper's "one tile per warp" -- left 84 %
// of the lanes idle on the grid and serialised the hub rows on R-MAT s22.
//
//   k_tile_excl_bits  CUDA cores: one tile per thread (coalesced 4 B column +
//                     4 B row + 32 B payload when the segment is non-zero);
//                     (row_i & seg) != 0 gives the tile's row mask; lanes of
//                     the same block row OR-reduce (__match_any_sync) and one
//                     atomicOr per block row segment of the warp.
//   k_tile_excl_mma   tensor cores: a warp takes 32 consecutive tiles; the
//                     non-skipped ones of one block row are K-concatenated two
//                     at a time into one mma.sync.m16n8k32 s8 x s8 -> s32 (A =
//                     two 16x16 bit tiles expanded to 0/1 bytes in registers,
//                     B column 0 = their candidate segments) -- Listing 1's
//                     WMMA on the native IMMA path; the b1
//                     .and.popc MMA is emulated on sm_100a.  The
//                     accumulator is flushed when the block row changes.
//
// The candidate segments come from a bitmap the select kernels fill
// (publish()), bit v of word v/32, so segment b is bits 16*(b&1).. of word b/2.
#pragma once

#include "common.cuh"

namespace tcmis_b200 {

struct TileExclArgs {
  int64_t tiles;
  const int32_t *trow;           // block row per tile
  const int32_t *tcol;           // block column per tile
  const uint16_t *tbits;         // 16 rows of 16 bits per tile
  const uint32_t *cbits;         // this round's candidates, bit per vertex
  uint32_t *hit;                 // out: per block row, rows with a candidate neighbour
  const Ctrl *gate_ctrl;         // Phase 1 use: run only in a tile round (alive >= gate)
  int32_t gate;
};

__device__ __forceinline__ uint32_t seg16(const uint32_t *__restrict__ cbits, int32_t c) {
  return (__ldg(&cbits[c >> 1]) >> ((c & 1) * 16)) & 0xffffu;
}

// OR-combine m over the lanes holding the same block row b and let the lowest
// such lane publish it (one atomic per block-row run of the warp)
__device__ __forceinline__ void or_by_row(uint32_t *hit, int32_t b, uint32_t m, bool valid) {
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned grp = __match_any_sync(act, b);
  const uint32_t r = __reduce_or_sync(grp, m);
  const int lane = threadIdx.x & 31;
  if (r && lane == __ffs(grp) - 1) atomicOr(&hit[b], r);
}

__global__ void __launch_bounds__(256) k_tile_excl_bits(TileExclArgs a) {
  if (a.gate_ctrl && a.gate_ctrl->alive < a.gate) return;
  const uint4 *__restrict__ pay = reinterpret_cast<const uint4 *>(a.tbits);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < a.tiles;
       base += stride) {
    const int64_t t = base + (threadIdx.x & 31);
    const bool valid = t < a.tiles;
    uint32_t m = 0;
    int32_t b = 0;
    if (valid) {
      b = __ldg(&a.trow[t]);
      const uint32_t sg = seg16(a.cbits, __ldg(&a.tcol[t]));
      if (sg) {  // spmv.cpp:40-43: a zero segment skips the tile
        const uint4 lo = __ldg(&pay[2 * t]), hi = __ldg(&pay[2 * t + 1]);
        const uint32_t w[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          m |= ((w[k] & sg) != 0u) << (2 * k);
          m |= (((w[k] >> 16) & sg) != 0u) << (2 * k + 1);
        }
      }
    }
    or_by_row(a.hit, b, m, valid);
  }
}

// 4 bits -> 4 bytes of 0/1 (bit i -> byte i)
__device__ __forceinline__ uint32_t nib_s8(uint32_t x) {
  x &= 0xfu;
  return (x & 1u) | ((x & 2u) << 7) | ((x & 4u) << 14) | ((x & 8u) << 21);
}

__global__ void __launch_bounds__(256) k_tile_excl_mma(TileExclArgs a) {
  const int lane = threadIdx.x & 31;
  const int grp = lane >> 2, tig = lane & 3;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); base < a.tiles;
       base += stride) {
    // lane j looks up tile base + j; the warp then multiplies the non-zero
    // ones in order
    const int64_t tl = base + lane;
    int32_t row = -1;
    uint32_t sg = 0;
    if (tl < a.tiles) {
      row = __ldg(&a.trow[tl]);
      sg = seg16(a.cbits, __ldg(&a.tcol[tl]));
    }
    unsigned act = __ballot_sync(0xffffffffu, sg != 0u);
    int32_t cur = -1;
    int d0 = 0, d1 = 0, d2 = 0, d3 = 0;
    auto flush = [&]() {
      // D column 0 (the block row's nc) sits in d0 (row grp) and d2 (row
      // grp + 8) of the lanes with tig == 0
      const uint32_t mine =
          tig == 0 ? ((d0 > 0 ? 1u : 0u) << grp) | ((d2 > 0 ? 1u : 0u) << (grp + 8)) : 0u;
      const uint32_t m = __reduce_or_sync(0xffffffffu, mine);
      if (lane == 0 && m) atomicOr(&a.hit[cur], m);
      d0 = d1 = d2 = d3 = 0;
    };
    while (act) {
      const int ja = __ffs(act) - 1;
      act &= act - 1;
      const int32_t ra = __shfl_sync(0xffffffffu, row, ja);
      if (ra != cur) {
        if (cur >= 0) flush();
        cur = ra;
      }
      int jb = -1;
      if (act) {
        const int j2 = __ffs(act) - 1;
        if (__shfl_sync(0xffffffffu, row, j2) == ra) {
          jb = j2;
          act &= act - 1;
        }
      }
      const uint32_t sa = __shfl_sync(0xffffffffu, sg, ja);
      const uint32_t sb = __shfl_sync(0xffffffffu, sg, jb < 0 ? ja : jb);
      const int64_t ta = base + ja;
      const uint32_t ra0 = __ldg(&a.tbits[ta * 16 + grp]);
      const uint32_t ra1 = __ldg(&a.tbits[ta * 16 + grp + 8]);
      uint32_t rb0 = 0, rb1 = 0;
      if (jb >= 0) {
        const int64_t tb = base + jb;
        rb0 = __ldg(&a.tbits[tb * 16 + grp]);
        rb1 = __ldg(&a.tbits[tb * 16 + grp + 8]);
      }
      // A (16 x 32, row-major s8): a0/a1 = rows grp/grp+8 of tile a, cols
      // tig*4..+3; a2/a3 = the same rows of tile b (cols 16 + tig*4..+3)
      const uint32_t a0 = nib_s8(ra0 >> (tig * 4)), a1 = nib_s8(ra1 >> (tig * 4));
      const uint32_t a2 = nib_s8(rb0 >> (tig * 4)), a3 = nib_s8(rb1 >> (tig * 4));
      // B (32 x 8, col-major s8): column 0 = [seg_a; seg_b], rows tig*4..+3
      const uint32_t b0 = grp == 0 ? nib_s8(sa >> (tig * 4)) : 0u;
      const uint32_t b1 = (grp == 0 && jb >= 0) ? nib_s8(sb >> (tig * 4)) : 0u;
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 "
          "{%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, {%0, %1, %2, %3};\n"
          : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3)
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    if (cur >= 0) flush();
  }
}

// ---------------------------------------------- Phase 1 as a tile product
// (tile_cand.cu): the round's alive set as a bitmap, k_tile_excl_bits over
// the A-up store and that bitmap (blocked[b] = rows of block row b with an
// alive higher-key neighbour), then the candidates.

// bit v of word v/32 = (state[v] == Alive), 32 states per thread (two
// 16-byte loads); the round's Phase 1 start stamp
__global__ void __launch_bounds__(256)
    k_alive_bits(int32_t n, const uint8_t *__restrict__ state, uint32_t *__restrict__ bits,
                 DevRound *rounds, const Ctrl *ctrl, int32_t gate) {
  if (ctrl->alive < gate) return;  // not a tile round: the CSR select kernels run
  stamp_phase(rounds, ctrl, ctrl->round, 0, 0);
  const int64_t words = ((int64_t)n + 31) / 32;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v0 = w * 32;
    uint32_t m = 0;
    if (v0 + 32 <= n) {
      const uint4 a = __ldg(reinterpret_cast<const uint4 *>(state + v0));
      const uint4 b = __ldg(reinterpret_cast<const uint4 *>(state + v0 + 16));
      const uint32_t x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t e = __vcmpeq4(x[k], 0u);  // 0xff per Alive byte
#pragma unroll
        for (int j = 0; j < 4; ++j) m |= ((e >> (8 * j + 7)) & 1u) << (4 * k + j);
      }
    } else {
      for (int64_t v = v0; v < n; ++v) m |= (uint32_t)(state[v] == TCMIS_ALIVE) << (v - v0);
    }
    bits[w] = m;
  }
}

// The candidates: a warp per 32-vertex word, C = alive AND NOT blocked from
// one word of each bitmap (the round's alive set is exactly the alive
// bitmap, so no worklist is read).  Lane j owns vertex 32w + j: the marks are
// coalesced byte stores (generate_candidates, engine.cpp:105-119) and, with
// the push exclusion, each candidate lane excludes its own CSR neighbours (the
// pull form reads next == 1 itself).  C also goes out as the candidate bitmap
// of the tile-form exclusion, and blocked is cleared behind the read for the
// next tile round.
__global__ void __launch_bounds__(256)
    k_tile_mark(int32_t n, const uint32_t *__restrict__ alive, uint32_t *__restrict__ blocked,
                uint32_t *__restrict__ cbits, uint8_t *__restrict__ next, uint8_t *__restrict__ state,
                uint8_t *__restrict__ segflag, int T, Ctrl *ctrl, int32_t gate, int push,
                const int64_t *__restrict__ off, const int32_t *__restrict__ nbr) {
  if (ctrl->alive < gate) return;
  const int lane = threadIdx.x & 31;
  const int64_t words = ((int64_t)n + 31) / 32;
  unsigned long long sel = 0;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < words;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    uint32_t c = 0;
    if (lane == 0) {
      const uint32_t a = __ldg(&alive[w]);
      const bool hi = (2 * w + 1) * 16 < n;
      const uint32_t blk = (blocked[2 * w] & 0xffffu) | (hi ? (blocked[2 * w + 1] << 16) : 0u);
      if (blk) {
        blocked[2 * w] = 0;
        if (hi) blocked[2 * w + 1] = 0;
      }
      c = a & ~blk;
      cbits[w] = c;
      sel += __popc(c);
    }
    c = __shfl_sync(0xffffffffu, c, 0);
    if ((c >> lane) & 1u) {
      const int32_t v = (int32_t)(w * 32 + lane);
      next[v] = 1;
      state[v] = TCMIS_IN_MIS;
      if (segflag) segflag[seg_of(v, T)] = 1;
      if (push)  // (a 16-byte window of the row's last 4 entries measured slower)
        for (int64_t e = __ldg(&off[v]), e1 = __ldg(&off[v + 1]); e < e1; ++e)
          next[__ldg(&nbr[e])] = 2;
    }
  }
  block_add3(sel, 0, 0, ctrl);
}

}  // namespace tcmis_b200
