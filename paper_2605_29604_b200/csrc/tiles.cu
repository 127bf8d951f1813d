// tiles.cu -- K1, the CSR -> T x T tile converter (tiling.cpp:44-84).
//
// The reference tiles serially: per block row it gathers every entry, sorts by
// block column and ORs payload bits (41.6 s at R-MAT s22).  Here a
// warp owns one (block row, block-column range) work item and merges the T
// sorted neighbour rows of the block on the fly: lane i holds a cursor into
// row b*T+i (lanes i and i+32 for T > 32), the warp takes the minimum current
// block column with a single __reduce_min_sync, emits one tile and advances
// every lane whose cursor sits in that column.  Neighbour lists are read once,
// coalesced per lane run; no sort, no scratch.  Block rows with more than
// kChunk entries (hubs) are split into block-column ranges so no warp walks a
// 162k-entry row alone.
//
// Pass 1 counts tiles per work item (and per block row: the tile counters of
// run_tc_mis need exactly `tiles in block column b`, which equals `tiles in
// block row b` because A is symmetric).  Pass 2 (export only) writes the tiles
// in the reference layout: (tile_row, tile_col, T u64 row words).
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "internal.cuh"

namespace tcmis_b200 {

namespace {

constexpr int64_t kChunk = 2048;  // entries per work item before splitting
constexpr uint32_t kNone = 0xffffffffu;

__global__ void k_item_counts(int32_t n, int T, int32_t nb, const int64_t *__restrict__ off,
                              int64_t *__restrict__ items) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = b * T, hi = std::min<int64_t>(n, lo + T);
    const int64_t nnz = off[hi] - off[lo];
    items[b] = std::max<int64_t>(1, (nnz + kChunk - 1) / kChunk);
  }
}

__global__ void k_item_rows(int32_t nb, const int64_t *__restrict__ item_start,
                            int32_t *__restrict__ item_row) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    for (int64_t i = item_start[b]; i < item_start[b + 1]; ++i) item_row[i] = (int32_t)b;
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t *__restrict__ a, int64_t lo,
                                                   int64_t hi, int64_t x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One warp per work item.  emit == false: count; emit == true: write tiles
// starting at item_off[item], each row word as `row_bytes` bytes: 8 = the
// reference layout (u64 per row, tiling.hpp:21-24), 2 / 1 = the compact
// device layout of T = 16 / T = 8 (internal.cuh "tile store").
template <bool emit>
__global__ void __launch_bounds__(256)
    k_tile_merge(int32_t n, int T, int32_t nb, const int64_t *__restrict__ off,
                 const int32_t *__restrict__ nbr, int64_t n_items,
                 const int32_t *__restrict__ item_row, const int64_t *__restrict__ item_start,
                 int64_t *__restrict__ item_cnt, int32_t *__restrict__ rowtiles,
                 const int64_t *__restrict__ item_off, int32_t *__restrict__ tile_row,
                 int32_t *__restrict__ tile_col, void *__restrict__ row_bits, int row_bytes) {
  const int lane = threadIdx.x & 31;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < n_items;
       it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t b = item_row[it];
    const int64_t j = it - item_start[b];
    const int64_t c = item_start[b + 1] - item_start[b];
    const int64_t bc_lo = j * nb / c, bc_hi = (j + 1) * nb / c;
    // up to two rows per lane (T <= 64)
    int64_t pos[2], end[2];
    uint32_t cur[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = lane + 32 * k;
      const int64_t r = (int64_t)b * T + i;
      pos[k] = end[k] = 0;
      cur[k] = kNone;
      if (i < T && r < n) {
        end[k] = off[r + 1];
        pos[k] = lower_bound_i32(nbr, off[r], end[k], bc_lo * T);
        if (pos[k] < end[k]) {
          const int64_t bc = nbr[pos[k]] / T;
          if (bc < bc_hi) cur[k] = (uint32_t)bc;
        }
      }
    }
    int64_t count = 0;
    for (;;) {
      const uint32_t m = __reduce_min_sync(0xffffffffu, min(cur[0], cur[1]));
      if (m == kNone) break;
      uint64_t word[2] = {0, 0};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (cur[k] == m) {
          const int64_t base = (int64_t)m * T;
          int64_t p = pos[k];
          while (p < end[k]) {
            const int64_t u = nbr[p];
            if (u - base >= T) break;
            if (emit) word[k] |= 1ull << (u - base);
            ++p;
          }
          pos[k] = p;
          cur[k] = kNone;
          if (p < end[k]) {
            const int64_t bc = nbr[p] / T;
            if (bc < bc_hi) cur[k] = (uint32_t)bc;
          }
        }
      }
      if (emit) {
        const int64_t t = item_off[it] + count;
        if (lane == 0) {
          if (tile_row) tile_row[t] = b;
          tile_col[t] = (int32_t)m;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int i = lane + 32 * k;
          if (i < T) {
            if (row_bytes == 8) static_cast<uint64_t *>(row_bits)[t * T + i] = word[k];
            else if (row_bytes == 2) static_cast<uint16_t *>(row_bits)[t * T + i] = (uint16_t)word[k];
            else static_cast<uint8_t *>(row_bits)[t * T + i] = (uint8_t)word[k];
          }
        }
      }
      ++count;
    }
    if (!emit && lane == 0) {
      item_cnt[it] = count;
      if (count) atomicAdd(&rowtiles[b], (int32_t)count);
    }
  }
}

// ------------------------------------------------------------ tile counts
//
// The solve needs only rowtiles[b] = |{distinct block columns among the
// entries of block row b}| (tiles in block column b by symmetry), not the
// tiles themselves.  The entries of a block row are contiguous in the CSR
// (rows b*T .. b*T+T-1), so both kernels stream them coalesced and count
// distinct block columns in shared memory -- one pass over nbr, no merge:
//
//  k_count_light  one warp per block row with <= kHashMax entries (88 % of
//                 R-MAT s22's block rows): a 1024-slot open-addressing set
//                 in shared memory (atomicCAS), cleared after each row.
//  k_count_mid    <= kMidMax entries: one 256-thread CTA per row (dynamic
//                 work counter), an 8192-slot shared set -- or, when the
//                 graph has at most 2^18 block columns, every non-light row
//                 on an exact 2^18-bit shared bitmap.
//  k_count_big    the rest: one 512-thread CTA per row, 64 KB of dynamic
//                 shared memory used as a set sized to the row (<= kBigHashMax
//                 entries) or, for the hub rows beyond, as a 2^19-bit bitmap
//                 swept window by window (one binary search per row and
//                 window: the rows are sorted).
//  The first version had only the light set and a bitmap CTA per (block row,
//  2^18-column window) that located each window by binary search in all T
//  rows: 202 ms at R-MAT s26 (half the block rows exceed 512 entries there).
constexpr int kLightBlock = 256;
constexpr int kHashSlots = 1024;
constexpr int64_t kHashMax = 512;
constexpr int kMidBlock = 256;
constexpr int kMidSlots = 8192;           // 32 KB: 7 CTAs per SM
constexpr int64_t kMidMax = 4096;
constexpr int kBigBlock = 512;
constexpr int kBigWords = 16384;          // 64 KB of dynamic shared memory: 3 CTAs per SM
constexpr int64_t kBigHashMax = 8192;     // set of <= 16384 slots
constexpr int64_t kBigBits = 32ll * kBigWords;
constexpr int kBigGroup = 8;
constexpr int kUploadChunks = 8;          // upload_tiled: chunks of the neighbour-id upload              // windows whose row boundaries are searched together
// hub block rows (R-MAT s22's block row 0 holds ~1M entries): one CTA per
// row serialised the whole count behind it (0.5-1.1 ms); they are counted by
// kHubCTAs CTAs each on a global bitmap (L2 atomics), kHubBatch rows at a time
constexpr int64_t kHubMin = 65536;
constexpr int kHubCTAs = 64;
constexpr int kHubBatch = 64;

__global__ void __launch_bounds__(256)
    k_count_hub(int32_t n, int T, int32_t nb, const int64_t *__restrict__ off,
                const int32_t *__restrict__ nbr, int32_t *__restrict__ rowtiles,
                const int32_t *__restrict__ hubs, int first, uint32_t *__restrict__ bitmaps) {
  __shared__ int s_red[8];
  const int h = blockIdx.y;
  const int32_t b = hubs[first + h];
  const int64_t r0 = (int64_t)b * T, r1 = min((int64_t)n, r0 + T);
  const int64_t s = off[r0], e = off[r1];
  uint32_t *bm = bitmaps + (size_t)h * (((size_t)nb + 31) / 32);
  const uint32_t uT = (uint32_t)T;
  int cnt = 0;
  const int64_t stride = (int64_t)gridDim.x * 256 * 4;
  for (int64_t base = s + (int64_t)blockIdx.x * 256 * 4; base < e; base += stride) {
    uint32_t c[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t p = base + threadIdx.x + 256ll * j;
      c[j] = p < e ? (uint32_t)__ldg(&nbr[p]) / uT : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (c[j] == 0xffffffffu) continue;
      const uint32_t bit = 1u << (c[j] & 31u);
      cnt += (atomicOr(&bm[c[j] >> 5], bit) & bit) ? 0 : 1;
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < 8; ++i) t += s_red[i];
    if (t) atomicAdd(&rowtiles[b], t);
  }
}

__global__ void __launch_bounds__(kLightBlock)
    k_count_light(int32_t n, int T, int32_t nb, int32_t b_lo, int32_t b_hi,
                  const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                  int32_t *__restrict__ rowtiles, int32_t *__restrict__ lists,
                  int32_t *__restrict__ counts, int bitmap, int32_t *__restrict__ hubs) {
  __shared__ __align__(16) uint32_t tab[kLightBlock / 32][kHashSlots];
  const int lane = threadIdx.x & 31;
  uint32_t *t = tab[threadIdx.x >> 5];
  uint4 *t4 = reinterpret_cast<uint4 *>(t);
  for (int i = lane; i < kHashSlots / 4; i += 32) t4[i] = make_uint4(0, 0, 0, 0);
  __syncwarp();
  const uint32_t uT = (uint32_t)T;
  for (int64_t b = b_lo + (((int64_t)blockIdx.x * kLightBlock + threadIdx.x) >> 5); b < b_hi;
       b += ((int64_t)gridDim.x * kLightBlock) >> 5) {
    const int64_t r0 = b * T, r1 = min((int64_t)n, r0 + T);
    const int64_t s = off[r0], e = off[r1];
    if (e - s > kHashMax) {  // mid rows from the front of `lists`, big rows from the back
      if (lane == 0) {
        if (e - s > kHubMin) hubs[atomicAdd(&counts[4], 1)] = (int32_t)b;
        else if (bitmap || e - s <= kMidMax) lists[atomicAdd(&counts[0], 1)] = (int32_t)b;
        else lists[nb - 1 - atomicAdd(&counts[1], 1)] = (int32_t)b;
      }
      continue;
    }
    int cnt = 0;
    for (int64_t base = s; base < e; base += 128) {
      uint32_t c[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t p = base + lane + 32 * j;
        c[j] = p < e ? (uint32_t)__ldg(&nbr[p]) / uT + 1u : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!c[j]) continue;
        uint32_t h = (c[j] * 0x9E3779B1u) >> 22;
        for (;;) {
          const uint32_t old = atomicCAS(&t[h], 0u, c[j]);
          if (old == 0u) {
            ++cnt;
            break;
          }
          if (old == c[j]) break;
          h = (h + 1) & (kHashSlots - 1);
        }
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) rowtiles[b] = cnt;
    if (e > s) {
      __syncwarp();
      for (int i = lane; i < kHashSlots / 4; i += 32) t4[i] = make_uint4(0, 0, 0, 0);
      __syncwarp();
    }
  }
}

// CTA-wide insert of block columns [s, e) into a shared set of `slots`
// (power of two) slots; returns the CTA's count of first insertions (valid in
// every thread) and leaves the set cleared.
__device__ __forceinline__ int cta_hash_count(uint32_t *tab, int slots, const int32_t *__restrict__ nbr,
                                              int64_t s, int64_t e, uint32_t uT, int *s_red) {
  const int shift = 32 - (__ffs(slots) - 1);
  int cnt = 0;
  for (int64_t base = s; base < e; base += 4 * (int64_t)blockDim.x) {
    uint32_t cc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // 4 independent loads in flight per thread
      const int64_t p = base + threadIdx.x + (int64_t)blockDim.x * j;
      cc[j] = p < e ? (uint32_t)__ldg(&nbr[p]) / uT + 1u : 0u;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t c = cc[j];
      if (!c) continue;
      uint32_t h = (c * 0x9E3779B1u) >> shift;
      for (;;) {
        const uint32_t old = atomicCAS(&tab[h], 0u, c);
        if (old == 0u) {
          ++cnt;
          break;
        }
        if (old == c) break;
        h = (h + 1) & (slots - 1);
      }
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
  __syncthreads();
  int total = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) total += s_red[w];
  uint4 *t4 = reinterpret_cast<uint4 *>(tab);
  for (int i = threadIdx.x; i < slots / 4; i += blockDim.x) t4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kMidBlock)
    k_count_mid(int32_t n, int T, const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                int32_t *__restrict__ rowtiles, const int32_t *__restrict__ list,
                const int32_t *__restrict__ count, unsigned *__restrict__ next_item, int bitmap) {
  __shared__ __align__(16) uint32_t tab[kMidSlots];
  __shared__ int s_red[kMidBlock / 32];
  __shared__ unsigned s_item;
  uint4 *t4 = reinterpret_cast<uint4 *>(tab);
  for (int i = threadIdx.x; i < kMidSlots / 4; i += kMidBlock) t4[i] = make_uint4(0, 0, 0, 0);
  const unsigned items = (unsigned)*count;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(next_item, 1u);
    __syncthreads();
    const unsigned it = s_item;
    if (it >= items) break;
    const int32_t b = list[it];
    const int64_t r0 = (int64_t)b * T, r1 = min((int64_t)n, r0 + T);
    const int64_t s = off[r0], e = off[r1];
    int total;
    if (bitmap) {  // every block column has its own bit (nb <= 32 * kMidSlots)
      int cnt = 0;
      for (int64_t base = s; base < e; base += 4 * kMidBlock) {
        uint32_t c[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // 4 independent loads in flight per thread
          const int64_t p = base + threadIdx.x + (int64_t)kMidBlock * j;
          c[j] = p < e ? (uint32_t)__ldg(&nbr[p]) / (uint32_t)T : 0xffffffffu;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (c[j] == 0xffffffffu) continue;
          const uint32_t bit = 1u << (c[j] & 31u);
          cnt += (atomicOr(&tab[c[j] >> 5], bit) & bit) ? 0 : 1;
        }
      }
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
      __syncthreads();
      total = 0;
      for (int w = 0; w < kMidBlock / 32; ++w) total += s_red[w];
      for (int i = threadIdx.x; i < kMidSlots / 4; i += kMidBlock) t4[i] = make_uint4(0, 0, 0, 0);
      __syncthreads();
    } else {
      int slots = 1024;
      while (slots < 2 * (e - s) && slots < kMidSlots) slots <<= 1;
      total = cta_hash_count(tab, slots, nbr, s, e, (uint32_t)T, s_red);
    }
    if (threadIdx.x == 0) rowtiles[b] = total;
  }
}

__global__ void __launch_bounds__(kBigBlock)
    k_count_big(int32_t n, int T, int32_t nb, const int64_t *__restrict__ off,
                const int32_t *__restrict__ nbr, int32_t *__restrict__ rowtiles,
                const int32_t *__restrict__ list_end, const int32_t *__restrict__ count,
                unsigned *__restrict__ next_item) {
  extern __shared__ __align__(16) uint32_t big[];  // kBigWords
  __shared__ int s_red[kBigBlock / 32];
  __shared__ int64_t s_bound[64][kBigGroup + 1];
  __shared__ int64_t s_pre[65];
  __shared__ unsigned s_item;
  uint4 *b4 = reinterpret_cast<uint4 *>(big);
  for (int i = threadIdx.x; i < kBigWords / 4; i += kBigBlock) b4[i] = make_uint4(0, 0, 0, 0);
  const unsigned items = (unsigned)*count;
  const uint32_t uT = (uint32_t)T;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(next_item, 1u);
    __syncthreads();
    const unsigned it = s_item;
    if (it >= items) break;
    const int32_t b = list_end[-(int64_t)it];
    const int64_t r0 = (int64_t)b * T;
    const int rows = (int)min((int64_t)T, (int64_t)n - r0);
    const int64_t s = off[r0], e = off[r0 + rows];
    if (e - s <= kBigHashMax) {
      int slots = 1024;
      while (slots < 2 * (e - s) && slots < kBigWords) slots <<= 1;
      const int total = cta_hash_count(big, slots, nbr, s, e, uT, s_red);
      if (threadIdx.x == 0) rowtiles[b] = total;
      continue;
    }
    // rows beyond the set: windows of kBigBits block columns.  Row k's
    // entries of window w are [lower_bound(k, w), lower_bound(k, w + 1))
    // (sorted rows).  The boundaries of kBigGroup windows are searched at
    // once, one thread per (row, boundary), and each window is then ONE flat
    // pass over the concatenated row segments.  (The previous version ran the
    // T searches of a window and then T per-row loops one after another: a
    // chain of dependent loads per window, 13.7 of the 23.5 ms of R-MAT s26's
    // tile count.)
    int cnt = 0;
    const int64_t windows = ((int64_t)nb + kBigBits - 1) / kBigBits;
    for (int64_t w0 = 0; w0 < windows; w0 += kBigGroup) {
      const int gw = (int)min((int64_t)kBigGroup, windows - w0);
      for (int i = threadIdx.x; i < rows * (gw + 1); i += kBigBlock) {
        const int k = i / (gw + 1), jb = i % (gw + 1);
        const int64_t wb = w0 + jb;
        const int64_t rs = off[r0 + k], re = off[r0 + k + 1];
        s_bound[k][jb] = wb == 0 ? rs
                         : wb >= windows ? re
                                         : lower_bound_i32(nbr, rs, re, wb * kBigBits * T);
      }
      __syncthreads();
      for (int jw = 0; jw < gw; ++jw) {
        const uint32_t wlo = (uint32_t)((w0 + jw) * kBigBits);
        if (threadIdx.x < 32) {  // segment prefix over the rows (rows <= 64)
          const int k0 = threadIdx.x, k1 = threadIdx.x + 32;
          const int64_t l0 = k0 < rows ? s_bound[k0][jw + 1] - s_bound[k0][jw] : 0;
          const int64_t l1 = k1 < rows ? s_bound[k1][jw + 1] - s_bound[k1][jw] : 0;
          int64_t x0 = l0, x1 = l1;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int64_t y0 = __shfl_up_sync(0xffffffffu, x0, d);
            const int64_t y1 = __shfl_up_sync(0xffffffffu, x1, d);
            if (k0 >= d) {
              x0 += y0;
              x1 += y1;
            }
          }
          const int64_t tot0 = __shfl_sync(0xffffffffu, x0, 31);
          s_pre[k0] = x0 - l0;
          s_pre[k1] = tot0 + x1 - l1;
          if (k0 == 31) s_pre[64] = tot0 + x1;
        }
        __syncthreads();
        const int64_t total = s_pre[64];
        for (int64_t q0 = threadIdx.x; q0 < total; q0 += 4 * kBigBlock) {
          uint32_t c[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t q = q0 + (int64_t)kBigBlock * j;
            c[j] = 0xffffffffu;
            if (q < total) {
              int lo = 0, hi = rows - 1;  // last row with s_pre[k] <= q
              while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (s_pre[mid] <= q) lo = mid;
                else hi = mid - 1;
              }
              c[j] = (uint32_t)__ldg(&nbr[s_bound[lo][jw] + (q - s_pre[lo])]) / uT - wlo;
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (c[j] == 0xffffffffu) continue;
            const uint32_t bit = 1u << (c[j] & 31u);
            cnt += (atomicOr(&big[c[j] >> 5], bit) & bit) ? 0 : 1;
          }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kBigWords / 4; i += kBigBlock) b4[i] = make_uint4(0, 0, 0, 0);
        __syncthreads();
      }
    }
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      int total = 0;
      for (int i = 0; i < kBigBlock / 32; ++i) total += s_red[i];
      rowtiles[b] = total;
    }
  }
}

__global__ void k_sum_rowtiles(const int32_t *__restrict__ rowtiles, int32_t nb,
                               unsigned long long *__restrict__ total) {
  unsigned long long s = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    s += (unsigned long long)rowtiles[b];
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(total, s);
}

struct Items {
  int64_t *start = nullptr;  // nb + 1
  int32_t *row = nullptr;
  int64_t *cnt = nullptr;
  int64_t n_items = 0;
  void *tmp = nullptr;
  ~Items() {
    dev_free(start);
    dev_free(row);
    dev_free(cnt);
    dev_free(tmp);
  }
};

int plan_items(tcmis_graph *g, int T, int32_t nb, Items &it) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (int rc = dev_alloc(&it.start, (size_t)nb + 1)) return rc;
  k_item_counts<<<grid_for(ctx, nb, 256, 8), 256, 0, st>>>(g->n, T, nb, g->d_off, it.start);
  TCMIS_LAUNCHED(ctx);
  size_t bytes = 0;
  TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it.start, it.start, (int64_t)nb + 1,
                                           st));
  if (int rc_ = dev_alloc((char **)&it.tmp, bytes)) return rc_;
  // the extra (nb-th) slot is garbage before the scan; zero it so the scan
  // yields start[nb] = total items
  TCMIS_CUDA(cudaMemsetAsync(it.start + nb, 0, sizeof(int64_t), st));
  TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(it.tmp, bytes, it.start, it.start, (int64_t)nb + 1,
                                           st));
  ctx->launches++;
  TCMIS_CUDA(cudaMemcpyAsync(&it.n_items, it.start + nb, sizeof(int64_t), cudaMemcpyDeviceToHost,
                             st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (int rc = dev_alloc(&it.row, (size_t)it.n_items)) return rc;
  if (int rc = dev_alloc(&it.cnt, (size_t)it.n_items)) return rc;
  k_item_rows<<<grid_for(ctx, nb, 256, 8), 256, 0, st>>>(nb, it.start, it.row);
  TCMIS_LAUNCHED(ctx);
  return 0;
}

}  // namespace

// K1 in three steps, so the light pass can run block-row range by range
// while the neighbour ids are still arriving (upload_tiled).
struct K1Plan {
  int T = 0;
  int32_t nb = 0;
  int bitmap = 0;
  int32_t *lists = nullptr, *cnt = nullptr, *hubs = nullptr;
  uint32_t *bms = nullptr;  // hub bitmaps, kHubBatch of them
};

int k1_begin(tcmis_graph *g, int T, K1Plan &p) {
  if (T < 1 || T > 64)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tile_dim must be in [1, 64], got " + std::to_string(T));
  cudaStream_t st = g->ctx->stream;
  const int32_t nb = (int32_t)(((int64_t)g->n + T - 1) / T);
  dev_free(g->d_rowtiles);
  g->d_rowtiles = nullptr;
  g->tile_T = 0;
  g->tile_nb = nb;
  g->tile_total = 0;
  p = K1Plan{};
  p.T = T;
  p.nb = nb;
  if (int rc = dev_alloc(&g->d_rowtiles, (size_t)nb + 1)) return rc;
  TCMIS_CUDA(cudaMemsetAsync(g->d_rowtiles, 0, sizeof(int32_t) * ((size_t)nb + 1), st));
  if (nb == 0) return 0;
  // lists: mid rows from the front, big rows from the back; cnt[0..1] list
  // sizes, cnt[2..3] the dynamic work counters, cnt[4] the hub count.  Few
  // enough block columns for one shared bitmap (R-MAT s22: nb = 2^18): every
  // non-light row goes to k_count_mid's exact bitmap, no hashing.
  p.bitmap = (int64_t)nb <= 32ll * kMidSlots ? 1 : 0;
  if (int rc = dev_alloc(&p.lists, (size_t)nb)) return rc;
  if (int rc = dev_alloc(&p.hubs, (size_t)nb)) return rc;
  if (int rc = dev_alloc(&p.cnt, 8)) return rc;
  TCMIS_CUDA(cudaMemsetAsync(p.cnt, 0, 8 * sizeof(int32_t), st));
  return 0;
}

// light block rows of [b_lo, b_hi) counted, the rest listed (stream st)
int k1_light(tcmis_graph *g, const K1Plan &p, int32_t b_lo, int32_t b_hi, cudaStream_t st) {
  tcmis_ctx *ctx = g->ctx;
  if (b_hi <= b_lo) return 0;
  k_count_light<<<grid_for(ctx, 32ll * (b_hi - b_lo), kLightBlock, 8), kLightBlock, 0, st>>>(
      g->n, p.T, p.nb, b_lo, b_hi, g->d_off, g->d_nbr, g->d_rowtiles, p.lists, p.cnt, p.bitmap,
      p.hubs);
  TCMIS_LAUNCHED(ctx);
  return 0;
}

// The heavy rows k_count_light listed: hubs [hub_lo, hub_hi), mid rows
// [mid_lo, mid_hi) of the front list and big rows [big_lo, big_hi) of the
// back list, on stream st.  The work counters are set to the range starts so
// the list can be processed in instalments as the light pass extends it.
int k1_heavy(tcmis_graph *g, K1Plan &p, int32_t hub_lo, int32_t hub_hi, int32_t mid_lo,
             int32_t mid_hi, int32_t big_lo, int32_t big_hi, cudaStream_t st) {
  tcmis_ctx *ctx = g->ctx;
  const int T = p.T;
  const int32_t nb = p.nb;
  if (hub_hi > hub_lo) {
    // rowtiles[hub] was never written by k_count_light: start from 0
    const size_t words = ((size_t)nb + 31) / 32;
    if (!p.bms) {
      if (int rc = dev_alloc(&p.bms, words * kHubBatch)) return rc;
    }
    for (int first = hub_lo; first < hub_hi; first += kHubBatch) {
      const int nh = std::min(kHubBatch, hub_hi - first);
      TCMIS_CUDA(cudaMemsetAsync(p.bms, 0, 4 * words * nh, st));
      k_count_hub<<<dim3(kHubCTAs, nh), 256, 0, st>>>(g->n, T, nb, g->d_off, g->d_nbr,
                                                      g->d_rowtiles, p.hubs, first, p.bms);
      TCMIS_LAUNCHED(ctx);
    }
  }
  const int32_t starts[2] = {mid_lo, big_lo};
  TCMIS_CUDA(cudaMemcpyAsync(p.cnt + 2, starts, sizeof(starts), cudaMemcpyHostToDevice, st));
  if (mid_hi > mid_lo) {
    int mid_per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&mid_per_sm, k_count_mid, kMidBlock, 0);
    const int64_t grid = std::min<int64_t>((int64_t)ctx->num_sms * std::max(1, mid_per_sm),
                                           mid_hi - mid_lo);
    k_count_mid<<<(int)grid, kMidBlock, 0, st>>>(g->n, T, g->d_off, g->d_nbr, g->d_rowtiles,
                                                 p.lists, p.cnt,
                                                 reinterpret_cast<unsigned *>(p.cnt + 2), p.bitmap);
    TCMIS_LAUNCHED(ctx);
  }
  if (big_hi > big_lo) {
    const size_t big_smem = sizeof(uint32_t) * kBigWords;
    TCMIS_CUDA(cudaFuncSetAttribute(k_count_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)big_smem));
    int big_per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&big_per_sm, k_count_big, kBigBlock, big_smem);
    const int64_t grid = std::min<int64_t>((int64_t)ctx->num_sms * std::max(1, big_per_sm),
                                           big_hi - big_lo);
    k_count_big<<<(int)grid, kBigBlock, big_smem, st>>>(
        g->n, T, nb, g->d_off, g->d_nbr, g->d_rowtiles, p.lists + nb - 1, p.cnt + 1,
        reinterpret_cast<unsigned *>(p.cnt + 3));
    TCMIS_LAUNCHED(ctx);
  }
  return 0;
}

// list sizes after the light passes so far: hub, mid, big (host sync of st)
int k1_lists(K1Plan &p, cudaStream_t st, int32_t *hub, int32_t *mid, int32_t *big) {
  int32_t c[5] = {0, 0, 0, 0, 0};
  TCMIS_CUDA(cudaMemcpyAsync(c, p.cnt, sizeof(c), cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  *mid = c[0];
  *big = c[1];
  *hub = c[4];
  return 0;
}

// the tile total, buffers released (context stream; after every pass)
int k1_total(tcmis_graph *g, K1Plan &p) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (p.nb > 0) {
    dev_free(p.bms);
    dev_free(p.lists);
    dev_free(p.hubs);
    dev_free(p.cnt);
    p.bms = nullptr;
    p.lists = p.hubs = p.cnt = nullptr;
    unsigned long long *d_total = nullptr;
    if (int rc = dev_alloc(&d_total, 1)) return rc;
    cudaMemsetAsync(d_total, 0, 8, st);
    k_sum_rowtiles<<<grid_for(ctx, p.nb, 256, 4), 256, 0, st>>>(g->d_rowtiles, p.nb, d_total);
    ctx->launches++;
    unsigned long long total = 0;
    cudaMemcpyAsync(&total, d_total, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    dev_free(d_total);
    if (e != cudaSuccess) return cuda_error(e, "tile counts");
    g->tile_total = (int64_t)total;
  }
  g->tile_T = p.T;
  return 0;
}

int build_tile_counts(tcmis_graph *g, int T) {
  K1Plan p;
  cudaStream_t st = g->ctx->stream;
  if (int rc = k1_begin(g, T, p)) return rc;
  if (p.nb > 0) {
    if (int rc = k1_light(g, p, 0, p.nb, st)) return rc;
    int32_t hub = 0, mid = 0, big = 0;
    if (int rc = k1_lists(p, st, &hub, &mid, &big)) return rc;
    if (int rc = k1_heavy(g, p, 0, hub, 0, mid, 0, big, st)) return rc;
  }
  return k1_total(g, p);
}

// Host CSR -> device graph with the K1 counts of tile_dim T, the count
// overlapping the upload: the neighbour ids go up in chunks of block rows on
// the context stream (copy engine) and a side stream counts each chunk's
// light rows as soon as it has landed; the hub / mid / big rows follow the
// last chunk.  The drop-in path's upload + tile_graph in one call.
int upload_tiled(tcmis_ctx *ctx, int32_t n, const int64_t *off, const int32_t *nbr, int T,
                 tcmis_graph **out) {
  *out = nullptr;
  if (T < 1 || T > 64)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tile_dim must be in [1, 64], got " + std::to_string(T));
  cudaStream_t st = ctx->stream;
  const int64_t nnz = off ? off[n] : 0;
  int64_t *d_off = nullptr;
  int32_t *d_nbr = nullptr;
  if (int rc = dev_alloc(&d_off, (size_t)n + 1)) return rc;
  if (int rc = dev_alloc(&d_nbr, (size_t)nnz)) {
    dev_free(d_off);
    return rc;
  }
  if (off) {
    if (int rc = h2d(ctx, d_off, off, 8ull * (n + 1), st)) return rc;
  } else {
    TCMIS_CUDA(cudaMemsetAsync(d_off, 0, 8, st));
  }
  tcmis_graph *g = nullptr;
  if (int rc = wrap_owned(ctx, n, nnz, d_off, d_nbr, &g)) return rc;
  *out = g;
  K1Plan p;
  if (int rc = k1_begin(g, T, p)) return rc;
  if (p.nb > 0) {  // hub bitmaps up front: the side stream must not allocate
    if (int rc = dev_alloc(&p.bms, (((size_t)p.nb + 31) / 32) * kHubBatch)) return rc;
  }
  if (!ctx->side) {
    TCMIS_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
    for (cudaEvent_t &e : ctx->side_ev)
      TCMIS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  // ~16M ids per chunk, at most 8 chunks, cut at block-row boundaries.  All
  // copies are enqueued first (copy engine, context stream); the side stream
  // then counts chunk by chunk -- light rows, then the heavy rows the light
  // pass listed -- each chunk as soon as its ids have landed.
  const int K = (int)std::min<int64_t>(kUploadChunks, std::max<int64_t>(1, nnz >> 24));
  std::vector<int32_t> bnd{0};
  for (int c = 1; c <= K && p.nb > 0; ++c) {
    int32_t b_c = p.nb;
    if (c < K) {
      // shrinking chunks (boundary at 1 - (1 - c/K)^2 of the ids): the count of
      // the last chunk, which nothing overlaps, is the smallest
      const double f = 1.0 - (1.0 - (double)c / K) * (1.0 - (double)c / K);
      const int64_t want = (int64_t)(f * (double)nnz);
      int32_t lo = bnd.back(), hi = p.nb;  // first block row whose first entry >= want
      while (lo < hi) {
        const int32_t mid = lo + (hi - lo) / 2;
        if (off[std::min<int64_t>(n, (int64_t)mid * T)] < want) lo = mid + 1;
        else hi = mid;
      }
      b_c = lo;
    }
    if (b_c > bnd.back()) bnd.push_back(b_c);
  }
  const int chunks = (int)bnd.size() - 1;
  int32_t hub0 = 0, mid0 = 0, big0 = 0;
  auto count_chunk = [&](int c) -> int {
    TCMIS_CUDA(cudaStreamWaitEvent(ctx->side, ctx->side_ev[c], 0));
    if (int rc = k1_light(g, p, bnd[c], bnd[c + 1], ctx->side)) return rc;
    int32_t hub = 0, mid = 0, big = 0;
    if (int rc = k1_lists(p, ctx->side, &hub, &mid, &big)) return rc;
    if (int rc = k1_heavy(g, p, hub0, hub, mid0, mid, big0, big, ctx->side)) return rc;
    hub0 = hub;
    mid0 = mid;
    big0 = big;
    return 0;
  };
  // pinned ids: every copy is enqueued at once, then the counts chunk by
  // chunk; pageable ids keep the host busy staging each chunk (staging.cu),
  // so chunk c-1 is counted right after chunk c's ids are staged
  const bool staged = nnz > 0 && !host_pinned(nbr);
  for (int c = 0; c < chunks; ++c) {
    const int64_t e0 = off[(int64_t)bnd[c] * T];
    const int64_t e1 = off[std::min<int64_t>(n, (int64_t)bnd[c + 1] * T)];
    if (e1 > e0)
      if (int rc = h2d(ctx, d_nbr + e0, nbr + e0, 4ull * (e1 - e0), st)) return rc;
    TCMIS_CUDA(cudaEventRecord(ctx->side_ev[c], st));
    if (staged && c > 0)
      if (int rc = count_chunk(c - 1)) return rc;
  }
  if (p.nb == 0 && nnz)
    if (int rc = h2d(ctx, d_nbr, nbr, 4ull * nnz, st)) return rc;
  for (int c = staged ? std::max(0, chunks - 1) : 0; c < chunks; ++c)
    if (int rc = count_chunk(c)) return rc;
  if (chunks > 0) {
    TCMIS_CUDA(cudaEventRecord(ctx->side_ev[kUploadChunks], ctx->side));
    TCMIS_CUDA(cudaStreamWaitEvent(st, ctx->side_ev[kUploadChunks], 0));
  }
  if (int rc = k1_total(g, p)) return rc;
  TCMIS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int export_tiles(tcmis_graph *g, int T, int32_t *tile_row, int32_t *tile_col,
                 uint64_t *row_bits, int64_t *bro) {
  if (g->tile_T != T)
    if (int rc = build_tile_counts(g, T)) return rc;
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int32_t nb = g->tile_nb;
  const int64_t tiles = g->tile_total;
  if (nb == 0) {
    bro[0] = 0;
    return 0;
  }
  Items it;
  if (int rc = plan_items(g, T, nb, it)) return rc;
  // recount per item (cheap) to get exact output offsets per item
  int32_t *scratch_rows = nullptr;
  if (int rc = dev_alloc(&scratch_rows, (size_t)nb + 1)) return rc;
  cudaMemsetAsync(scratch_rows, 0, sizeof(int32_t) * ((size_t)nb + 1), st);
  k_tile_merge<false><<<grid_for(ctx, 32 * it.n_items, 256, 16), 256, 0, st>>>(
      g->n, T, nb, g->d_off, g->d_nbr, it.n_items, it.row, it.start, it.cnt, scratch_rows,
      nullptr, nullptr, nullptr, nullptr, 8);
  ctx->launches++;
  int64_t *item_off = nullptr;
  int32_t *d_tr = nullptr, *d_tc = nullptr;
  uint64_t *d_rb = nullptr;
  int rc = dev_alloc(&item_off, (size_t)it.n_items + 1);
  if (!rc) rc = dev_alloc(&d_tr, (size_t)tiles);
  if (!rc) rc = dev_alloc(&d_tc, (size_t)tiles);
  if (!rc) rc = dev_alloc(&d_rb, (size_t)tiles * T);
  if (!rc) {
    size_t bytes = 0;
    void *tmp = nullptr;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, it.cnt, item_off, it.n_items, st);
    dev_alloc((char **)&tmp, bytes);
    cub::DeviceScan::ExclusiveSum(tmp, bytes, it.cnt, item_off, it.n_items, st);
    k_tile_merge<true><<<grid_for(ctx, 32 * it.n_items, 256, 16), 256, 0, st>>>(
        g->n, T, nb, g->d_off, g->d_nbr, it.n_items, it.row, it.start, it.cnt, scratch_rows,
        item_off, d_tr, d_tc, d_rb, 8);
    ctx->launches += 2;
    std::vector<int64_t> h_start(nb + 1), h_off(it.n_items);
    cudaMemcpyAsync(h_start.data(), it.start, 8ull * (nb + 1), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h_off.data(), item_off, 8ull * it.n_items, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(tile_row, d_tr, 4ull * tiles, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(tile_col, d_tc, 4ull * tiles, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(row_bits, d_rb, 8ull * tiles * T, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    dev_free(tmp);
    if (e != cudaSuccess) {
      rc = cuda_error(e, "export tiles");
    } else {
      for (int32_t b = 0; b < nb; ++b) bro[b] = h_off[h_start[b]];
      bro[nb] = tiles;
    }
  }
  dev_free(scratch_rows);
  dev_free(item_off);
  dev_free(d_tr);
  dev_free(d_tc);
  dev_free(d_rb);
  return rc;
}

namespace {

__global__ void k_store_bro(int32_t nb, const int64_t *__restrict__ start,
                            const int64_t *__restrict__ item_off, int64_t tiles,
                            int64_t *__restrict__ bro) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= nb;
       b += (int64_t)gridDim.x * blockDim.x)
    bro[b] = b < nb ? item_off[start[b]] : tiles;
}

}  // namespace

void free_tile_store(tcmis_graph *g) {
  dev_free(g->d_tbro);
  dev_free(g->d_trow);
  dev_free(g->d_tcol);
  dev_free(g->d_tbits);
  g->d_tbro = nullptr;
  g->d_trow = nullptr;
  g->store_tiles = 0;
  g->d_tcol = nullptr;
  g->d_tbits = nullptr;
  g->store_T = 0;
}

// The compact device tile store of T = 16 (32 B payload: 16 u16 rows) or
// T = 8 (8 B: 8 u8 rows) plus one int32 block column per tile and int64
// block-row offsets -- the layout SURVEY 8 "format byte budget" prices
// (36 B / 12 B per tile against the reference's 136 B).  Same tile set and
// order as tile_graph (tiling.cpp:44-84): per block row, ascending columns.
int build_tile_store(tcmis_graph *g, int T) {
  if (T != 8 && T != 16)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "the compact tile store holds T = 8 or T = 16");
  if (g->store_T == T) return 0;
  free_tile_store(g);
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const int32_t nb = (int32_t)(((int64_t)g->n + T - 1) / T);
  const int row_bytes = T / 8;
  if (int rc = dev_alloc(&g->d_tbro, (size_t)nb + 1)) return rc;
  if (nb == 0) {
    TCMIS_CUDA(cudaMemsetAsync(g->d_tbro, 0, sizeof(int64_t), st));
    if (int rc = dev_alloc(&g->d_tcol, 1)) return rc;
    if (int rc = dev_alloc(&g->d_trow, 1)) return rc;
    if (int rc = dev_alloc((uint8_t **)&g->d_tbits, 16)) return rc;
    g->store_T = T;
    return 0;
  }
  // (the solve's own tile counts, g->tile_T, are left alone: the store is
  // independent of cfg.tile_dim)
  Items it;
  if (int rc = plan_items(g, T, nb, it)) return rc;
  int32_t *scratch_rows = nullptr;
  int64_t *item_off = nullptr;
  void *tmp = nullptr;
  size_t bytes = 0;
  int64_t tiles = 0;
  int rc = dev_alloc(&scratch_rows, (size_t)nb + 1);
  if (!rc) rc = dev_alloc(&item_off, (size_t)it.n_items + 1);
  if (!rc) {
    cudaMemsetAsync(scratch_rows, 0, sizeof(int32_t) * ((size_t)nb + 1), st);
    k_tile_merge<false><<<grid_for(ctx, 32 * it.n_items, 256, 16), 256, 0, st>>>(
        g->n, T, nb, g->d_off, g->d_nbr, it.n_items, it.row, it.start, it.cnt, scratch_rows,
        nullptr, nullptr, nullptr, nullptr, row_bytes);
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, it.cnt, item_off, it.n_items, st);
    rc = dev_alloc((char **)&tmp, bytes);
  }
  if (!rc) {
    cub::DeviceScan::ExclusiveSum(tmp, bytes, it.cnt, item_off, it.n_items, st);
    int64_t last[2] = {0, 0};
    cudaMemcpyAsync(&last[0], item_off + it.n_items - 1, 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&last[1], it.cnt + it.n_items - 1, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "tile store count");
    tiles = last[0] + last[1];
  }
  if (!rc) rc = dev_alloc(&g->d_tcol, (size_t)tiles);
  if (!rc) rc = dev_alloc(&g->d_trow, (size_t)tiles);
  if (!rc) rc = dev_alloc((uint8_t **)&g->d_tbits, (size_t)tiles * T * row_bytes + 16);
  if (!rc) {
    k_tile_merge<true><<<grid_for(ctx, 32 * it.n_items, 256, 16), 256, 0, st>>>(
        g->n, T, nb, g->d_off, g->d_nbr, it.n_items, it.row, it.start, it.cnt, scratch_rows,
        item_off, g->d_trow, g->d_tcol, g->d_tbits, row_bytes);
    k_store_bro<<<grid_for(ctx, (int64_t)nb + 1, 256, 8), 256, 0, st>>>(nb, it.start, item_off,
                                                                        tiles, g->d_tbro);
    ctx->launches += 4;
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "tile store");
  }
  dev_free(scratch_rows);
  dev_free(item_off);
  dev_free(tmp);
  if (!rc) {
    g->store_T = T;
    g->store_tiles = tiles;
  }
  return rc;
}

}  // namespace tcmis_b200
