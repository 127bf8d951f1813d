// scan.cuh -- the per-thread row-scan engine shared by the round kernels.
//
// Both Phase 1 (candidate detection: "is any neighbour key above mine?") and
// the pull form of Phase 2 ("is any neighbour a candidate?") are an
// early-exit search over one CSR row per worklist vertex.  Profiling the
// first version (one scalar load per entry, one vertex fetch per lane at
// arbitrary times) showed the kernel bound by L1 wavefronts: every
// thread-private access of a warp touches a different 128-byte line, so each
// scalar load costs ~32 wavefronts per warp instruction.  The engine
// therefore
//   * reads the row in 16-byte aligned windows (one LDG.128 per lane per
//     step, 1-4 entries), newest entries first, so a step costs one
//     wavefront per lane for the row plus one per gathered entry;
//   * keeps every lane busy with its own vertex (no lockstep over vertices).
// A vertex whose row is not settled within kThreadMax entries is handed to a
// warp-wide kernel through a list.
#pragma once

#include "common.cuh"

namespace tcmis_b200 {

// One aligned 16-byte window of a row, read downward: entries
// [max(s, w), hi) with w = (hi - 1) & ~3, newest first in u[0..3] (unused
// slots = -1).  Returns w, i.e. the new exclusive upper end once this window
// is examined.  Falls back to scalar loads when the window would cross the
// end of the neighbour array (nnz not a multiple of 4).
__device__ __forceinline__ int64_t load_window_down(const int32_t *__restrict__ nbr, int64_t nnz,
                                                    int64_t s, int64_t hi, int32_t u[4]) {
  const int64_t w = (hi - 1) & ~(int64_t)3;
  int4 q;
  if (w + 4 <= nnz) {  // nnz < 0 flags a neighbour array that is not 16-byte aligned
    q = ld_stream(reinterpret_cast<const int4 *>(nbr + w));
  } else {
    const int64_t lim = nnz < 0 ? -nnz : nnz;
    q.x = w < lim ? __ldg(&nbr[w]) : -1;
    q.y = w + 1 < lim ? __ldg(&nbr[w + 1]) : -1;
    q.z = w + 2 < lim ? __ldg(&nbr[w + 2]) : -1;
    q.w = w + 3 < lim ? __ldg(&nbr[w + 3]) : -1;
  }
  u[0] = (w + 3 < hi && w + 3 >= s) ? q.w : -1;
  u[1] = (w + 2 < hi && w + 2 >= s) ? q.z : -1;
  u[2] = (w + 1 < hi && w + 1 >= s) ? q.y : -1;
  u[3] = (w >= s) ? q.x : -1;
  return w;
}

// Upward window for pushes: entries [p, min(e, w + 4)) with w = p & ~3.
__device__ __forceinline__ int64_t load_window_up(const int32_t *__restrict__ nbr, int64_t nnz,
                                                  int64_t p, int64_t e, int32_t u[4]) {
  const int64_t w = p & ~(int64_t)3;
  int4 q;
  if (w + 4 <= nnz) {  // nnz < 0: scalar path (unaligned neighbour array)
    q = ld_stream(reinterpret_cast<const int4 *>(nbr + w));
  } else {
    const int64_t lim = nnz < 0 ? -nnz : nnz;
    q.x = w < lim ? __ldg(&nbr[w]) : -1;
    q.y = w + 1 < lim ? __ldg(&nbr[w + 1]) : -1;
    q.z = w + 2 < lim ? __ldg(&nbr[w + 2]) : -1;
    q.w = w + 3 < lim ? __ldg(&nbr[w + 3]) : -1;
  }
  u[0] = (w >= p && w < e) ? q.x : -1;
  u[1] = (w + 1 >= p && w + 1 < e) ? q.y : -1;
  u[2] = (w + 2 >= p && w + 2 < e) ? q.z : -1;
  u[3] = (w + 3 >= p && w + 3 < e) ? q.w : -1;
  return w + 4;
}

}  // namespace tcmis_b200

namespace tcmis_b200 {

// The last <= 8 entries of a row [s, e) with two aligned 16-byte loads:
// u[0] = nbr[e-1], u[1] = nbr[e-2], ... (-1 where outside [s, e)).  Covers
// the whole row when e - s <= 5, and always at least min(5, e - s) entries.
__device__ __forceinline__ void load_tail8(const int32_t *__restrict__ nbr, int64_t nnz,
                                           int64_t s, int64_t e, int32_t u[8]) {
  const int64_t w1 = (e - 1) & ~(int64_t)3;  // window holding e-1
  const int64_t w0 = w1 - 4;
  int4 a, b;
  if (w0 >= 0 && w1 + 4 <= nnz) {
    a = ld_stream(reinterpret_cast<const int4 *>(nbr + w0));
    b = ld_stream(reinterpret_cast<const int4 *>(nbr + w1));
  } else {
    const int64_t lim = nnz < 0 ? -nnz : nnz;
    int32_t t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = (w0 + j >= 0 && w0 + j < lim) ? __ldg(&nbr[w0 + j]) : -1;
    a = make_int4(t[0], t[1], t[2], t[3]);
    b = make_int4(t[4], t[5], t[6], t[7]);
  }
  // e-1 sits at offset r of window b; u[j] = c[4 + r - j] over c = (a, b)
  const int r = (int)((e - 1) - w1);
  int32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  int32_t t[8];
  switch (r) {
    case 0: t[0] = c[4]; t[1] = c[3]; t[2] = c[2]; t[3] = c[1]; t[4] = c[0]; t[5] = t[6] = t[7] = -1; break;
    case 1: t[0] = c[5]; t[1] = c[4]; t[2] = c[3]; t[3] = c[2]; t[4] = c[1]; t[5] = c[0]; t[6] = t[7] = -1; break;
    case 2: t[0] = c[6]; t[1] = c[5]; t[2] = c[4]; t[3] = c[3]; t[4] = c[2]; t[5] = c[1]; t[6] = c[0]; t[7] = -1; break;
    default: t[0] = c[7]; t[1] = c[6]; t[2] = c[5]; t[3] = c[4]; t[4] = c[3]; t[5] = c[2]; t[6] = c[1]; t[7] = c[0]; break;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) u[j] = e - 1 - j >= s ? t[j] : -1;
}

// The last <= 4 entries of a row [s, e): u[0] = nbr[e-1], u[1] = nbr[e-2],
// ... (-1 outside [s, e)).  The aligned 16-byte window holding e-1 supplies
// r+1 of them (r = (e-1) mod 4); the window before it is loaded only when
// the row reaches back into it.  Used by the straight-line probes, which
// examine 4 entries (a smaller instruction footprint than load_tail8: the
// grid's round-1 probe is issue-bound).
__device__ __forceinline__ void load_tail4(const int32_t *__restrict__ nbr, int64_t nnz,
                                           int64_t s, int64_t e, int32_t u[4]) {
  const int64_t w1 = (e - 1) & ~(int64_t)3;
  const int r = (int)((e - 1) - w1);
  const bool need0 = r < 3 && s < w1;  // entries e-2..e-4 reach below w1
  int4 a = make_int4(-1, -1, -1, -1), b;
  if (w1 + 4 <= nnz) {
    b = ld_stream(reinterpret_cast<const int4 *>(nbr + w1));
    if (need0) a = ld_stream(reinterpret_cast<const int4 *>(nbr + w1 - 4));
  } else {
    const int64_t lim = nnz < 0 ? -nnz : nnz;
    int32_t t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t p = w1 - 4 + j;
      t[j] = (p >= 0 && p < lim) ? __ldg(&nbr[p]) : -1;
    }
    a = make_int4(t[0], t[1], t[2], t[3]);
    b = make_int4(t[4], t[5], t[6], t[7]);
  }
  const int32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  int32_t t0, t1, t2, t3;
  switch (r) {
    case 0: t0 = c[4]; t1 = c[3]; t2 = c[2]; t3 = c[1]; break;
    case 1: t0 = c[5]; t1 = c[4]; t2 = c[3]; t3 = c[2]; break;
    case 2: t0 = c[6]; t1 = c[5]; t2 = c[4]; t3 = c[3]; break;
    default: t0 = c[7]; t1 = c[6]; t2 = c[5]; t3 = c[4]; break;
  }
  u[0] = e - 1 >= s ? t0 : -1;
  u[1] = e - 2 >= s ? t1 : -1;
  u[2] = e - 3 >= s ? t2 : -1;
  u[3] = e - 4 >= s ? t3 : -1;
}

}  // namespace tcmis_b200
