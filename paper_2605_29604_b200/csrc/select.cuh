// select.cuh -- Phase 1 (+ the push form of Phase 2) of one TC-MIS round.
//
// Reference: compute_max_np + generate_candidates (engine.cpp:86-119): v is a
// candidate iff its key exceeds every alive neighbour's key.  With key[u] = 0
// for dead u (kNoNeighborKey, priorities.hpp:57) that is "no neighbour key
// above key[v]", and a single higher neighbour settles the answer, so the
// scan exits early.  Any scan order gives the same set.
//
// Cost model: at R-MAT s22 round 1 only 9.5M of the 128M
// adjacency entries must be examined (scanning each row from its end: the
// high ids there are the low-degree, high-priority vertices), and 99.9 % of
// the vertices are settled within their last 32 entries.  The kernel is
// therefore bound by memory latency and L1 wavefronts of random key gathers,
// not by HBM bytes.  Layout of the work:
//
//  k_select       one thread per worklist vertex (coalesced offsets, the next
//                 vertex's row extent prefetched while the current one is
//                 scanned), probing the last kProbe entries, then kStep-entry
//                 chunks up to kThreadMax entries, independent loads per
//                 chunk.  A decided candidate with a short row pushes
//                 "excluded" to its neighbours itself.  A vertex still
//                 undecided after kThreadMax entries goes to a global list.
//  k_select_long  one warp per long-list vertex over the whole grid: 128
//                 entries per step (4 independent loads per lane), early exit,
//                 and the push of long candidates.
//
// Push stores are filtered through L1 (`ld.ca` of next[u] first): on R-MAT
// the neighbours of candidates concentrate on hubs -- one 128-byte line of
// next[] receives 139k of the 7.1M round-1 stores at s22 -- and unfiltered
// same-line stores serialise at one L2 slice.
#pragma once

#include "internal.cuh"

namespace tcmis_b200 {

constexpr int kSelBlock = 256;
constexpr int kProbe = 4;
constexpr int kStep = 4;
constexpr int kThreadMax = 32;

__device__ __forceinline__ void mark_candidate(int32_t v, uint8_t *next, uint8_t *segflag, int T) {
  next[v] = 1;
  if (segflag) segflag[v / T] = 1;
}

// push: every neighbour of a candidate is excluded this round (spmv.cpp:18-59
// nc > 0, engine.cpp:144-147).  Neighbours of a candidate are never
// candidates, so next[u] is 0 or 2 and the filtered store is idempotent.
__device__ __forceinline__ void exclude(uint8_t *__restrict__ next, int32_t u) {
  if (__ldca(&next[u]) != 2) next[u] = 2;
}

__device__ __forceinline__ void push_row_thread(const int32_t *__restrict__ nbr, int64_t s,
                                                int64_t e, uint8_t *__restrict__ next) {
  for (int64_t p = s; p < e; p += kStep) {
    int32_t u[kStep];
#pragma unroll
    for (int j = 0; j < kStep; ++j) u[j] = p + j < e ? __ldg(&nbr[p + j]) : -1;
#pragma unroll
    for (int j = 0; j < kStep; ++j)
      if (u[j] >= 0) exclude(next, u[j]);
  }
}

__global__ void __launch_bounds__(kSelBlock)
    k_select(int32_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
             const uint64_t *__restrict__ key, uint8_t *__restrict__ next,
             uint8_t *__restrict__ segflag, int T, int push, Ctrl *__restrict__ ctrl,
             const int32_t *__restrict__ wl0, const int32_t *__restrict__ wl1,
             int32_t *__restrict__ long_list) {
  const int round = ctrl->round;
  const int64_t cnt = round == 1 ? n : ctrl->wl_count[round & 1];
  const int32_t *wl = (round & 1) ? wl1 : wl0;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * kSelBlock;
  // software pipeline: (v, s, e, kv) of the next vertex are loaded while the
  // current row is being scanned
  int64_t i = (int64_t)blockIdx.x * kSelBlock + threadIdx.x;
  int32_t nv = 0;
  int64_t ns = 0, ne = 0;
  uint64_t nk = 0;
  if (i < cnt) {
    nv = round == 1 ? (int32_t)i : __ldg(&wl[i]);
    ns = __ldg(&off[nv]);
    ne = __ldg(&off[nv + 1]);
    nk = __ldg(&key[nv]);
  }
  // the loop bound is uniform per warp (i advances by the grid stride), so
  // the ballot below sees the whole warp
  for (int64_t wbase = i - lane; wbase < cnt; wbase += stride, i += stride) {
    const bool have = i < cnt;
    const int32_t v = nv;
    const int64_t s = ns, e = ne;
    const uint64_t kv = nk;
    const int64_t inext = i + stride;
    if (inext < cnt) {
      nv = round == 1 ? (int32_t)inext : __ldg(&wl[inext]);
      ns = __ldg(&off[nv]);
      ne = __ldg(&off[nv + 1]);
      nk = __ldg(&key[nv]);
    }
    bool defer = false;
    if (have) {
      int64_t hi = e;  // [s, hi) not yet examined
      bool blocked = false;
      int32_t u[kProbe];
#pragma unroll
      for (int j = 0; j < kProbe; ++j) u[j] = hi - 1 - j >= s ? __ldg(&nbr[hi - 1 - j]) : -1;
#pragma unroll
      for (int j = 0; j < kProbe; ++j)
        if (u[j] >= 0) blocked |= __ldg(&key[u[j]]) > kv;
      hi -= kProbe;
      while (!blocked && hi > s && e - hi < kThreadMax) {
        int32_t w[kStep];
#pragma unroll
        for (int j = 0; j < kStep; ++j) w[j] = hi - 1 - j >= s ? __ldg(&nbr[hi - 1 - j]) : -1;
#pragma unroll
        for (int j = 0; j < kStep; ++j)
          if (w[j] >= 0) blocked |= __ldg(&key[w[j]]) > kv;
        hi -= kStep;
      }
      if (!blocked) {
        if (hi <= s) {
          mark_candidate(v, next, segflag, T);
          if (push) {
            if (e - s <= kProbe) {  // the whole row is still in registers
#pragma unroll
              for (int j = 0; j < kProbe; ++j)
                if (u[j] >= 0) exclude(next, u[j]);
            } else {
              push_row_thread(nbr, s, e, next);
            }
          }
        } else {
          defer = true;
        }
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, defer);
    if (m) {
      const int leader = __ffs(m) - 1;
      int pos = 0;
      if (lane == leader) pos = atomicAdd(&ctrl->long_count, __popc(m));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (defer) long_list[pos + __popc(m & ((1u << lane) - 1u))] = v;
    }
  }
}

__global__ void __launch_bounds__(kSelBlock)
    k_select_long(const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                  const uint64_t *__restrict__ key, uint8_t *__restrict__ next,
                  uint8_t *__restrict__ segflag, int T, int push, Ctrl *__restrict__ ctrl,
                  const int32_t *__restrict__ long_list) {
  const int lane = threadIdx.x & 31;
  const int cnt = ctrl->long_count;
  for (int64_t q = ((int64_t)blockIdx.x * kSelBlock + threadIdx.x) >> 5; q < cnt;
       q += ((int64_t)gridDim.x * kSelBlock) >> 5) {
    const int32_t v = long_list[q];
    const int64_t s = __ldg(&off[v]), e = __ldg(&off[v + 1]);
    const uint64_t kv = __ldg(&key[v]);
    int64_t hi = e - kThreadMax;
    bool blocked = false;
    while (!blocked && hi > s) {
      int32_t u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t idx = hi - 1 - lane - 32 * j;
        u[j] = idx >= s ? __ldg(&nbr[idx]) : -1;
      }
      bool b = false;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (u[j] >= 0) b |= __ldg(&key[u[j]]) > kv;
      blocked = __any_sync(0xffffffffu, b);
      hi -= 128;
    }
    if (!blocked) {
      if (lane == 0) mark_candidate(v, next, segflag, T);
      if (push)
        for (int64_t idx = s + lane; idx < e; idx += 32) exclude(next, __ldg(&nbr[idx]));
    }
  }
}

}  // namespace tcmis_b200
