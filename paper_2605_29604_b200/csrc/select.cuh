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
constexpr int kStep = 4;
constexpr int kThreadMax = 32;

__device__ __forceinline__ void mark_candidate(int32_t v, uint8_t *next, uint8_t *segflag, int T) {
  next[v] = 1;
  if (segflag) segflag[v / T] = 1;
}

// push: every neighbour of a candidate is excluded this round (spmv.cpp:18-59
// nc > 0, engine.cpp:144-147).  Neighbours of a candidate are never
// candidates, so next[u] is 0 or 2 and the filtered store is idempotent.
#ifndef TCMIS_PUSH_FILTER
#define TCMIS_PUSH_FILTER 2  // 0 none, 1 ld.ca of next[u], 2 per-block shared-memory tag table
#endif
#ifndef TCMIS_FILTER_LOG
#define TCMIS_FILTER_LOG 11
#endif
constexpr int kFilterLog = TCMIS_FILTER_LOG;
constexpr int kFilterSlots = 1 << kFilterLog;

struct PushFilter {
  int32_t *tags;  // shared memory, kFilterSlots entries, -1 = empty
};

__device__ __forceinline__ void exclude(uint8_t *__restrict__ next, int32_t u, PushFilter f) {
#if TCMIS_PUSH_FILTER == 1
  if (__ldca(&next[u]) != 2) next[u] = 2;
#elif TCMIS_PUSH_FILTER == 2
  // hub neighbours are pushed by thousands of candidates; a per-block
  // direct-mapped table of recent targets removes the repeats (a miss or a
  // racing duplicate only costs one redundant, idempotent store)
  // hashed: R-MAT hubs are ids with many zero low bits and would all
  // collide in a table indexed by the low bits
  int32_t *slot = &f.tags[((uint32_t)u * 2654435761u) >> (32 - kFilterLog)];
  if (*slot != u) {
    *slot = u;
    next[u] = 2;
  }
#else
  next[u] = 2;
#endif
}

__device__ __forceinline__ void push_row_thread(const int32_t *__restrict__ nbr, int64_t s,
                                                int64_t e, uint8_t *__restrict__ next,
                                                PushFilter f) {
  for (int64_t p = s; p < e; p += kStep) {
    int32_t u[kStep];
#pragma unroll
    for (int j = 0; j < kStep; ++j) u[j] = p + j < e ? __ldg(&nbr[p + j]) : -1;
#pragma unroll
    for (int j = 0; j < kStep; ++j)
      if (u[j] >= 0) exclude(next, u[j], f);
  }
}

#ifndef TCMIS_SEL_MINB
#define TCMIS_SEL_MINB 8
#endif

// Per-thread state machine: every loop iteration each lane does ONE unit of
// work -- fetch a vertex and probe the last kStep entries of its row, probe
// the next kStep entries, or push to kStep neighbours -- so lanes never wait
// for the slowest vertex of their warp (the SIMT lockstep of a plain
// per-vertex loop cost ~4x at R-MAT s22, where a few candidates per warp have
// 20-50-entry rows to scan and push).
enum : int { kFetch = 0, kScan = 1, kPush = 2, kDone = 3 };

__global__ void __launch_bounds__(kSelBlock, TCMIS_SEL_MINB)
    k_select(int32_t n1, const int32_t *__restrict__ nz, const int64_t *__restrict__ off,
             const int32_t *__restrict__ nbr,
             const uint64_t *__restrict__ key, uint8_t *__restrict__ next,
             uint8_t *__restrict__ segflag, int T, int push, Ctrl *__restrict__ ctrl,
             const int32_t *__restrict__ wl0, const int32_t *__restrict__ wl1,
             int32_t *__restrict__ long_list) {
  const int round = ctrl->round;
  // round 1 visits only the non-isolated vertices (k_priorities already
  // marked the isolated ones as candidates)
  const int64_t cnt = round == 1 ? n1 : ctrl->wl_count[round & 1];
  const int32_t *wl = round == 1 ? nz : ((round & 1) ? wl1 : wl0);
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * kSelBlock;
  __shared__ int32_t s_tags[TCMIS_PUSH_FILTER == 2 ? kFilterSlots : 1];
  PushFilter f{s_tags};
  if (TCMIS_PUSH_FILTER == 2) {
    for (int t = threadIdx.x; t < kFilterSlots; t += kSelBlock) s_tags[t] = -1;
    __syncthreads();
  }
  int64_t i = (int64_t)blockIdx.x * kSelBlock + threadIdx.x - stride;
  int mode = kFetch;
  int32_t v = 0;
  int64_t s = 0, e = 0, hi = 0;
  uint64_t kv = 0;
  // fetch: the next vertex of this thread's strided sequence; issued at the
  // end of an iteration so its loads overlap the loop back-edge
  auto fetch = [&]() {
    i += stride;
    if (i < cnt) {
      v = __ldg(&wl[i]);
      s = __ldg(&off[v]);
      e = __ldg(&off[v + 1]);
      kv = __ldg(&key[v]);
      hi = e;
      mode = kScan;
    } else {
      mode = kDone;
    }
  };
  fetch();
  while (__any_sync(0xffffffffu, mode != kDone)) {
    bool defer = false;
    if (mode == kScan) {
      int32_t u[kStep];
#pragma unroll
      for (int j = 0; j < kStep; ++j) u[j] = hi - 1 - j >= s ? __ldg(&nbr[hi - 1 - j]) : -1;
      bool blocked = false;
#pragma unroll
      for (int j = 0; j < kStep; ++j)
        if (u[j] >= 0) blocked |= __ldg(&key[u[j]]) > kv;
      hi -= kStep;
      if (blocked) {
        mode = kFetch;
      } else if (hi <= s) {
        mark_candidate(v, next, segflag, T);
        if (push && e - s <= kStep) {  // the whole row is still in registers
#pragma unroll
          for (int j = 0; j < kStep; ++j)
            if (u[j] >= 0) exclude(next, u[j], f);
          mode = kFetch;
        } else {
          mode = push ? kPush : kFetch;
          hi = s;  // push cursor runs upward from s
        }
      } else if (e - hi >= kThreadMax) {
        defer = true;
        mode = kFetch;
      }
    } else if (mode == kPush) {
      int32_t u[kStep];
#pragma unroll
      for (int j = 0; j < kStep; ++j) u[j] = hi + j < e ? __ldg(&nbr[hi + j]) : -1;
#pragma unroll
      for (int j = 0; j < kStep; ++j)
        if (u[j] >= 0) exclude(next, u[j], f);
      hi += kStep;
      if (hi >= e) mode = kFetch;
    }
    const unsigned m = __ballot_sync(0xffffffffu, defer);
    if (m) {
      const int leader = __ffs(m) - 1;
      int pos = 0;
      if (lane == leader) pos = atomicAdd(&ctrl->long_count, __popc(m));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (defer) long_list[pos + __popc(m & ((1u << lane) - 1u))] = v;
    }
    if (mode == kFetch) fetch();
  }
}

__global__ void __launch_bounds__(kSelBlock)
    k_select_long(const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                  const uint64_t *__restrict__ key, uint8_t *__restrict__ next,
                  uint8_t *__restrict__ segflag, int T, int push, Ctrl *__restrict__ ctrl,
                  const int32_t *__restrict__ long_list) {
  const int lane = threadIdx.x & 31;
  const int cnt = ctrl->long_count;
  if (cnt == 0) return;
  __shared__ int32_t s_tags[TCMIS_PUSH_FILTER == 2 ? kFilterSlots : 1];
  PushFilter f{s_tags};
  if (TCMIS_PUSH_FILTER == 2) {
    for (int t = threadIdx.x; t < kFilterSlots; t += kSelBlock) s_tags[t] = -1;
    __syncthreads();
  }

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
        for (int64_t idx = s + lane; idx < e; idx += 32) exclude(next, __ldg(&nbr[idx]), f);
    }
  }
}

}  // namespace tcmis_b200
