// tail.cuh -- the small late rounds of a solve in ONE persistent kernel.
//
// After the first one or two rounds the alive worklist is small (R-MAT s22:
// 57k, 1.7k, 23 vertices in rounds 2-4), and four kernel launches per round
// plus the per-thread scan latency (8 dependent steps for a 32-entry row)
// cost ~50 us per round while the work is a few microseconds.  k_tail runs
// all remaining rounds with grid-wide barriers instead of kernel boundaries:
//
//   S  select: a group of kGroup lanes per worklist vertex scans its row from
//      the end, kGroup*4 entries per step (4 independent loads per lane), and
//      stops at the first higher alive neighbour (engine.cpp:86-119).  A
//      candidate is marked (next = 1, state = InMIS) and, in push mode,
//      excludes its neighbours; in pull mode non-candidates go to the check
//      list.
//   U  update (engine.cpp:121-160): push mode reads next[v] of every worklist
//      vertex; pull mode scans each check-list row for a candidate neighbour.
//      Survivors form the next worklist.
//   F  one thread publishes the round's IterationStats exactly like
//      k_round_end and advances the round.
//
// The rounds stay bulk-synchronous (barriers between S, U and F), so round
// count and every statistic equal the reference's.  Launched cooperatively,
// which guarantees that all blocks are co-resident for the barriers.  Data
// written by other blocks in an earlier phase is read with ld.global.cg (L2),
// never through the SM's non-coherent L1.
#pragma once

#include "common.cuh"

namespace tcmis_b200 {

constexpr int kGroup = 8;             // lanes per vertex in the tail kernel
#ifndef TCMIS_TAIL_UNROLL
#define TCMIS_TAIL_UNROLL 16
#endif
constexpr int kTU = TCMIS_TAIL_UNROLL;  // independent loads per lane per step
constexpr int kTailBlock = 1024;  // one block per SM: 148 arrivals per barrier

struct TailArgs {
  const int64_t *off;
  const int32_t *nbr;
  uint32_t *prio;
  uint16_t *q;
  uint8_t *next;
  uint8_t *state;
  uint8_t *segflag;         // byte flags (seg_mode 2) -- also mode 1 sanity
  uint32_t *segmark;        // seg_mode 1: round that last counted the segment
  const int32_t *rowtiles;
  int32_t nseg;
  int64_t total_tiles;
  int seg_mode;
  int T;
  int push;
  int fresh;
  uint64_t seed;
  Ctrl *ctrl;
  int32_t *wl0, *wl1;
  int32_t *check;
  DevRound *rounds;
  unsigned *bar;            // [0] arrivals, [1] generation
};

__device__ __forceinline__ void grid_barrier(unsigned *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned *gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// the lanes of one group stay converged (same vertex, same trip count);
// different groups of a warp may diverge, so the vote uses the group's mask
__device__ __forceinline__ unsigned group_any(bool b, unsigned gmask) {
  return __ballot_sync(gmask, b);
}

#ifndef TCMIS_TAIL_LONG
#define TCMIS_TAIL_LONG 512
#endif
#ifndef TCMIS_TAIL_SMALL
#define TCMIS_TAIL_SMALL 128
#endif
constexpr int64_t kTailLong = TCMIS_TAIL_LONG;    // rows above this are scanned by a whole block
constexpr int kTailLongCap = 256;                 // per-block list of such rows per phase
constexpr int64_t kTailSmall = TCMIS_TAIL_SMALL;  // rounds at or below this run in block 0 alone

// A candidate of the tail (mark_candidate + the tile counter of seg_mode 1:
// exactly one candidate of the round counts its block column).
__device__ __forceinline__ void tail_candidate(const TailArgs &a, int32_t v, int round,
                                               unsigned long long &sel,
                                               unsigned long long &ev) {
  a.next[v] = 1;
  a.state[v] = TCMIS_IN_MIS;
  ++sel;
  const int32_t sb = v / a.T;
  if (a.seg_mode == 2) {
    a.segflag[sb] = 1;
  } else if (a.seg_mode == 1) {
    if (atomicMax(&a.segmark[sb], (unsigned)round) < (unsigned)round)
      ev += (unsigned long long)a.rowtiles[sb];
  }
}

// Block-wide scan of one long row [s, e) from its end, kTailBlock * 4 entries
// per step, early exit; mode 0: "an alive neighbour with a higher key"
// (Phase 1), mode 1: "a candidate neighbour" (Phase 2, pull).
__device__ __forceinline__ bool block_scan_any(const TailArgs &a, int64_t s, int64_t e, int mode,
                                               uint32_t qv, uint64_t kv) {
  bool any = false;
  for (int64_t hi = e; hi > s && !any; hi -= 4 * kTailBlock) {
    int32_t u[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t idx = hi - 1 - threadIdx.x - (int64_t)kTailBlock * j;
      u[j] = idx >= s ? __ldg(&a.nbr[idx]) : -1;
    }
    bool b = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (u[j] < 0) continue;
      if (mode == 0) {
        const uint32_t qu = __ldcg(&a.q[u[j]]);
        b |= qu != qv ? qu > qv : key_of(__ldcg(&a.prio[u[j]]), u[j]) > kv;
      } else {
        b |= __ldcg(&a.next[u[j]]) == 1;
      }
    }
    any = __syncthreads_or(b) != 0;
  }
  return any;
}

// A long row is handed to the block (list in shared memory, capacity
// kTailLongCap; on overflow the group scans it itself).  Returns whether the
// group should skip the row -- the same answer for all lanes of the group.
__device__ __forceinline__ bool defer_long(int32_t v, int32_t *s_long, int *s_nlong, int gl,
                                           unsigned gmask, int lane) {
  int listed = 0;
  if (gl == 0) {
    const int k = atomicAdd(s_nlong, 1);
    if (k < kTailLongCap) {
      s_long[k] = v;
      listed = 1;
    }
  }
  return __shfl_sync(gmask, listed, lane & ~(kGroup - 1)) != 0;
}

// One round of the tail by the groups [gfirst, gfirst + k*gstride) of the
// participating blocks; `grid` selects grid-wide barriers (all blocks) or
// block barriers (block 0 alone, the small rounds).
__device__ void tail_round(const TailArgs &a, int round, int64_t cnt, int64_t gfirst,
                           int64_t gstride, int64_t tfirst, int64_t tstride, bool grid,
                           int32_t *s_long, int *s_nlong) {
  Ctrl *ctrl = a.ctrl;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (kGroup - 1);
  const unsigned gmask = ((1u << kGroup) - 1u) << (lane & ~(kGroup - 1));
  constexpr int kW = kGroup * kTU;  // entries per group step: short rows settle in one step
  int *check_count = &ctrl->tail_check[round & 1];
  const int32_t *in = (round & 1) ? a.wl1 : a.wl0;
  int32_t *out = (round & 1) ? a.wl0 : a.wl1;
  int *tail = &ctrl->wl_count[(round + 1) & 1];
  const uint64_t fresh_m = a.fresh ? mix64(combine_seed(a.seed, (uint64_t)round + 1)) : 0;
  unsigned long long sel = 0, rem = 0, ev = 0;
  // ---- S: candidate detection (+ push)
  for (int64_t q = gfirst; q < cnt; q += gstride) {
    const int32_t v = __ldcg(&in[q]);
    const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
    if (e - s > kTailLong && defer_long(v, s_long, s_nlong, gl, gmask, lane)) continue;
    const uint64_t kv = key_of(__ldcg(&a.prio[v]), v);
    const uint32_t qv = __ldcg(&a.q[v]);
    bool blocked = false;
    for (int64_t hi = e; hi > s && !blocked; hi -= kW) {
      int32_t u[kTU];
#pragma unroll
      for (int j = 0; j < kTU; ++j) {
        const int64_t idx = hi - 1 - gl - kGroup * j;
        u[j] = idx >= s ? __ldg(&a.nbr[idx]) : -1;
      }
      bool b = false;
#pragma unroll
      for (int j = 0; j < kTU; ++j)
        if (u[j] >= 0) {
          const uint32_t qu = __ldcg(&a.q[u[j]]);
          b |= qu != qv ? qu > qv : key_of(__ldcg(&a.prio[u[j]]), u[j]) > kv;
        }
      blocked = group_any(b, gmask) != 0;
    }
    if (!blocked) {
      if (gl == 0) tail_candidate(a, v, round, sel, ev);
      if (a.push)
        for (int64_t idx = s + gl; idx < e; idx += kGroup) a.next[__ldg(&a.nbr[idx])] = 2;
    } else if (!a.push && gl == 0) {
      a.check[atomicAdd(check_count, 1)] = v;
    }
  }
  __syncthreads();
  const int nlong = min(*s_nlong, kTailLongCap);
  for (int k = 0; k < nlong; ++k) {
    const int32_t v = s_long[k];
    const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
    const bool blocked = block_scan_any(a, s, e, 0, __ldcg(&a.q[v]), key_of(__ldcg(&a.prio[v]), v));
    if (!blocked) {
      if (threadIdx.x == 0) tail_candidate(a, v, round, sel, ev);
      if (a.push)
        for (int64_t idx = s + threadIdx.x; idx < e; idx += kTailBlock)
          a.next[__ldg(&a.nbr[idx])] = 2;
    } else if (!a.push && threadIdx.x == 0) {
      a.check[atomicAdd(check_count, 1)] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *s_nlong = 0;
  if (grid) grid_barrier(a.bar);
  else __syncthreads();

  // ---- U: exclusion (pull) + state update + compaction
  if (a.push) {
    for (int64_t q = tfirst; q < cnt; q += tstride) {
      const int32_t v = __ldcg(&in[q]);
      const uint8_t d = __ldcg(&a.next[v]);
      if (d == 2) {
        mark_removed(v, a.state, a.q);
        ++rem;
      } else if (d == 0) {
        if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m);
        out[atomicAdd(tail, 1)] = v;
      }
    }
  } else {
    const int64_t nc = *(volatile int *)check_count;
    for (int64_t q = gfirst; q < nc; q += gstride) {
      const int32_t v = __ldcg(&a.check[q]);
      const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
      if (e - s > kTailLong && defer_long(v, s_long, s_nlong, gl, gmask, lane)) continue;
      bool hit = false;
      for (int64_t hi = e; hi > s && !hit; hi -= kW) {
        int32_t u[kTU];
#pragma unroll
        for (int j = 0; j < kTU; ++j) {
          const int64_t idx = hi - 1 - gl - kGroup * j;
          u[j] = idx >= s ? __ldg(&a.nbr[idx]) : -1;
        }
        bool b = false;
#pragma unroll
        for (int j = 0; j < kTU; ++j)
          if (u[j] >= 0) b |= __ldcg(&a.next[u[j]]) == 1;
        hit = group_any(b, gmask) != 0;
      }
      if (gl == 0) {
        if (hit) {
          mark_removed(v, a.state, a.q);
          ++rem;
        } else {
          if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m);
          out[atomicAdd(tail, 1)] = v;
        }
      }
    }
  }
  if (!a.push) {
    __syncthreads();
    const int nl = min(*s_nlong, kTailLongCap);
    for (int k = 0; k < nl; ++k) {
      const int32_t v = s_long[k];
      const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
      const bool hit = block_scan_any(a, s, e, 1, 0, 0);
      if (threadIdx.x == 0) {
        if (hit) {
          mark_removed(v, a.state, a.q);
          ++rem;
        } else {
          if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m);
          out[atomicAdd(tail, 1)] = v;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) *s_nlong = 0;
  }
  block_add3(sel, rem, ev, ctrl);
  if (grid) grid_barrier(a.bar);
  else __syncthreads();
}
// The persistent tail: every block walks the rounds in lockstep, so the
// round number is local.  Two barriers per round (after S, after U).  Block
// 0 publishes round r-1's IterationStats at the start of round r and clears
// the counters; nobody else touches them before the next barrier.  The pull
// check list is double-buffered by round parity for the same reason.  Once a
// round has <= kTailSmall alive vertices, the other blocks leave and block 0
// finishes alone with block barriers (a grid barrier costs ~2 us, a round of
// a few hundred vertices ~3 us).
__global__ void __launch_bounds__(kTailBlock) k_tail(TailArgs a) {
  __shared__ int32_t s_long[kTailLongCap];
  __shared__ int s_nlong;
  Ctrl *ctrl = a.ctrl;
  if (threadIdx.x == 0) s_nlong = 0;
  __syncthreads();
  bool grid = true;
  int round = *(volatile int *)&ctrl->round;
  for (;; ++round) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && round > *(volatile int *)&ctrl->round) {
      volatile Ctrl *vc = ctrl;
      const int pr = round - 1;
      const int32_t alive = vc->wl_count[round & 1];
      DevRound r;
      r.sel = vc->sel;
      r.rem = vc->rem;
      r.alive = (unsigned long long)alive;
      r.eval = a.seg_mode == 1 ? vc->eval : 0;
      r.skip = a.seg_mode == 1 ? (unsigned long long)a.total_tiles - vc->eval : 0;
      a.rounds[(pr - 1) % vc->max_rounds] = r;
      if (pr > vc->max_rounds) vc->overflow = 1;
      vc->alive = alive;
      vc->sel = 0;
      vc->rem = 0;
      vc->eval = 0;
      vc->wl_count[pr & 1] = 0;       // this round's output slot (U, after a barrier)
      vc->tail_check[pr & 1] = 0;     // next round's check list
      vc->round = round;
      __threadfence();
    }
    if (!grid) __syncthreads();
    const int64_t cnt = *(volatile int *)&ctrl->wl_count[round & 1];
    if (cnt == 0) break;  // nothing alive (alive == 0 after the last round)
    if (grid && cnt <= kTailSmall) {
      if (blockIdx.x != 0) return;
      grid = false;
    }
    if (grid) {
      const int64_t gid = ((int64_t)blockIdx.x * kTailBlock + threadIdx.x) / kGroup;
      const int64_t ngroups = ((int64_t)gridDim.x * kTailBlock) / kGroup;
      tail_round(a, round, cnt, gid, ngroups, (int64_t)blockIdx.x * kTailBlock + threadIdx.x,
                 (int64_t)gridDim.x * kTailBlock, true, s_long, &s_nlong);
    } else {
      tail_round(a, round, cnt, threadIdx.x / kGroup, kTailBlock / kGroup, threadIdx.x,
                 kTailBlock, false, s_long, &s_nlong);
    }
  }
}

}  // namespace tcmis_b200
