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
// high ids there are the low-degree, high-priority vertices), and 84 % of the
// vertices are settled by their last 4 entries.  The kernels are bound by
// memory latency of the random q gathers, not by HBM bytes.  Layout:
//
//  k_probe_select one thread per worklist vertex, straight-line: the last 4
//                 entries; settles short rows and blocked vertices.
//  k_select       the probe's undecided rows, one lane per row as a per-lane
//                 state machine: every loop iteration each lane scans the
//                 next 8 entries of its row (two 16-byte windows, from the
//                 end) or fetches its next row, so a lane never idles behind
//                 the slowest row of its warp.  A row unsettled after
//                 kThreadMax entries goes to a list for k_select_long.
//  k_select_long  one warp per listed row: 256 entries per step (8 loads per
//                 lane), early exit; rows beyond kBlockRow entries block-wide.
//
// Outputs: candidates get next = 1 and state = InMIS; in push mode their
// neighbours get next = 2; in pull mode nothing else (the pull kernels walk
// the same worklist and test state == Alive, update.cuh).
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace tcmis_b200 {

#ifndef TCMIS_SEL_MINB
#define TCMIS_SEL_MINB 8
#endif
#ifndef TCMIS_PROBE_MINB
#define TCMIS_PROBE_MINB 8  // resident blocks of the probes (k_probe_select, k_probe_pull)
#endif


struct SelectArgs {
  int32_t n1;              // round-1 list length (non-isolated vertices)
  const int32_t *nz;       // round-1 list
  int nz_identity;         // no isolated vertices: the round-1 list is 0..n-1
  const int64_t *off;
  const int32_t *nbr;
  int64_t vnnz;            // nnz, negated if nbr is not 16-byte aligned (scan.cuh)
  const uint32_t *prio;
  const uint16_t *q;        // q_of(p), 0 once removed (common.cuh)
  uint8_t *next;
  uint8_t *state;
  uint8_t *segflag;        // null: no tile counters
  int T;
  int push;                // 1: push exclusion (candidates scatter next = 2)
  Ctrl *ctrl;
  const int32_t *wl0, *wl1;
  int32_t *long_list;      // rows outliving the thread probe (ctrl->long_count)
  int32_t *vlong;          // ... longer than kBlockRow (ctrl->sel_vlong)
  int32_t *undecided;      // rows the probe could not settle (ctrl->sel_undec)
  Publish pub;             // multi-GPU: this round's candidates of the own range
  DevRound *rounds;        // Phase 1 start stamp (null: none)
  const int32_t *perm;     // solve id -> caller id (relabeled graphs), else null
  uint8_t *mis_o;          // ... and the membership in the caller's order
  int32_t tile_gate;       // > 0: rounds starting with >= this many alive vertices run
                           // Phase 1 as A-up tiles (k_tile_mark), these kernels idle
  const int2 *cb;          // degree-class bounds (common.cuh class_bounds), or null
  // round 1 on a degree-ordered graph: k_prio_settle (solver.cu) decided
  // every vertex it could from the class bounds and listed the rest in wl1
  // (ctrl->r1_sel_left) for the probe.  Null: off.
  const int32_t *r1_max;
  const uint16_t *r1_cls;
  const int2 *cbc;
};

// kU row entries of v against the class bounds: in round 1 (everybody alive)
// an entry >= hi blocks without a gather; entries < lo never block and are
// not gathered; the rest take the key comparison.  `below`: an examined
// entry lies under lo, so the rest of the row (smaller ids) cannot block.
template <int kU>
__device__ __forceinline__ bool blocks_row(const SelectArgs &a, const int32_t *u, int2 cb,
                                           bool all_alive, uint32_t qv, int32_t v, bool &below) {
  bool blocked = false;
  below = false;
#pragma unroll
  for (int j = 0; j < kU; ++j) below |= u[j] >= 0 && u[j] < cb.x;
  if (all_alive) {
#pragma unroll
    for (int j = 0; j < kU; ++j) blocked |= u[j] >= cb.y;
  }
  if (!blocked) {
#pragma unroll
    for (int j = 0; j < kU; ++j)
      if (u[j] >= cb.x) blocked |= blocks(a.q, a.prio, u[j], qv, v, a.perm);
  }
  return blocked;
}

// push: every neighbour of a candidate is excluded this round (spmv.cpp:18-59
// nc > 0, engine.cpp:144-147).  Neighbours of a candidate are never
// candidates, so the store is idempotent.
__device__ __forceinline__ void exclude(uint8_t *__restrict__ next, int32_t u) { next[u] = 2; }

constexpr int kProbeK = 4;  // row entries the straight-line probe examines

// Probe: one thread per worklist vertex, straight-line code in warp lockstep
// (no per-lane loop): coalesced row extents and own key, the last <= 8 row
// entries with two aligned 16-byte loads, keys of the last kProbeK gathered.
// This settles 84 % of R-MAT s22's round-1 vertices and every vertex of
// rows <= kProbeK (the whole grid, most of the RGG).
__global__ void __launch_bounds__(kBlock, TCMIS_PROBE_MINB) k_probe_select(SelectArgs a) {
  pdl_entry();
  if (a.tile_gate && a.ctrl->alive >= a.tile_gate) return;  // a tile round (tile_cand.cu)
  __shared__ int32_t s_und[kBlock / 32][64];
  Ctrl *ctrl = a.ctrl;
  const int round = ctrl->round;
  stamp_phase(a.rounds, ctrl, round, 0, 0);
  // round 1 visits only the non-isolated vertices (k_priorities already made
  // the isolated ones candidates), and on a degree order only those that
  // k_prio_settle (solver.cu) left undecided
  const bool r1s = round == 1 && a.r1_max;
  const int64_t cnt = r1s ? ctrl->r1_sel_left : round == 1 ? a.n1 : ctrl->wl_count[round & 1];
  if ((int64_t)blockIdx.x * kBlock >= cnt) return;
  const int32_t *wl = r1s ? a.wl1 : round == 1 ? a.nz : ((round & 1) ? a.wl1 : a.wl0);
  const int32_t *__restrict__ nbr = a.nbr;
  const uint16_t *__restrict__ q = a.q;
  const int lane = threadIdx.x & 31;
  WarpOut und{s_und[threadIdx.x >> 5], 0};
  unsigned long long sel = 0;
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  for (int64_t wb = (int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31); wb < cnt; wb += stride) {
    const int64_t i = wb + lane;
    bool undecided = false, pub = false;
    int32_t v = 0;
    if (i < cnt) {
      v = (round == 1 && a.nz_identity && !r1s) ? (int32_t)i : __ldg(&wl[i]);
      {
        const int64_t s = ld_stream(&a.off[v]), e = ld_stream(&a.off[v + 1]);
        const uint32_t qv = __ldg(&q[v]);
        const int2 cb = class_bounds(a.cb, e - s);
        int32_t u[4];
        load_tail4(nbr, a.vnnz, s, e, u);
        bool below;
        const bool blocked = blocks_row<kProbeK>(a, u, cb, round == 1, qv, v, below);
        if (blocked) {
          // a non-candidate: the pull exclusion finds it on the worklist
        } else if (e - s <= kProbeK || (below && !a.push)) {  // push: the whole row in k_select
          mark_candidate(v, a.next, a.state, a.segflag, a.T, a.perm, a.mis_o);
          pub = true;
          ++sel;
          if (a.push) {
#pragma unroll
            for (int j = 0; j < kProbeK; ++j)
              if (u[j] >= 0) exclude(a.next, u[j]);
          }
        } else {
          undecided = true;
        }
      }
    }
    publish_warp(a.pub, v, pub);
    warp_emit(und, undecided, v, a.undecided, &ctrl->sel_undec);
  }
  warp_flush(und, a.undecided, &ctrl->sel_undec);
  block_add3(sel, 0, 0, ctrl);
}

// Engine: the probe's undecided rows, one lane per row as a per-lane state
// machine (scan down in 16-byte windows from e - kProbeK; push up), so a
// lane never idles behind another lane's longer row.
// kWin 16-byte windows per step.  Four on graphs whose q vector outgrows a
// good part of L2 (more gathers in flight per lane against the misses: R-MAT
// s26 round 1 1.07 -> 0.93 ms); two elsewhere (s22: 57 / 55 / 61 us for two /
// three / four, and the pull engine is best at two everywhere).
constexpr int32_t kSelWideN = 1 << 25;
template <int kWin>
__global__ void __launch_bounds__(kBlock, TCMIS_SEL_MINB) k_select(SelectArgs a) {
  pdl_entry();
  if (a.tile_gate && a.ctrl->alive >= a.tile_gate) return;  // a tile round (tile_cand.cu)
  Ctrl *ctrl = a.ctrl;
  const int64_t cnt = ctrl->sel_undec;
  if ((int64_t)blockIdx.x * kBlock >= cnt) return;
  const int32_t *__restrict__ nbr = a.nbr;
  const uint16_t *__restrict__ q = a.q;
  const bool all_alive = ctrl->round == 1;
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  unsigned long long sel = 0;
  int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x - stride;
  int mode = kFetch;
  int32_t v = 0;
  int64_t s = 0, e = 0, hi = 0;
  uint32_t qv = 0;
  int2 cb = make_int2(0, 0);
  auto fetch = [&]() {
    i += stride;
    if (i < cnt) {
      v = __ldg(&a.undecided[i]);
      s = __ldg(&a.off[v]);
      e = __ldg(&a.off[v + 1]);
      qv = __ldg(&q[v]);
      cb = class_bounds(a.cb, e - s);
      hi = e - kProbeK;  // the probe examined the last kProbeK entries
      mode = kScan;
    } else {
      mode = kDone;
    }
  };
  fetch();
  while (__any_sync(0xffffffffu, mode != kDone)) {
    bool defer = false, pub = false;
    if (mode == kScan) {
      // kWin 16-byte windows per step: 4 kWin entries and their q gathers in flight
      constexpr int kU = 4 * kWin;
      int32_t u[kU];
      int64_t w = load_window_down(nbr, a.vnnz, s, hi, u);
#pragma unroll
      for (int k = 1; k < kWin; ++k) {
        if (w > s) {
          w = load_window_down(nbr, a.vnnz, s, w, u + 4 * k);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) u[4 * k + j] = -1;
        }
      }
      bool below;
      const bool blocked = blocks_row<kU>(a, u, cb, all_alive, qv, v, below);
      hi = w;
      if (blocked) {
        mode = kFetch;
      } else if (hi <= s || below) {
        mark_candidate(v, a.next, a.state, a.segflag, a.T, a.perm, a.mis_o);
        pub = true;
        ++sel;
        mode = a.push ? kPush : kFetch;
        hi = s;  // push cursor runs upward from s
      } else if (e - hi >= kThreadMax) {
        defer = true;
        mode = kFetch;
      }
    } else if (mode == kPush) {
      int32_t u[4];
      const int64_t p = load_window_up(nbr, a.vnnz, hi, e, u);
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (u[j] >= 0) exclude(a.next, u[j]);
      hi = p;
      if (hi >= e) mode = kFetch;
    }
    publish_warp(a.pub, v, pub);
    const bool vl = defer && e - s > kBlockRow;
    warp_append(defer && !vl, v, a.long_list, &ctrl->long_count);
    warp_append(vl, v, a.vlong, &ctrl->sel_vlong);
    if (mode == kFetch) fetch();
  }
  block_add3(sel, 0, 0, ctrl);
}

__global__ void __launch_bounds__(kBlock) k_select_long(SelectArgs a) {
  pdl_entry();
  if (a.tile_gate && a.ctrl->alive >= a.tile_gate) return;  // a tile round (tile_cand.cu)
  Ctrl *ctrl = a.ctrl;
  const int cnt = ctrl->long_count, nvl = ctrl->sel_vlong;
  if ((int64_t)blockIdx.x * (kBlock / 32) >= cnt && blockIdx.x >= nvl) return;
  const int lane = threadIdx.x & 31;
  const int32_t *__restrict__ nbr = a.nbr;
  const bool all_alive = ctrl->round == 1;
  unsigned long long sel = 0;
  // one warp per row; rows longer than kBlockRow by the whole block below
  for (int64_t q = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5; q < cnt;
       q += ((int64_t)gridDim.x * kBlock) >> 5) {
    const int32_t v = a.long_list[q];
    const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
    const uint32_t qv = __ldg(&a.q[v]);
    const int2 cb = class_bounds(a.cb, e - s);
    // the thread stage examined at least the last kThreadMax - 3 entries (its
    // first window may be short); rescanning an entry is harmless
    int64_t hi = e - (kThreadMax - 3);
    bool blocked = false, done = false;
    while (!blocked && !done && hi > s) {
      int32_t u[kWarpU];
#pragma unroll
      for (int j = 0; j < kWarpU; ++j) {
        const int64_t idx = hi - 1 - lane - 32 * j;
        u[j] = idx >= s ? ld_stream(&nbr[idx]) : -1;
      }
      bool below;
      const bool b = blocks_row<kWarpU>(a, u, cb, all_alive, qv, v, below);
      blocked = __any_sync(0xffffffffu, b);
      done = __any_sync(0xffffffffu, below);
      hi -= 32 * kWarpU;
    }
    if (!blocked) {
      if (lane == 0) {
        mark_candidate(v, a.next, a.state, a.segflag, a.T, a.perm, a.mis_o);
        publish(a.pub, v);
        ++sel;
      }
      if (a.push)
        for (int64_t idx = s + lane; idx < e; idx += 32) exclude(a.next, __ldg(&nbr[idx]));
    }
  }
  for (int64_t q = blockIdx.x; q < nvl; q += gridDim.x) {
    const int32_t v = a.vlong[q];
    const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
    const uint32_t qv = __ldg(&a.q[v]);
    const int2 cb = class_bounds(a.cb, e - s);
    int64_t hi = e - (kThreadMax - 3);
    bool blocked = false, done = false;
    while (!blocked && !done && hi > s) {
      int32_t u[kWarpU];
#pragma unroll
      for (int j = 0; j < kWarpU; ++j) {
        const int64_t idx = hi - 1 - threadIdx.x - (int64_t)kBlock * j;
        u[j] = idx >= s ? ld_stream(&nbr[idx]) : -1;
      }
      bool below;
      const bool b = blocks_row<kWarpU>(a, u, cb, all_alive, qv, v, below);
      blocked = __syncthreads_or(b) != 0;
      done = __syncthreads_or(below) != 0;
      hi -= (int64_t)kBlock * kWarpU;
    }
    if (!blocked) {
      if (threadIdx.x == 0) {
        mark_candidate(v, a.next, a.state, a.segflag, a.T, a.perm, a.mis_o);
        publish(a.pub, v);
        ++sel;
      }
      if (a.push)
        for (int64_t idx = s + threadIdx.x; idx < e; idx += kBlock) exclude(a.next, __ldg(&nbr[idx]));
    }
  }
  block_add3(sel, 0, 0, ctrl);
}

}  // namespace tcmis_b200
