// update.cuh -- Phase 2 (pull form) + Phase 3 + worklist compaction + the
// round's statistics.
//
// Reference: tiled_spmv's nc = A * c restricted to "nc > 0" (spmv.cpp:18-59)
// and phase3_update (engine.cpp:121-160): a candidate joins the MIS; an alive
// non-candidate with a candidate neighbour is removed; every other alive
// vertex survives into the next round.
//
// The decision array `next` is never reset inside a solve: next[v] == 1 marks
// the round in which v became a candidate and stays 1 once v is InMIS.  An
// alive vertex never sees a neighbour with a stale 1 (that neighbour's round
// removed all of its neighbours), so "next[u] == 1" is exactly "u is a
// candidate of this round" for every neighbour u of an alive vertex.
//
// Two exclusion forms:
//   push  k_select already wrote next[u] = 2 for every neighbour of every
//         candidate; k_update is a coalesced striped pass over the worklist
//         (block-scan compaction, one atomic per 2048 vertices).
//   pull  k_probe_pull walks the round's worklist again; every vertex still
//         Alive after the select kernels is a non-candidate, and its row is
//         scanned from the end for next[u] == 1, stopping at the first hit
//         (R-MAT s22 round 1: 5.3M entries examined instead of 7.1M push
//         stores concentrated on hub lines).  Rows the probe cannot settle go
//         to k_update_pull; rows still unsettled after kThreadMax entries are
//         cut into chunks of kPullChunk entries that k_round_end's warps scan
//         independently, so one long surviving row no longer sets the
//         kernel's duration (a row of 64k entries was 256 dependent warp
//         steps; R-MAT s26 round 1).  (A first version had
//         the select kernels emit a non-candidate list: on the grid that
//         emission alone cost as much as the select, ncu round 1.)
// k_round_end then also folds the tile counters, elects the last block, and
// publishes the round's IterationStats and the graph's loop condition.
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"
#include "scan.cuh"

namespace tcmis_b200 {

constexpr int kUpdItems = 8;

struct UpdateArgs {
  int32_t n;
  const int64_t *off;
  const int32_t *nbr;
  int64_t vnnz;            // nnz, negated if nbr is not 16-byte aligned (scan.cuh)
  uint32_t *prio;
  uint16_t *q;
  uint8_t *state;
  const uint8_t *next;
  Ctrl *ctrl;
  int32_t *wl0, *wl1;
  int fresh;
  uint64_t seed;
  int32_t n1;              // round-1 list (non-isolated vertices) for the pull probe
  const int32_t *nz;
  int nz_identity;
  PullRow *prow;           // pull: rows outliving the engine (ctrl->pull_count)
  int32_t *pitems;         // ... their chunks, row index per item (ctrl->pull_items)
  int32_t *undecided;      // pull: rows the probe could not settle (ctrl->pull_undec)
  Publish pub;             // multi-GPU: this round's removals of the own range
  const uint32_t *tile_hit;  // tile exclusion: per T=16 block row, rows with a candidate nbr
  uint8_t *segflag;
  const int32_t *rowtiles;
  int32_t nseg;
  int64_t total_tiles;
  int seg_mode;            // 0 none, 1 count + clear per round, 2 accumulate (h3)
  DevRound *rounds;
  int32_t tail_thr;        // the WHILE loop continues while alive > tail_thr
  const int32_t *perm;     // solve id -> caller id (relabeled graphs), else null
  const int2 *cb;          // degree-class bounds (common.cuh class_bounds), or null
  const int32_t *r1_max;   // round 1: the largest neighbour id first (select.cuh), or null
};

// kU row entries of v: a candidate neighbour has a key above v's (it beat v,
// alive at the round's start), so entries under the class bound lo are
// neither gathered nor, with the rows sorted, followed by anything that could
// be one (`below`).
template <int kU>
__device__ __forceinline__ bool hits_row(const uint8_t *__restrict__ next, const int32_t *u,
                                         int2 cb, bool &below) {
  bool hit = false;
  below = false;
#pragma unroll
  for (int j = 0; j < kU; ++j) {
    below |= u[j] >= 0 && u[j] < cb.x;
    if (u[j] >= cb.x) hit |= next[u[j]] == 1;
  }
  return hit;
}

// The end of a round, run by every block of the round's last kernel: the
// segment flags swept into the tile counters, the block's counts added, and
// the last block to arrive publishes the round's DevRound, resets the
// per-round counters and sets the graph's loop condition.
__device__ __forceinline__ void round_end_tail(const UpdateArgs &a, unsigned long long rem,
                                               cudaGraphConditionalHandle cond, int use_cond) {
  Ctrl *ctrl = a.ctrl;
  const int round = ctrl->round;
  const int out_slot = (round + 1) & 1;
  unsigned long long ev = 0;
  if (a.seg_mode == 1) {  // spmv.cpp:37-46, per block column (A is symmetric)
    // 16 flags per thread with one 16-byte load (the sweep is one pass, not a
    // grid-stride chain of byte loads); tile counts only for the set flags
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    int64_t head = 0;
    if ((((uintptr_t)a.segflag | (uintptr_t)a.rowtiles) & 15) == 0) {
      const int64_t nv = a.nseg / 16;
      for (int64_t c = gt; c < nv; c += gs) {
        uint4 *fp = reinterpret_cast<uint4 *>(a.segflag + 16 * c);
        const uint4 f = *fp;
        if (!(f.x | f.y | f.z | f.w)) continue;
        const uint32_t w[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!w[k]) continue;
          const int4 t = __ldg(reinterpret_cast<const int4 *>(a.rowtiles + 16 * c + 4 * k));
          if (w[k] & 0xffu) ev += (unsigned long long)t.x;
          if (w[k] & 0xff00u) ev += (unsigned long long)t.y;
          if (w[k] & 0xff0000u) ev += (unsigned long long)t.z;
          if (w[k] & 0xff000000u) ev += (unsigned long long)t.w;
        }
        *fp = make_uint4(0, 0, 0, 0);
      }
      head = nv * 16;
    }
    for (int64_t b = head + gt; b < a.nseg; b += gs) {
      if (a.segflag[b]) {
        ev += (unsigned long long)a.rowtiles[b];
        a.segflag[b] = 0;
      }
    }
  }
  block_add3(0, rem, ev, ctrl);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ctrl->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    volatile Ctrl *vc = ctrl;
    const int32_t alive = vc->wl_count[out_slot];
    // a ring: the host loop drains one slot per round; the graph loop flags
    // the (pathological, > max_rounds) case and the host re-runs step-wise.
    // The Phase start stamps t[0..2] are already in the slot.
    DevRound *r = &a.rounds[(round - 1) % vc->max_rounds];
    const unsigned long long sel = vc->sel, rem_all = vc->rem;
    r->sel = sel;
    r->rem = rem_all;
    r->alive = (unsigned long long)alive;
    r->eval = a.seg_mode == 1 ? vc->eval : 0;
    r->skip = a.seg_mode == 1 ? (unsigned long long)a.total_tiles - vc->eval : 0;
    r->t[3] = gtimer_ns();
    if (round > vc->max_rounds) vc->overflow = 1;
    // engine.cpp:138-160: every alive vertex leaves as selected or removed or
    // stays alive; anything else is a corrupt candidate (logic_error).  On a
    // rank of a partitioned solve the counts are the rank's own.
    if (!a.pub.bits && !a.pub.list && (unsigned long long)vc->alive != sel + rem_all + (unsigned long long)alive)
      vc->corrupt = 1;
    // progress: the alive vertex of the largest key is always a candidate, so
    // a round that selects nothing while vertices are alive can only come from
    // corrupt state -- stop there instead of spinning to the iteration cap
    if (!a.pub.bits && !a.pub.list && vc->alive > 0 && sel == 0) vc->corrupt = 1;
    vc->alive = alive;
    vc->sel = 0;
    vc->rem = 0;
    vc->eval = 0;
    vc->ticket = 0;
    vc->wl_count[round & 1] = 0;
    vc->long_count = 0;
    vc->pull_count = 0;
    vc->sel_vlong = 0;
    vc->pull_items = 0;
    vc->sel_undec = 0;
    vc->pull_undec = 0;
    vc->main_rounds = vc->main_rounds + 1;
    vc->round = round + 1;
    if (use_cond) cudaGraphSetConditional(cond, alive > a.tail_thr && !vc->corrupt ? 1u : 0u);
  }
}

// ---------------------------------------------------------------- push

// kEnd: the push round's last kernel also ends the round (round_end_tail),
// so the push form runs no separate k_round_end.
template <bool kEnd>
__global__ void __launch_bounds__(kBlock)
    k_update(UpdateArgs a, cudaGraphConditionalHandle cond, int use_cond) {
  pdl_entry();
  using BlockScan = cub::BlockScan<int, kBlock>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  __shared__ int s_base;
  Ctrl *ctrl = a.ctrl;
  const int round = ctrl->round;
  // push: Phase 2 is fused into the select kernels (its time is Phase 1's)
  stamp_phase(a.rounds, ctrl, round, kEnd ? 1 : 2, 2);
  const int64_t cnt = round == 1 ? a.n : ctrl->wl_count[round & 1];
  constexpr int64_t kChunk = (int64_t)kBlock * kUpdItems;
  if (!kEnd && (int64_t)blockIdx.x * kChunk >= cnt) return;  // kEnd: every block ends the round
  const int32_t *in = (round & 1) ? a.wl1 : a.wl0;
  int32_t *out = (round & 1) ? a.wl0 : a.wl1;
  const int out_slot = (round + 1) & 1;
  const uint64_t fresh_m = a.fresh ? mix64(combine_seed(a.seed, (uint64_t)round + 1)) : 0;
  unsigned long long rem = 0;
  for (int64_t base = (int64_t)blockIdx.x * kChunk; base < cnt;
       base += (int64_t)gridDim.x * kChunk) {
    // striped: item j of thread t is base + j*kBlock + t, so every load and
    // store instruction of the warp is coalesced on the identity worklist
    int32_t vs[kUpdItems];
    uint8_t ds[kUpdItems];
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j) {
      const int64_t i = base + (int64_t)j * kBlock + threadIdx.x;
      vs[j] = i < cnt ? (round == 1 ? (int32_t)i : in[i]) : -1;
    }
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j) ds[j] = vs[j] >= 0 ? a.next[vs[j]] : 1;
    if (a.tile_hit) {  // tile-form exclusion (tile_excl.cuh): nc > 0 from the row masks
#pragma unroll
      for (int j = 0; j < kUpdItems; ++j)
        if (ds[j] == 0 && ((__ldg(&a.tile_hit[vs[j] >> 4]) >> (vs[j] & 15)) & 1u)) ds[j] = 2;
    }
    int mine = 0;
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j) {
      const int32_t v = vs[j];
      publish_warp(a.pub, v, v >= 0 && ds[j] == 2);
      if (v < 0 || ds[j] == 1) continue;  // candidates were settled by k_select
      if (ds[j] == 2) {
        mark_removed(v, a.state, a.q);
        ++rem;
      } else {
        ++mine;
        if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m, a.perm);
      }
    }
    int pos, total;
    BlockScan(scan_tmp).ExclusiveSum(mine, pos, total);
    if (threadIdx.x == 0) s_base = total ? atomicAdd(&ctrl->wl_count[out_slot], total) : 0;
    __syncthreads();
    pos += s_base;
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j)
      if (vs[j] >= 0 && ds[j] == 0) out[pos++] = vs[j];
    __syncthreads();  // scan_tmp / s_base reuse
  }
  if (kEnd) round_end_tail(a, rem, cond, use_cond);
  else block_add3(0, rem, 0, ctrl);
}

// ---------------------------------------------------------------- pull

constexpr int kPullK = 4;  // row entries the straight-line pull probe examines

// Pull probe: one thread per vertex of the round's worklist (the same list the
// select kernels walked); the select kernels turned this round's candidates
// InMIS, so state == Alive marks exactly the alive non-candidates.
// Straight-line: the last <= 8 row entries with two aligned 16-byte loads,
// candidate flags of the last kPullK.
__global__ void __launch_bounds__(kBlock, TCMIS_PROBE_MINB) k_probe_pull(UpdateArgs a) {
  pdl_entry();
  __shared__ int32_t s_srv[kBlock / 32][64];
  __shared__ int32_t s_und[kBlock / 32][64];
  Ctrl *ctrl = a.ctrl;
  const int round = ctrl->round;
  const bool r1s = round == 1 && a.r1_max;  // after k_r1_pull: the vertices it left
  if (!r1s) stamp_phase(a.rounds, ctrl, round, 1, 1);
  const int64_t cnt = r1s ? ctrl->r1_pull_left : round == 1 ? a.n1 : ctrl->wl_count[round & 1];
  if ((int64_t)blockIdx.x * kBlock >= cnt) return;
  const int32_t *wl = r1s ? a.wl1 : round == 1 ? a.nz : ((round & 1) ? a.wl1 : a.wl0);
  int32_t *out = (round & 1) ? a.wl0 : a.wl1;
  int *tail = &ctrl->wl_count[(round + 1) & 1];
  const uint64_t fresh_m = a.fresh ? mix64(combine_seed(a.seed, (uint64_t)round + 1)) : 0;
  const uint8_t *__restrict__ next = a.next;
  const int lane = threadIdx.x & 31;
  WarpOut srv{s_srv[threadIdx.x >> 5], 0}, und{s_und[threadIdx.x >> 5], 0};
  unsigned long long rem = 0;
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  for (int64_t wb = (int64_t)blockIdx.x * kBlock + (threadIdx.x & ~31); wb < cnt; wb += stride) {
    const int64_t i = wb + lane;
    bool survive = false, undecided = false, pub = false;
    int32_t v = 0;
    if (i < cnt) {
      v = (round == 1 && a.nz_identity && !r1s) ? (int32_t)i : __ldg(&wl[i]);
    }
    if (i < cnt && a.state[v] == TCMIS_ALIVE) {
      const int64_t s = ld_stream(&a.off[v]), e = ld_stream(&a.off[v + 1]);
      int32_t u[4];
      load_tail4(a.nbr, a.vnnz, s, e, u);
      bool below;
      const bool hit = hits_row<kPullK>(next, u, class_bounds(a.cb, e - s), below);
      if (hit) {
        mark_removed(v, a.state, a.q);
        pub = true;
        ++rem;
      } else if (e - s <= kPullK || below) {
        survive = true;
        if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m, a.perm);
      } else {
        undecided = true;
      }
    }
    publish_warp(a.pub, v, pub);
    warp_emit(srv, survive, v, out, tail);
    warp_emit(und, undecided, v, a.undecided, &ctrl->pull_undec);
  }
  warp_flush(srv, out, tail);
  warp_flush(und, a.undecided, &ctrl->pull_undec);
  block_add3(0, rem, 0, ctrl);
}

// Round 1 on a degree-ordered graph: an alive non-candidate's largest
// neighbour id is its lowest-degree, highest-priority neighbour, most often
// a candidate -- one gather of next, no row.  Four consecutive vertices per
// thread (state and r1_max as vector loads, four gathers in flight); an
// alive vertex not settled so goes to wl1 (the select side is done with it)
// for k_probe_pull.
__global__ void __launch_bounds__(kBlock) k_r1_pull(UpdateArgs a) {
  pdl_entry();
  Ctrl *ctrl = a.ctrl;
  if (ctrl->round != 1) return;
  stamp_phase(a.rounds, ctrl, 1, 1, 1);
  constexpr int kV = 4;
  __shared__ BlockOut<kBlock, kV> left;
  left.reset();
  const int64_t n1 = a.n1;
  unsigned long long rem = 0;
  const int64_t quads = (n1 + kV - 1) / kV;
  for (int64_t t = blockIdx.x * (int64_t)kBlock + threadIdx.x; t - threadIdx.x < quads;
       t += (int64_t)gridDim.x * kBlock) {
    const int64_t v0 = t * kV;
    int32_t mx[kV];
    uint32_t st4 = 0;
    if (v0 + kV <= n1) {
      const int4 m4 = __ldg(reinterpret_cast<const int4 *>(a.r1_max + v0));
      mx[0] = m4.x; mx[1] = m4.y; mx[2] = m4.z; mx[3] = m4.w;
      st4 = *reinterpret_cast<const uint32_t *>(a.state + v0);
    } else {
#pragma unroll
      for (int j = 0; j < kV; ++j) {
        const bool ok = t < quads && v0 + j < n1;
        mx[j] = ok ? __ldg(&a.r1_max[v0 + j]) : -1;
        st4 |= (uint32_t)(ok ? a.state[v0 + j] : TCMIS_REMOVED) << (8 * j);
      }
    }
    bool alive[kV], hit[kV];
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      alive[j] = ((st4 >> (8 * j)) & 0xffu) == TCMIS_ALIVE;
      hit[j] = alive[j] && a.next[mx[j]] == 1;
    }
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      const int32_t v = (int32_t)(v0 + j);
      if (hit[j]) {
        mark_removed(v, a.state, a.q);
        ++rem;
      }
      publish_warp(a.pub, v, hit[j]);
      left.put(alive[j] && !hit[j], v);
    }
    left.flush(a.wl1, &ctrl->r1_pull_left);
  }
  block_add3(0, rem, 0, ctrl);
}

// Pull engine over the probe's undecided rows (per-lane state machine,
// 16-byte windows downward from e - kPullK).
__global__ void __launch_bounds__(kBlock) k_update_pull(UpdateArgs a) {
  pdl_entry();
  __shared__ int32_t s_buf[kBlock / 32][64];
  Ctrl *ctrl = a.ctrl;
  const int round = ctrl->round;
  const int64_t cnt = ctrl->pull_undec;
  if ((int64_t)blockIdx.x * kBlock >= cnt) return;
  int32_t *out = (round & 1) ? a.wl0 : a.wl1;
  int *tail = &ctrl->wl_count[(round + 1) & 1];
  const uint64_t fresh_m = a.fresh ? mix64(combine_seed(a.seed, (uint64_t)round + 1)) : 0;
  const int32_t *__restrict__ nbr = a.nbr;
  const uint8_t *__restrict__ next = a.next;
  WarpOut wo{s_buf[threadIdx.x >> 5], 0};
  const int64_t stride = (int64_t)gridDim.x * kBlock;
  unsigned long long rem = 0;
  int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x - stride;
  int mode = kFetch;
  int32_t v = 0;
  int64_t s = 0, e = 0, hi = 0;
  int2 cb = make_int2(0, 0);
  auto fetch = [&]() {
    i += stride;
    if (i < cnt) {
      v = __ldg(&a.undecided[i]);
      s = __ldg(&a.off[v]);
      e = __ldg(&a.off[v + 1]);
      cb = class_bounds(a.cb, e - s);
      hi = e - kPullK;
      mode = kScan;
    } else {
      mode = kDone;
    }
  };
  fetch();
  while (__any_sync(0xffffffffu, mode != kDone)) {
    bool survive = false, defer = false, pub = false;
    if (mode == kScan) {
      constexpr int kU = 4 * kSelWin;
      int32_t u[kU];
      int64_t w = load_window_down(nbr, a.vnnz, s, hi, u);
#pragma unroll
      for (int k = 1; k < kSelWin; ++k) {
        if (w > s) {
          w = load_window_down(nbr, a.vnnz, s, w, u + 4 * k);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) u[4 * k + j] = -1;
        }
      }
      bool below;
      const bool hit = hits_row<kU>(next, u, cb, below);
      hi = w;
      if (hit) {
        mark_removed(v, a.state, a.q);
        pub = true;
        ++rem;
        mode = kFetch;
      } else if (hi <= s || below) {
        survive = true;
        if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m, a.perm);
        mode = kFetch;
      } else if (e - hi >= kThreadMax) {
        defer = true;
        mode = kFetch;
      }
    }
    publish_warp(a.pub, v, pub);
    warp_emit(wo, survive, v, out, tail);
    if (__any_sync(0xffffffffu, defer)) {  // entries [s, hi) are left
      const int nch = defer ? (int)((hi - s + kPullChunk - 1) / kPullChunk) : 0;
      const int slot = warp_reserve(defer ? 1 : 0, &ctrl->pull_count);
      const int first = warp_reserve(nch, &ctrl->pull_items);
      if (defer) {
        a.prow[slot] = PullRow{s, hi, v, first, nch, 0};
        for (int c = 0; c < nch; ++c) a.pitems[first + c] = slot;
      }
    }
    if (mode == kFetch) fetch();
  }
  warp_flush(wo, out, tail);
  block_add3(0, rem, 0, ctrl);
}

// ------------------------------------------------------------ round end

__global__ void __launch_bounds__(kBlock)
    k_round_end(UpdateArgs a, cudaGraphConditionalHandle cond, int use_cond) {
  pdl_entry();
  Ctrl *ctrl = a.ctrl;
  const int round = ctrl->round;
  stamp_phase(a.rounds, ctrl, round, 2, 2);
  int32_t *out = (round & 1) ? a.wl0 : a.wl1;
  const int out_slot = (round + 1) & 1;
  const int lane = threadIdx.x & 31;
  const uint64_t fresh_m = a.fresh ? mix64(combine_seed(a.seed, (uint64_t)round + 1)) : 0;
  const int32_t *__restrict__ nbr = a.nbr;
  const uint8_t *__restrict__ next = a.next;
  unsigned long long rem = 0;
  // pull rows that outlived the engine, one chunk of kPullChunk entries per
  // warp (chunk c covers [hi - (c+1) kPullChunk, hi - c kPullChunk) of the
  // row); a chunk stops at its first candidate neighbour or once another
  // chunk of the row has found one, and the last chunk to finish decides
  auto decide = [&](int32_t v, bool hit) {
    if (hit) {
      mark_removed(v, a.state, a.q);
      publish(a.pub, v);
      ++rem;
    } else {
      if (a.fresh) set_fresh(a.prio, a.q, v, fresh_m, a.perm);
      out[atomicAdd(&ctrl->wl_count[out_slot], 1)] = v;
    }
  };
  const int ni = ctrl->pull_items;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < ni;
       it += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t slot = __ldcg(&a.pitems[it]);
    PullRow *row = &a.prow[slot];
    const int64_t lo0 = __ldcg(&row->lo), hi0 = __ldcg(&row->hi);
    const int32_t v = __ldcg(&row->v), first = __ldcg(&row->first);
    int64_t hi = hi0 - (int64_t)(it - first) * kPullChunk;
    const int64_t lo = hi - kPullChunk > lo0 ? hi - kPullChunk : lo0;
    const int2 cb = class_bounds(a.cb, a.cb ? __ldg(&a.off[v + 1]) - lo0 : 0);
    bool hit = false, other = false, done = false;
    while (!hit && !other && !done && hi > lo) {
      int32_t u[kWarpU];
#pragma unroll
      for (int j = 0; j < kWarpU; ++j) {
        const int64_t idx = hi - 1 - lane - 32 * j;
        u[j] = idx >= lo ? ld_stream(&nbr[idx]) : -1;
      }
      other = __ldcg(&row->hit) != 0;  // in flight with the row loads
      bool below;
      const bool b = hits_row<kWarpU>(next, u, cb, below);
      hit = __any_sync(0xffffffffu, b);
      done = __any_sync(0xffffffffu, below);
      other = __shfl_sync(0xffffffffu, other, 0);
      hi -= 32 * kWarpU;
    }
    if (lane == 0) {
      if (hit) atomicExch(&row->hit, 1);
      __threadfence();
      if (atomicSub(&row->left, 1) == 1) {
        __threadfence();
        decide(v, atomicAdd(&row->hit, 0) != 0);
      }
    }
  }
  round_end_tail(a, rem, cond, use_cond);
}

}  // namespace tcmis_b200
