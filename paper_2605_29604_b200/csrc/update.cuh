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
// alive vertex can never see a neighbour whose 1 is stale (that neighbour's
// round removed all of its neighbours), so "next[u] == 1" is exactly
// "u is a candidate of this round" for every neighbour u of an alive vertex.
//
// Two exclusion forms:
//   push  k_select already wrote next[u] = 2 for every neighbour of every
//         candidate; k_update is a coalesced striped pass (block-scan
//         compaction, one atomic per 2048 vertices).
//   pull  k_update_pull is a per-thread state machine: a non-candidate scans
//         its row from the end for next[u] == 1 and stops at the first hit
//         (R-MAT s22 round 1: 5.3M entries examined instead of 7.1M push
//         stores concentrated on hub lines).  Rows still unsettled after
//         kThreadMax entries go to a list that k_round_end scans warp-wide.
// k_round_end then also folds the tile counters, elects the last block, and
// publishes the round's IterationStats and the graph's loop condition.
#pragma once

#include <cub/cub.cuh>

#include "internal.cuh"
#include "select.cuh"

namespace tcmis_b200 {

constexpr int kUpdBlock = 256;
constexpr int kUpdItems = 8;

// Block-wide sum of three counters into the control block.
__device__ __forceinline__ void block_add3(unsigned long long a, unsigned long long b,
                                           unsigned long long c, Ctrl *ctrl) {
  __shared__ unsigned long long sh[3][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    sh[0][w] = a;
    sh[1][w] = b;
    sh[2][w] = c;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    a = lane < nw ? sh[0][lane] : 0;
    b = lane < nw ? sh[1][lane] : 0;
    c = lane < nw ? sh[2][lane] : 0;
    for (int o = 16; o; o >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, o);
      b += __shfl_down_sync(0xffffffffu, b, o);
      c += __shfl_down_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
      if (a) atomicAdd(&ctrl->sel, a);
      if (b) atomicAdd(&ctrl->rem, b);
      if (c) atomicAdd(&ctrl->eval, c);
    }
  }
}

__device__ __forceinline__ void leave(int32_t v, uint8_t st, uint8_t *state, uint64_t *key) {
  state[v] = st;
  key[v] = 0;  // kNoNeighborKey: v can no longer block anyone
}

__device__ __forceinline__ uint64_t fresh_key(int32_t v, uint64_t fresh_m) {
  // engine.cpp:324-325: next round's redrawn h1 priority
  return ((vertex_hash_m((uint64_t)v, fresh_m) >> 32) << 32) | (uint64_t)(v + 1);
}

// ---------------------------------------------------------------- push

__global__ void __launch_bounds__(kUpdBlock)
    k_update(int32_t n, uint64_t *__restrict__ key, uint8_t *__restrict__ state,
             const uint8_t *__restrict__ next, Ctrl *__restrict__ ctrl,
             int32_t *__restrict__ wl0, int32_t *__restrict__ wl1, int fresh, uint64_t seed) {
  using BlockScan = cub::BlockScan<int, kUpdBlock>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  __shared__ int s_base;
  const int round = ctrl->round;
  const int64_t cnt = round == 1 ? n : ctrl->wl_count[round & 1];
  const int32_t *in = (round & 1) ? wl1 : wl0;
  int32_t *out = (round & 1) ? wl0 : wl1;
  const int out_slot = (round + 1) & 1;
  const uint64_t fresh_m = fresh ? mix64(combine_seed(seed, (uint64_t)round + 1)) : 0;
  unsigned long long sel = 0, rem = 0;
  constexpr int64_t kChunk = (int64_t)kUpdBlock * kUpdItems;
  for (int64_t base = (int64_t)blockIdx.x * kChunk; base < cnt;
       base += (int64_t)gridDim.x * kChunk) {
    // striped: item j of thread t is base + j*kUpdBlock + t, so every load and
    // store instruction of the warp is coalesced on the identity worklist
    int32_t vs[kUpdItems];
    uint8_t ds[kUpdItems];
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j) {
      const int64_t i = base + (int64_t)j * kUpdBlock + threadIdx.x;
      vs[j] = i < cnt ? (round == 1 ? (int32_t)i : in[i]) : -1;
    }
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j) ds[j] = vs[j] >= 0 ? next[vs[j]] : 0;
    int mine = 0;
#pragma unroll
    for (int j = 0; j < kUpdItems; ++j) {
      const int32_t v = vs[j];
      if (v < 0) continue;
      if (ds[j] == 1) {  // engine.cpp:137-143: candidate joins the MIS
        leave(v, TCMIS_IN_MIS, state, key);
        ++sel;
      } else if (ds[j] == 2) {  // engine.cpp:144-147: alive with a candidate neighbour
        leave(v, TCMIS_REMOVED, state, key);
        ++rem;
      } else {
        ++mine;
        if (fresh) key[v] = fresh_key(v, fresh_m);
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
  block_add3(sel, rem, 0, ctrl);
}

// ---------------------------------------------------------------- pull

// Per-warp survivor buffer in shared memory, flushed 32 at a time with one
// atomic (survivors are decided at different loop iterations per lane).
struct WarpOut {
  int32_t *buf;  // 64 entries
  int fill;      // warp-uniform
};

__device__ __forceinline__ void warp_emit(WarpOut &w, bool have, int32_t v, int32_t *out,
                                          int *tail) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, have);
  if (have) w.buf[w.fill + __popc(m & ((1u << lane) - 1u))] = v;
  w.fill += __popc(m);
  __syncwarp();
  if (w.fill >= 32) {
    int base = 0;
    if (lane == 0) base = atomicAdd(tail, 32);
    base = __shfl_sync(0xffffffffu, base, 0);
    out[base + lane] = w.buf[lane];
    __syncwarp();
    if (lane < w.fill - 32) w.buf[lane] = w.buf[lane + 32];
    __syncwarp();
    w.fill -= 32;
  }
}

__device__ __forceinline__ void warp_flush(WarpOut &w, int32_t *out, int *tail) {
  const int lane = threadIdx.x & 31;
  if (w.fill == 0) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(tail, w.fill);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < w.fill) out[base + lane] = w.buf[lane];
  __syncwarp();
  w.fill = 0;
}

__global__ void __launch_bounds__(kSelBlock)
    k_update_pull(int32_t n, const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                  uint64_t *__restrict__ key, uint8_t *__restrict__ state,
                  const uint8_t *__restrict__ next, Ctrl *__restrict__ ctrl,
                  int32_t *__restrict__ wl0, int32_t *__restrict__ wl1, int fresh, uint64_t seed,
                  int32_t *__restrict__ long_list) {
  __shared__ int32_t s_buf[kSelBlock / 32][64];
  const int round = ctrl->round;
  const int64_t cnt = round == 1 ? n : ctrl->wl_count[round & 1];
  const int32_t *in = (round & 1) ? wl1 : wl0;
  int32_t *out = (round & 1) ? wl0 : wl1;
  int *tail = &ctrl->wl_count[(round + 1) & 1];
  const uint64_t fresh_m = fresh ? mix64(combine_seed(seed, (uint64_t)round + 1)) : 0;
  const int lane = threadIdx.x & 31;
  WarpOut wo{s_buf[threadIdx.x >> 5], 0};
  const int64_t stride = (int64_t)gridDim.x * kSelBlock;
  unsigned long long sel = 0, rem = 0;
  int64_t i = (int64_t)blockIdx.x * kSelBlock + threadIdx.x - stride;
  int mode = kFetch;
  int32_t v = 0;
  int64_t s = 0, e = 0, hi = 0;
  bool survive = false, defer = false;
  auto fetch = [&]() {
    i += stride;
    if (i >= cnt) {
      mode = kDone;
      return;
    }
    v = round == 1 ? (int32_t)i : in[i];
    const uint8_t d = next[v];
    if (d == 1) {  // engine.cpp:137-143
      leave(v, TCMIS_IN_MIS, state, key);
      ++sel;
      mode = kFetch;
    } else if (d == 2) {  // a push-mode exclusion left by k_select_long
      leave(v, TCMIS_REMOVED, state, key);
      ++rem;
      mode = kFetch;
    } else {
      s = __ldg(&off[v]);
      e = __ldg(&off[v + 1]);
      hi = e;
      mode = kScan;
    }
  };
  fetch();
  while (__any_sync(0xffffffffu, mode != kDone)) {
    survive = defer = false;
    if (mode == kScan) {
      int32_t u[kStep];
#pragma unroll
      for (int j = 0; j < kStep; ++j) u[j] = hi - 1 - j >= s ? __ldg(&nbr[hi - 1 - j]) : -1;
      bool hit = false;
#pragma unroll
      for (int j = 0; j < kStep; ++j)
        if (u[j] >= 0) hit |= next[u[j]] == 1;
      hi -= kStep;
      if (hit) {  // engine.cpp:144-147
        leave(v, TCMIS_REMOVED, state, key);
        ++rem;
        mode = kFetch;
      } else if (hi <= s) {
        survive = true;
        if (fresh) key[v] = fresh_key(v, fresh_m);
        mode = kFetch;
      } else if (e - hi >= kThreadMax) {
        defer = true;
        mode = kFetch;
      }
    }
    warp_emit(wo, survive, v, out, tail);
    const unsigned m = __ballot_sync(0xffffffffu, defer);
    if (m) {
      const int leader = __ffs(m) - 1;
      int pos = 0;
      if (lane == leader) pos = atomicAdd(&ctrl->pull_count, __popc(m));
      pos = __shfl_sync(0xffffffffu, pos, leader);
      if (defer) long_list[pos + __popc(m & ((1u << lane) - 1u))] = v;
    }
    if (mode == kFetch) fetch();
  }
  warp_flush(wo, out, tail);
  block_add3(sel, rem, 0, ctrl);
}

// ------------------------------------------------------------ round end

// seg_mode: 0 = no tile counters, 1 = count and clear per round,
// 2 = accumulate (h3: counters are taken once at the end).
__global__ void __launch_bounds__(kSelBlock)
    k_round_end(const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                uint64_t *__restrict__ key, uint8_t *__restrict__ state,
                const uint8_t *__restrict__ next, Ctrl *__restrict__ ctrl,
                int32_t *__restrict__ wl0, int32_t *__restrict__ wl1, int fresh, uint64_t seed,
                const int32_t *__restrict__ long_list, uint8_t *__restrict__ segflag,
                const int32_t *__restrict__ rowtiles, int32_t nseg, int64_t total_tiles,
                int seg_mode, DevRound *__restrict__ rounds, cudaGraphConditionalHandle cond,
                int use_cond) {
  const int round = ctrl->round;
  int32_t *out = (round & 1) ? wl0 : wl1;
  const int out_slot = (round + 1) & 1;
  const int lane = threadIdx.x & 31;
  const uint64_t fresh_m = fresh ? mix64(combine_seed(seed, (uint64_t)round + 1)) : 0;
  unsigned long long rem = 0, ev = 0;
  // pull rows longer than the thread probe: one warp per row
  const int nl = ctrl->pull_count;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nl;
       q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t v = long_list[q];
    const int64_t s = __ldg(&off[v]), e = __ldg(&off[v + 1]);
    int64_t hi = e - kThreadMax;
    bool hit = false;
    while (!hit && hi > s) {
      int32_t u[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t idx = hi - 1 - lane - 32 * j;
        u[j] = idx >= s ? __ldg(&nbr[idx]) : -1;
      }
      bool b = false;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (u[j] >= 0) b |= next[u[j]] == 1;
      hit = __any_sync(0xffffffffu, b);
      hi -= 128;
    }
    if (lane == 0) {
      if (hit) {
        leave(v, TCMIS_REMOVED, state, key);
        ++rem;
      } else {
        if (fresh) key[v] = fresh_key(v, fresh_m);
        out[atomicAdd(&ctrl->wl_count[out_slot], 1)] = v;
      }
    }
  }
  if (seg_mode == 1) {  // spmv.cpp:37-46, per block column (A is symmetric)
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nseg;
         b += (int64_t)gridDim.x * blockDim.x) {
      if (segflag[b]) {
        ev += (unsigned long long)rowtiles[b];
        segflag[b] = 0;
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
    DevRound r;
    r.sel = vc->sel;
    r.rem = vc->rem;
    r.alive = (unsigned long long)alive;
    r.eval = seg_mode == 1 ? vc->eval : 0;
    r.skip = seg_mode == 1 ? (unsigned long long)total_tiles - vc->eval : 0;
    // a ring: the host loop drains one slot per round; the graph loop flags
    // the (pathological, > max_rounds) case and the host re-runs step-wise
    rounds[(round - 1) % vc->max_rounds] = r;
    if (round > vc->max_rounds) vc->overflow = 1;
    vc->alive = alive;
    vc->sel = 0;
    vc->rem = 0;
    vc->eval = 0;
    vc->ticket = 0;
    vc->wl_count[round & 1] = 0;
    vc->long_count = 0;
    vc->pull_count = 0;
    vc->round = round + 1;
    if (use_cond) cudaGraphSetConditional(cond, alive > 0 ? 1u : 0u);
  }
}

}  // namespace tcmis_b200
