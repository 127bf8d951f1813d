// tail.cuh -- the small late rounds of a solve in ONE persistent kernel.
//
// After the first one or two rounds the alive worklist is small (R-MAT s22:
// 57k, 1.7k, 23 vertices in rounds 2-4), and four kernel launches per round
// cost more than the work.  k_tail runs all remaining rounds in one
// cooperative launch with ONE grid barrier per round: round r's pass over its
// list L_r does
//
//   * the Phase 3 of round r-1 (engine.cpp:121-160): L_r holds round r-1's
//     non-candidates; a vertex whose decision byte says "excluded in round
//     r-1" is Removed now (state, q = 0), the rest are alive in round r;
//   * the Phase 1 of round r (engine.cpp:86-119) for the alive ones: a group
//     of kGroup lanes scans the row from its end, kGroup*kTU entries per step,
//     and stops at the first neighbour that is alive at the start of round r
//     (q != 0 and not excluded in round r-1) with a higher key; rows longer
//     than kTailLong are scanned by the whole block;
//   * the push form of Phase 2 (spmv.cpp:18-59, nc > 0) for round r's
//     candidates: a blind store xm[r & 1][u] = 1 for every neighbour u.  The
//     exclusion planes alternate with the round's parity, so round r's pushes
//     never touch the plane round r reads for round r-1's removals -- the
//     snapshot of the reference's bulk-synchronous round is kept, and round
//     count and every statistic equal the reference's.  A stale mark from
//     round r-2 (or an earlier solve) sits only on dead vertices (q = 0); the
//     kernel clears both planes of the vertices alive at its start;
//   * L_{r+1} = round r's non-candidates.
//
// Round r's IterationStats are complete after round r+1's pass (its removed /
// alive counts are counted there), so block 0 publishes round r-1 after
// barrier r.  The solve's MIS-id compaction is fused at the end.  Data
// written by other blocks in an earlier phase is read with ld.global.cg (L2).
// (The first version ran S and U as separate phases, two barriers per round:
// s22 rounds 2-4 took 75 us, ER rounds 2-6 65 us.)
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"

namespace tcmis_b200 {

#ifdef TCMIS_TAIL_PROF
// profiling build only: block 0 / thread 0 stamps %globaltimer at phase ends
// into g_tail_prof (read back by tcmis_debug_tail_prof, solver.cu)
__device__ unsigned long long g_tail_prof[256];
__device__ int g_tail_prof_n;
__device__ unsigned long long g_tail_blk[3][1024];  // first round: per block (t_short, t_long_end, nlong)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TAIL_MARK(tag, val)                                                   \
  do {                                                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_tail_prof_n < 128) {         \
      g_tail_prof[2 * g_tail_prof_n] = gtimer();                              \
      g_tail_prof[2 * g_tail_prof_n + 1] = ((unsigned long long)(tag) << 32) | \
                                           (unsigned)(val);                   \
      ++g_tail_prof_n;                                                        \
    }                                                                         \
  } while (0)
#else
#define TAIL_MARK(tag, val) \
  do {                    \
  } while (0)
#endif

#ifndef TCMIS_TAIL_GROUP
#define TCMIS_TAIL_GROUP 8
#endif
constexpr int kGroup = TCMIS_TAIL_GROUP;  // lanes per vertex in the tail kernel
#ifndef TCMIS_TAIL_UNROLL
#define TCMIS_TAIL_UNROLL 16
#endif
constexpr int kTU = TCMIS_TAIL_UNROLL;  // independent loads per lane per step
constexpr int kTailBlock = 1024;  // one block per SM: 148 arrivals per barrier
#ifndef TCMIS_TAIL_LONG
#define TCMIS_TAIL_LONG 512
#endif
constexpr int64_t kTailLong = TCMIS_TAIL_LONG;  // rows above this are scanned by a whole block
constexpr int kTailLongCap = 256;               // per-block list of such rows per round

struct TailArgs {
  const int64_t *off;
  const int32_t *nbr;
  uint32_t *prio;
  uint16_t *q;
  uint8_t *next;
  uint8_t *xm0, *xm1;       // exclusion planes by round parity
  uint8_t *state;
  uint8_t *segflag;         // byte flags (seg_mode 2)
  uint32_t *segmark;        // seg_mode 1: round that last counted the segment
  const int32_t *rowtiles;
  int32_t nseg;
  int64_t total_tiles;
  int seg_mode;
  int T;
  Ctrl *ctrl;
  int32_t *wl0, *wl1;
  DevRound *rounds;
  unsigned *bar;            // [0] arrivals, [1] generation
  // the solve's final step, fused: ascending MIS ids (engine.cpp:293)
  int compact;
  int32_t n;
  int32_t *mis;
  int64_t *mis_count;
  unsigned *blockcnt;       // gridDim.x per-block counts
  HostRes *pack;            // non-null: also leave the solve's results in mapped host memory
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


__device__ __forceinline__ uint8_t *xplane(const TailArgs &a, int r) {
  return (r & 1) ? a.xm1 : a.xm0;
}

// A candidate of the tail (mark_candidate + the tile counter of seg_mode 1:
// exactly one candidate of the round counts its block column).
__device__ __forceinline__ void tail_candidate(const TailArgs &a, int32_t v, int round,
                                               unsigned long long &sel,
                                               unsigned long long &ev) {
  a.next[v] = 1;
  a.state[v] = TCMIS_IN_MIS;
  ++sel;
  const int32_t sb = seg_of(v, a.T);
  if (a.seg_mode == 2) {
    a.segflag[sb] = 1;
  } else if (a.seg_mode == 1) {
    if (atomicMax(&a.segmark[sb], (unsigned)round) < (unsigned)round)
      ev += (unsigned long long)a.rowtiles[sb];
  }
}

// u blocks v in round r: alive at the start of round r (q != 0, not
// excluded in round r-1), higher key; `alive` reports the first part
__device__ __forceinline__ bool tail_blocks(const TailArgs &a, int32_t u, const uint8_t *dead,
                                            uint32_t qv, uint64_t kv, bool &alive) {
  const uint32_t qu = __ldcg(&a.q[u]);
  const uint8_t dx = __ldcg(&dead[u]);  // independent of qu: one round trip for both
  alive = qu != 0 && !dx;
  if (!alive) return false;
  return qu != qv ? qu > qv : key_of(__ldcg(&a.prio[u]), u) > kv;
}

__device__ __forceinline__ bool tail_alive(const TailArgs &a, int32_t u, const uint8_t *dead) {
  const uint32_t qu = __ldcg(&a.q[u]);
  const uint8_t dx = __ldcg(&dead[u]);
  return qu != 0 && !dx;
}

// the lanes of one group stay converged (same vertex, same trip count);
// different groups of a warp may diverge, so the vote uses the group's mask
__device__ __forceinline__ unsigned group_any(bool b, unsigned gmask) {
  return __ballot_sync(gmask, b);
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

__device__ __forceinline__ unsigned long long *slot_field(const TailArgs &a, int round, int f) {
  DevRound *r = &a.rounds[(round - 1) % a.ctrl->max_rounds];
  return f == 0 ? &r->sel : f == 1 ? &r->rem : f == 2 ? &r->alive : &r->eval;
}

// Ascending ids of the InMIS vertices (the reference sorts result.mis,
// engine.cpp:293): block b owns a contiguous range of 16-vertex units and
// walks it in tiles of kTailBlock units (one coalesced 16-byte state load per
// thread): per-block counts -> grid barrier -> every block sums the counts
// before it and writes its ids tile by tile (block scan of the per-thread
// counts).  Replaces a separate cub::DeviceSelect (2 launches, 17 us at
// R-MAT s22, 191 us at s26).
__device__ __forceinline__ uint32_t in_mis_mask16(const TailArgs &a, int64_t u) {
  const uint4 w = __ldcg(reinterpret_cast<const uint4 *>(a.state) + u);
  const uint32_t x[4] = {w.x, w.y, w.z, w.w};
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (((x[k] >> (8 * j)) & 0xffu) == TCMIS_IN_MIS) m |= 1u << (4 * k + j);
  const int64_t left = (int64_t)a.n - 16 * u;  // padding bytes past n
  if (left < 16) m &= (1u << left) - 1u;
  return m;
}

constexpr int kCU = 4;  // 16-vertex units per thread per tile (independent 16-B loads)

__device__ void compact_mis(const TailArgs &a) {
  __shared__ unsigned long long s_base;
  const int64_t units = ((int64_t)a.n + 15) / 16;
  const int64_t per_block = (units + gridDim.x - 1) / gridDim.x;
  const int64_t u0 = min(units, (int64_t)blockIdx.x * per_block);
  const int64_t u1 = min(units, u0 + per_block);
  constexpr int64_t kTile = (int64_t)kTailBlock * kCU;
  int cnt = 0;
  for (int64_t t0 = u0; t0 < u1; t0 += kTile) {
    uint32_t m[kCU];
#pragma unroll
    for (int k = 0; k < kCU; ++k) {
      const int64_t u = t0 + (int64_t)k * kTailBlock + threadIdx.x;
      m[k] = u < u1 ? in_mis_mask16(a, u) : 0u;
    }
#pragma unroll
    for (int k = 0; k < kCU; ++k) cnt += __popc(m[k]);
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(&s_base, (unsigned long long)cnt);
  __syncthreads();
  if (threadIdx.x == 0) a.blockcnt[blockIdx.x] = (unsigned)s_base;
  TAIL_MARK(5, 0);
  grid_barrier(a.bar);
  TAIL_MARK(6, 0);
  unsigned long long before = 0;
  for (int j = threadIdx.x; j < (int)blockIdx.x; j += kTailBlock) before += __ldcg(&a.blockcnt[j]);
  before = __reduce_add_sync(0xffffffffu, (unsigned)before);
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && before) atomicAdd(&s_base, before);
  __syncthreads();
  int64_t base = (int64_t)s_base;
  // write pass: warp w of a tile owns 256 consecutive vertices (8 per lane,
  // one 8-byte state load); the warp stages its ids in shared memory in order
  // and copies them out coalesced (a thread writing its own run directly
  // made every store instruction touch 32 sectors: 247 us at s26)
  __shared__ int32_t stage[kTailBlock / 32][256];
  __shared__ int s_woff[kTailBlock / 32 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t v_lo = u0 * 16, v_hi = min((int64_t)a.n, u1 * 16);
  constexpr int64_t kStep = 256ll * (kTailBlock / 32);
  // the next tile's 8 states per lane are loaded before this tile's barriers
  uint2 xn = make_uint2(0, 0);
  if (v_lo + (int64_t)w * 256 + lane * 8 < v_hi)
    xn = __ldcg(reinterpret_cast<const uint2 *>(a.state + v_lo + (int64_t)w * 256 + lane * 8));
  for (int64_t t0 = v_lo; t0 < v_hi; t0 += kStep) {
    const int64_t v0 = t0 + (int64_t)w * 256 + lane * 8;
    const uint2 x = xn;
    if (v0 + kStep < v_hi)
      xn = __ldcg(reinterpret_cast<const uint2 *>(a.state + v0 + kStep));
    uint32_t m = 0;
    if (v0 < v_hi) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (((x.x >> (8 * j)) & 0xffu) == TCMIS_IN_MIS) m |= 1u << j;
        if (((x.y >> (8 * j)) & 0xffu) == TCMIS_IN_MIS) m |= 1u << (4 + j);
      }
      const int64_t left = v_hi - v0;
      if (left < 8) m &= (1u << left) - 1u;
    }
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int excl = incl - c;
    if (lane == 31) s_woff[w] = incl;
    int k = excl;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      stage[w][k++] = (int32_t)(v0 + bit);
    }
    __syncthreads();
    if (w == 0) {  // exclusive scan of the 32 warp counts, by shuffles
      static_assert(kTailBlock / 32 == 32, "one warp count per lane");
      const int t = s_woff[lane];
      int sc = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, sc, o);
        if (lane >= o) sc += y;
      }
      s_woff[lane] = sc - t;
      if (lane == 31) s_woff[32] = sc;
    }
    __syncthreads();
    const int wc = (w + 1 < kTailBlock / 32 ? s_woff[w + 1] : s_woff[kTailBlock / 32]) - s_woff[w];
    for (int i = lane; i < wc; i += 32) a.mis[base + s_woff[w] + i] = stage[w][i];
    base += s_woff[kTailBlock / 32];
    __syncthreads();  // stage / s_woff reuse
  }
  if (blockIdx.x == gridDim.x - 1) {
    if (threadIdx.x == 0) *a.mis_count = base;
    if (a.pack) {  // k_pack's job, done here: one graph node less
      // word copies through L2 (ld.global.cg): written by other blocks
      const int32_t cap = __ldcg(&a.ctrl->max_rounds);
      const int nr = (int)(sizeof(DevRound) / 4) * (cap < 64 ? cap : 64);
      const uint32_t *rs = reinterpret_cast<const uint32_t *>(a.rounds);
      uint32_t *rd = reinterpret_cast<uint32_t *>(a.pack->rounds);
      for (int i = threadIdx.x; i < nr; i += kTailBlock) rd[i] = __ldcg(rs + i);
      const uint32_t *cs = reinterpret_cast<const uint32_t *>(a.ctrl);
      uint32_t *cd = reinterpret_cast<uint32_t *>(&a.pack->ctrl);
      for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += kTailBlock) cd[i] = __ldcg(cs + i);
      if (threadIdx.x == 0) a.pack->mis_count = (long long)base;
      __threadfence_system();
    }
  }
}

#ifndef TCMIS_TAIL_MINB
#define TCMIS_TAIL_MINB 1
#endif
__global__ void __launch_bounds__(kTailBlock, TCMIS_TAIL_MINB) k_tail(TailArgs a) {
  __shared__ int32_t s_long[kTailLongCap];
  __shared__ int s_nlong;
  __shared__ unsigned long long s_acc[4];
  Ctrl *ctrl = a.ctrl;
  const int lane = threadIdx.x & 31;
  const int gl = lane & (kGroup - 1);
  const unsigned gmask = ((1u << kGroup) - 1u) << (lane & ~(kGroup - 1));
  const int64_t gid = ((int64_t)blockIdx.x * kTailBlock + threadIdx.x) / kGroup;
  const int64_t ngroups = ((int64_t)gridDim.x * kTailBlock) / kGroup;
  constexpr int kW = kGroup * kTU;  // entries per group step: short rows settle in one step
  if (threadIdx.x == 0) s_nlong = 0;
  if (threadIdx.x < 4) s_acc[threadIdx.x] = 0;
  __syncthreads();
  const int r0 = *(volatile int *)&ctrl->round;
  const int64_t cnt0 = *(volatile int *)&ctrl->wl_count[r0 & 1];
  TAIL_MARK(1, cnt0);
  if (cnt0 > 0) {
    // the exclusion planes of the vertices alive at the tail's start (every
    // list below is a subset): stale marks elsewhere sit on dead vertices
    const int32_t *in0 = (r0 & 1) ? a.wl1 : a.wl0;
    for (int64_t i = (int64_t)blockIdx.x * kTailBlock + threadIdx.x; i < cnt0;
         i += (int64_t)gridDim.x * kTailBlock) {
      const int32_t v = __ldcg(&in0[i]);
      a.xm0[v] = 0;
      a.xm1[v] = 0;
    }
    grid_barrier(a.bar);
  }
  for (int round = r0; cnt0 > 0; ++round) {
    const bool first = round == r0;
    const int64_t cnt = first ? cnt0 : (int64_t) * (volatile int *)&ctrl->tail_cnt[round % 3];
    const int32_t *in = (round & 1) ? a.wl1 : a.wl0;
    int32_t *out = (round & 1) ? a.wl0 : a.wl1;
    int *out_cnt = &ctrl->tail_cnt[(round + 1) % 3];
    const uint8_t *dead = xplane(a, round - 1);
    uint8_t *push = xplane(a, round);
    unsigned long long sel = 0, ev = 0, rem = 0, alive = 0;
    for (int64_t i = gid; i < cnt; i += ngroups) {
      const int32_t v = __ldcg(&in[i]);
      if (!first && __ldcg(&dead[v])) {  // removed in round - 1
        if (gl == 0) {
          mark_removed(v, a.state, a.q);
          ++rem;
        }
        continue;
      }
      if (gl == 0) ++alive;
      const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
      if (e - s > kTailLong && defer_long(v, s_long, &s_nlong, gl, gmask, lane)) continue;
      const uint64_t kv = key_of(__ldcg(&a.prio[v]), v);
      const uint32_t qv = __ldcg(&a.q[v]);
      bool blocked = false;
      int32_t u[kTU];
      uint32_t live = 0;  // neighbours of the last chunk alive at the round's start
      for (int64_t hi = e; hi > s && !blocked; hi -= kW) {
#pragma unroll
        for (int j = 0; j < kTU; ++j) {
          const int64_t idx = hi - 1 - gl - kGroup * j;
          u[j] = idx >= s ? __ldg(&a.nbr[idx]) : -1;
        }
        bool b = false;
        live = 0;
#pragma unroll
        for (int j = 0; j < kTU; ++j)
          if (u[j] >= 0) {
            bool al;
            b |= tail_blocks(a, u[j], dead, qv, kv, al);
            live |= (uint32_t)al << j;
          }
        blocked = group_any(b, gmask) != 0;
      }
      if (!blocked) {
        if (gl == 0) tail_candidate(a, v, round, sel, ev);
        // push to the neighbours alive at the round's start only: after round
        // 1 most neighbours are dead, and every skipped byte store is a
        // random partial-sector write saved (R-MAT s22 round 2: ~1.4M)
        if (e - s <= kW) {  // the row was one chunk: its ids and flags are still here
#pragma unroll
          for (int j = 0; j < kTU; ++j)
            if ((live >> j) & 1u) push[u[j]] = 1;
        } else {
          for (int64_t hi = e; hi > s; hi -= kW) {
#pragma unroll
            for (int j = 0; j < kTU; ++j) {
              const int64_t idx = hi - 1 - gl - kGroup * j;
              u[j] = idx >= s ? __ldg(&a.nbr[idx]) : -1;
            }
#pragma unroll
            for (int j = 0; j < kTU; ++j)
              if (u[j] >= 0 && tail_alive(a, u[j], dead)) push[u[j]] = 1;
          }
        }
      } else if (gl == 0) {
        out[atomicAdd(out_cnt, 1)] = v;
      }
    }
    __syncthreads();
    const int nlong = min(s_nlong, kTailLongCap);
#ifdef TCMIS_TAIL_PROF
    if (first && threadIdx.x == 0) {
      g_tail_blk[0][blockIdx.x] = gtimer();
      g_tail_blk[2][blockIdx.x] = (unsigned long long)s_nlong;
    }
#endif
    for (int k = 0; k < nlong; ++k) {
      const int32_t v = s_long[k];
      const int64_t s = __ldg(&a.off[v]), e = __ldg(&a.off[v + 1]);
      const uint64_t kv = key_of(__ldcg(&a.prio[v]), v);
      const uint32_t qv = __ldcg(&a.q[v]);
      bool blocked = false;
      for (int64_t hi = e; hi > s && !blocked; hi -= 4 * kTailBlock) {
        bool b = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t idx = hi - 1 - threadIdx.x - (int64_t)kTailBlock * j;
          bool al;
          if (idx >= s) b |= tail_blocks(a, __ldg(&a.nbr[idx]), dead, qv, kv, al);
        }
        blocked = __syncthreads_or(b) != 0;
      }
      if (!blocked) {
        if (threadIdx.x == 0) tail_candidate(a, v, round, sel, ev);
        for (int64_t base = s; base < e; base += 4 * kTailBlock) {
          int32_t w[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int64_t idx = base + threadIdx.x + (int64_t)kTailBlock * j;
            w[j] = idx < e ? __ldg(&a.nbr[idx]) : -1;
          }
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (w[j] >= 0 && tail_alive(a, w[j], dead)) push[w[j]] = 1;
        }
      } else if (threadIdx.x == 0) {
        out[atomicAdd(out_cnt, 1)] = v;
      }
    }
#ifdef TCMIS_TAIL_PROF
    if (first && threadIdx.x == 0) g_tail_blk[1][blockIdx.x] = gtimer();
#endif
    // round's counters -> the DevRound ring (round: sel, eval; round-1: rem, alive)
    sel = __reduce_add_sync(0xffffffffu, (unsigned)sel);
    ev = __reduce_add_sync(0xffffffffu, (unsigned)ev);  // < 2^32 per warp
    rem = __reduce_add_sync(0xffffffffu, (unsigned)rem);
    alive = __reduce_add_sync(0xffffffffu, (unsigned)alive);
    if (lane == 0) {
      if (sel) atomicAdd(&s_acc[0], sel);
      if (ev) atomicAdd(&s_acc[1], ev);
      if (rem) atomicAdd(&s_acc[2], rem);
      if (alive) atomicAdd(&s_acc[3], alive);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_nlong = 0;
      if (s_acc[0]) atomicAdd(slot_field(a, round, 0), s_acc[0]);
      if (s_acc[1]) atomicAdd(slot_field(a, round, 3), s_acc[1]);
      if (!first) {
        if (s_acc[2]) atomicAdd(slot_field(a, round - 1, 1), s_acc[2]);
        if (s_acc[3]) atomicAdd(slot_field(a, round - 1, 2), s_acc[3]);
      }
      s_acc[0] = s_acc[1] = s_acc[2] = s_acc[3] = 0;
    }
    TAIL_MARK(2, cnt);
    grid_barrier(a.bar);
    TAIL_MARK(3, round);
    // round - 1 is complete: publish it; stop when it left nobody alive
    bool done = false;
    if (!first) {
      volatile DevRound *pr = &a.rounds[(round - 2) % ctrl->max_rounds];
      const unsigned long long alive_prev = pr->alive;
      done = alive_prev == 0;
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        volatile Ctrl *vc = ctrl;
        const unsigned long long evp = pr->eval;
        pr->eval = a.seg_mode == 1 ? evp : 0;
        pr->skip = a.seg_mode == 1 ? (unsigned long long)a.total_tiles - evp : 0;
        if (round - 1 > vc->max_rounds) vc->overflow = 1;
        vc->alive = (int32_t)alive_prev;
        vc->round = done ? round : round + 1;  // rounds run = round - 1 when done
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      // ready the ring slot two rounds ahead and the list count read this round
      volatile DevRound *z = &a.rounds[(round + 1) % ctrl->max_rounds];
      z->sel = z->rem = z->alive = z->eval = z->skip = 0;
      ctrl->tail_cnt[round % 3] = 0;
      __threadfence();
    }
    if (done) break;
  }
  if (a.compact) {
    grid_barrier(a.bar);
    TAIL_MARK(4, 0);
    compact_mis(a);
    TAIL_MARK(7, 0);
  }
}

}  // namespace tcmis_b200
