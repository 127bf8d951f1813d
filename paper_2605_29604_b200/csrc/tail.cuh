// tail.cuh -- the small late rounds of a solve in ONE persistent kernel.
//
// After the first one or two rounds the alive worklist is small (R-MAT s22:
// 57k, 1.7k, 23 vertices in rounds 2-4), and four kernel launches per round
// cost more than the work.  k_tail runs all remaining rounds in one
// cooperative launch with ONE grid barrier per round: round r's pass over its
// list L_r does
//
//   * the Phase 3 of round r-1 (engine.cpp:121-160): L_r holds round r-1's
//     non-candidates; a vertex tagged "excluded in round r-1" is Removed now
//     (state, q = 0), the rest are alive in round r;
//   * the Phase 1 of round r (engine.cpp:86-119) for the alive ones: a
//     neighbour blocks v iff it is alive at the start of round r (q != 0 and
//     not tagged for round r-1) and has a higher key;
//   * the push form of Phase 2 (spmv.cpp:18-59, nc > 0) for round r's
//     candidates: xt[u] = tag(r) for every neighbour u alive at the round's
//     start.  Round r reads only tag(r-1), so its own pushes never disturb the
//     snapshot it reads -- the reference's bulk-synchronous round is kept, and
//     the round count and every statistic equal the reference's;
//   * L_{r+1} = round r's non-candidates.
//
// Round tags.  xt is a u16 plane whose tags do not repeat across solves: the
// solve's tags are tag(r) = base + 2 + (r - r0), and the next solve's base is
// one past the last tag used, kept on the device (tslot[0]).  A vertex never
// tagged holds 0 or an older solve's tag, so nothing has to be cleared before
// the first round (the previous design cleared two byte planes of the
// starting list and paid a grid barrier for it).  Once base passes kTagWrap
// (every ~12k solves) the tags of the starting list are cleared and base
// restarts at 0; a solve runs at most kMaxTailRounds tail rounds (beyond, it
// flags the ring overflow and the host re-runs it step-wise).
// A neighbour's tag is loaded only when its q is non-zero: most neighbours
// of a late round's vertices left in round 1 (q = 0), and the tag plane is
// cold in L2 (the first version loaded both together: s22's first tail round
// took 29 us, mostly random DRAM sectors of a 4-byte tag plane).
//
// Block-resident lists.  The host caps the tail's starting list at 1024
// vertices per block (tail_thr <= grid x 1024).  Block b takes a contiguous
// slice of it, and from then on its survivors stay with it: the slice lives
// in shared memory (id, row extent, q), entry k with thread k.  A round costs
//   1. one THREAD per entry: its tag and the last kThrScan entries of its row
//      are loaded together (the row extent is in shared memory), then their
//      q / tag gathers -- two dependent round trips.  A blocker there (rows
//      are scanned from the end, where R-MAT's low-degree, high-priority
//      neighbours sit) settles a non-candidate; a row of <= kThrScan entries
//      is settled either way, and a candidate pushes from its registers;
//   2. rows left over: groups of kGroup lanes, kGroup*kTU entries per step
//      (rows above kTailLong: the whole block);
//   3. the survivors compacted in shared memory, and ONE grid barrier whose
//      arrival atomic also sums the survivors (grid_barrier_sum): the release
//      word says whether anyone is left, so no round trip decides the loop.
// The per-round statistics are accumulated with fire-and-forget atomics and
// published once, after the last round, by block 0.
#pragma once

#include <cub/cub.cuh>

#include "scan.cuh"

namespace tcmis_b200 {

#ifdef TCMIS_TAIL_PROF
// profiling build only: block 0 / thread 0 stamps %globaltimer at phase ends
// into g_tail_prof (read back by tcmis_debug_tail_prof, solver.cu)
__device__ unsigned long long g_tail_prof[256];
__device__ int g_tail_prof_n;
__device__ unsigned long long g_tail_blk[5][1024];  // first round, per block: t_thread, t_end, ndeferred, entries, t_start
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
#define TCMIS_TAIL_GROUP 16
#endif
constexpr int kGroup = TCMIS_TAIL_GROUP;  // lanes per deferred row
#ifndef TCMIS_TAIL_UNROLL
#define TCMIS_TAIL_UNROLL 8
#endif
constexpr int kTU = TCMIS_TAIL_UNROLL;  // independent loads per lane per group step
constexpr int kTailBlock = 1024;        // one block per SM: 148 arrivals per barrier
constexpr int kTailWarps = kTailBlock / 32;
constexpr int kTailGroups = kTailBlock / kGroup;
#ifndef TCMIS_TAIL_THR_SCAN
#define TCMIS_TAIL_THR_SCAN 8
#endif
constexpr int kThrScan = TCMIS_TAIL_THR_SCAN;  // row entries a thread scans on its own
#ifndef TCMIS_TAIL_LONG
#define TCMIS_TAIL_LONG 512
#endif
constexpr int64_t kTailLong = TCMIS_TAIL_LONG;  // rows above this are scanned by a whole block
constexpr int kTailLongCap = 256;               // per-block list of such rows per chunk
constexpr int kMaxTailRounds = 4096;            // = the host's round ring (DevRound) capacity
constexpr uint32_t kTagWrap = 0xFFFFu - kMaxTailRounds - 4;  // restart the round tags beyond this base
constexpr int kCompactV = 512;                  // vertices per warp step of the MIS write pass
constexpr int kTailMaxWarps = 32 * 2048;        // capacity of one per-warp count buffer
// dynamic shared memory of k_tail: the write pass's per-warp staging
constexpr size_t kTailDynSmem = sizeof(int32_t) * kTailWarps * kCompactV;
static_assert(sizeof(int32_t) * kTailBlock * kThrScan + sizeof(long long) * (kTailBlock + 1) +
                      sizeof(int16_t) * kTailBlock <= kTailDynSmem,
              "the windows, the push offsets and the push list share the staging area");

struct TailArgs {
  const int64_t *off;
  const int32_t *nbr;
  int64_t vnnz;             // nnz, negated if nbr is not 16-byte aligned (scan.cuh)
  const uint32_t *prio;
  uint16_t *q;
  const uint8_t *next;      // next[v] == 1: candidate of a per-round kernel round (read-only here)
  uint16_t *xt;             // round tags (see above)
  uint32_t *tslot;          // [0] tag base, [1] solve counter: persist across solves
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
  unsigned *bar;            // grid_barrier_sum: [0..1] arrivals | sum, [2] generation;
                            // [3] arrivals for the publishing block
  // the solve's final step, fused: ascending MIS ids (engine.cpp:293)
  int32_t n;
  int32_t *mis;
  int64_t *mis_count;
  unsigned *warpcnt;        // 2 x kTailMaxWarps per-warp InMIS counts, by solve parity
  HostRes *pack;            // non-null: also leave the solve's results in mapped host memory
  const int32_t *perm;      // solve id -> caller id (relabeled graphs), else null;
  uint8_t *mis_o;           // ... and, when kept, the membership in the caller's
                            // order, which the count pass and the compaction
                            // stream instead of the solve-order states
  // a solve that starts in the tail (round 1): its list is the non-isolated
  // vertices, and round 1's statistics also hold the isolated candidates
  // k_priorities marked (ctrl->sel, their segment flags)
  const int32_t *nz;
  int32_t nz_count;
  int nz_identity;
  // degree-class bounds of a degree-ordered H2 solve (common.cuh
  // class_bounds), or null: a row entry below its row's lo has a lower key,
  // and so has every entry before it (sorted rows), so a scan from the row's
  // end stops there
  const int2 *cb;
  int q_l1;        // 0: every q gather from L2 (TCMIS_TAIL_Q_L2, an A/B knob), 1: see tail_q
  int tag_par;     // A/B knob (TCMIS_TAIL_TAG_PAR): tag loaded with the L2 q (tail_blocks)
  int bar_fenced;  // 1: the __threadfence grid barrier (TCMIS_TAIL_BAR_FENCE, an A/B knob)
};

__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu(unsigned long long *p,
                                                                  unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(p), "l"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier whose arrival also sums one value per block: bar[0..1] is a
// u64 word (arrivals << 40 | sum), bar[2] the generation word (gen << 1 |
// "the sum was 0").  The last block to arrive resets the word and publishes
// the next generation with the flag, so the waiting blocks learn the sum's
// verdict from the very load that releases them.  Returns the flag.
// Ordering: the block's writes precede thread 0's arrival by the block
// barrier; the arrival is an acq_rel atomic and the release of the next
// generation a st.release, which the waiters' ld.acquire observes -- no
// separate fence.sc (`fenced`: the __threadfence form, an A/B knob).
__device__ __forceinline__ bool grid_barrier_sum(unsigned *bar, unsigned x, bool fenced = false) {
  __shared__ unsigned s_flag;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long *word = reinterpret_cast<unsigned long long *>(bar);
    unsigned res;
    if (fenced) {
      volatile unsigned *gen = bar + 2;
      const unsigned g = *gen;
      __threadfence();
      const unsigned long long old = atomicAdd(word, (1ull << 40) | (unsigned long long)x);
      if ((unsigned)(old >> 40) == gridDim.x - 1) {
        const unsigned long long sum = (old & ((1ull << 40) - 1)) + x;
        *word = 0;
        __threadfence();
        res = (((g >> 1) + 1u) << 1) | (sum == 0 ? 1u : 0u);
        atomicExch(bar + 2, res);
      } else {
        while (((res = *gen) >> 1) == (g >> 1)) __nanosleep(32);
      }
      __threadfence();
    } else {
      const unsigned g = ld_acquire_gpu(bar + 2);
      const unsigned long long old = atom_add_acq_rel_gpu(word, (1ull << 40) | (unsigned long long)x);
      if ((unsigned)(old >> 40) == gridDim.x - 1) {
        const unsigned long long sum = (old & ((1ull << 40) - 1)) + x;
        *(volatile unsigned long long *)word = 0;
        res = (((g >> 1) + 1u) << 1) | (sum == 0 ? 1u : 0u);
        st_release_gpu(bar + 2, res);
      } else {
        while (((res = ld_acquire_gpu(bar + 2)) >> 1) == (g >> 1)) __nanosleep(32);
      }
    }
    s_flag = res & 1u;
  }
  __syncthreads();
  return s_flag != 0;
}

// The compaction's range of warp gw: 16-vertex units, contiguous per warp.
struct WarpRange {
  int64_t lo, hi;  // vertices [lo, hi)
  int32_t len;     // vertices per warp (a multiple of 16)
};
__device__ __forceinline__ WarpRange warp_range(int32_t n, int nwarps, int gw) {
  const int64_t units = ((int64_t)n + 15) / 16;
  const int64_t per = (units + nwarps - 1) / nwarps;
  WarpRange r;
  r.len = (int32_t)(per * 16);
  r.lo = min((int64_t)n, (int64_t)gw * per * 16);
  r.hi = min((int64_t)n, r.lo + per * 16);
  return r;
}

// A candidate of the tail: InMIS, its compaction range counted, and for the
// tile counter of seg_mode 1 its block column queued in the block's pending
// list: the next pass decides (atomicMax on segmark) whether it is the
// round's first candidate there and adds the column's tiles, off the
// critical path (the atomic's round trip and the tile-count load used to
// sit between a candidate and the block's next barrier).  next[] is not
// written: it keeps marking the per-round kernels' candidates, which the
// compaction's count pass reads while the tail runs.
__device__ __forceinline__ void tail_candidate(const TailArgs &a, int32_t v, int32_t o,
                                               unsigned *wcnt, int32_t wlen,
                                               unsigned long long &sel, int32_t *pend,
                                               int *npend) {
  // o: the caller's id of v (relabeled graphs), kept with the list entry so
  // no permutation load sits between a decision and the block's barrier
  a.state[v] = TCMIS_IN_MIS;
  // 2, not 1: the count pass (other blocks may still be in it) counts the
  // per-round kernels' 1s; the compaction takes every non-zero byte
  if (a.mis_o) a.mis_o[o] = 2;
  if (!a.perm || a.mis_o) atomicAdd(&wcnt[o / wlen], 1u);
  ++sel;
  const int32_t sb = seg_of(o, a.T);
  if (a.seg_mode == 2) {
    a.segflag[sb] = 1;
  } else if (a.seg_mode == 1) {
    pend[atomicAdd(npend, 1)] = sb;
  }
}

// q[u] during the tail.  The tail never redraws priorities (no luby-fresh
// here), so q only falls, once, from its key summary to 0 (mark_removed): a 0
// read through the SM's L1 (ld.global.nc) is final, and only a non-zero one
// is re-read from L2.  Most neighbours the late rounds gather left in round
// 1 -- at R-MAT s22 the pushes of round 2's 45k candidates hit the same few
// hub lines from every SM --, so those gathers stay on-chip instead of
// queueing at the one L2 slice that holds each hot line.
// (`probe` is off in solves that start in this kernel, see k_tail.)
__device__ __forceinline__ uint32_t tail_q(const TailArgs &a, int32_t u, bool probe) {
  if (probe && __ldg(&a.q[u]) == 0) return 0u;
  return __ldcg(&a.q[u]);
}

// u blocks v in round r: alive at the start of round r (q != 0, not tagged
// for round r-1), higher key; `alive` reports the first part.
__device__ __forceinline__ bool tail_blocks(const TailArgs &a, int32_t u, uint32_t tprev,
                                            bool first, bool probe, uint32_t qv, int32_t v,
                                            bool &alive) {
  alive = false;
  uint32_t qu;
  if (probe && a.tag_par) {
    // past the L1 probe the neighbour is likely alive: its L2 q and its tag
    // in one round trip
    if (__ldg(&a.q[u]) == 0) return false;
    qu = __ldcg(&a.q[u]);
    const uint16_t tu = first ? (uint16_t)0 : __ldcg(&a.xt[u]);
    if (qu == 0) return false;
    alive = first || tu != (uint16_t)tprev;
  } else {
    qu = tail_q(a, u, probe);
    if (qu == 0) return false;
    alive = first || __ldcg(&a.xt[u]) != (uint16_t)tprev;  // no tag is tag(r0 - 1)
  }
  if (!alive) return false;
  if (qu != qv) return qu > qv;
  const uint32_t pu = __ldg(&a.prio[u]), pv = __ldg(&a.prio[v]);
  return pu != pv ? pu > pv : orig_id(a.perm, u) > orig_id(a.perm, v);
}

__device__ __forceinline__ bool tail_alive(const TailArgs &a, int32_t u, uint32_t tprev,
                                           bool first, bool probe) {
  if (probe && a.tag_par) {
    if (__ldg(&a.q[u]) == 0) return false;
    const uint32_t qu = __ldcg(&a.q[u]);
    const uint16_t tu = first ? (uint16_t)0 : __ldcg(&a.xt[u]);
    return qu != 0 && (first || tu != (uint16_t)tprev);
  }
  return tail_q(a, u, probe) != 0 && (first || __ldcg(&a.xt[u]) != (uint16_t)tprev);
}

__device__ __forceinline__ unsigned long long *slot_field(const TailArgs &a, int round, int f) {
  DevRound *r = &a.rounds[(round - 1) % a.ctrl->max_rounds];
  return f == 0 ? &r->sel : f == 1 ? &r->rem : f == 2 ? &r->alive : &r->eval;
}

// 16 states (or decision bytes) -> bit j set iff byte j == val
__device__ __forceinline__ uint32_t eq_mask16(uint4 w, uint32_t val) {
  const uint32_t x[4] = {w.x, w.y, w.z, w.w};
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t e = __vcmpeq4(x[k], val * 0x01010101u);  // 0xff per equal byte
#pragma unroll
    for (int j = 0; j < 4; ++j) m |= ((e >> (8 * j + 7)) & 1u) << (4 * k + j);
  }
  return m;
}

// Ascending ids of the InMIS vertices (the reference sorts result.mis,
// engine.cpp:293).  Warp gw of the grid owns a contiguous vertex range; its
// InMIS count is known without a pass at the end: the count pass at the
// tail's start counted the per-round kernels' candidates (next == 1, which
// the tail never writes) and every tail candidate added itself (atomic on its
// range).  After the rounds' last grid barrier every block sums the counts
// before it, and every warp writes its range's ids on its own: 16 states per
// lane per step (16-byte loads, the next step's prefetched), ids staged in
// the warp's shared-memory slice and copied out coalesced.  No block barrier
// inside the write loop, no grid barrier at all (the previous version counted
// per block at the end: a count pass plus a grid barrier, 6 us at s22).
__device__ void compact_mis(const TailArgs &a, unsigned *wcnt, unsigned *wnext, int32_t *stage) {
  __shared__ unsigned long long s_base;
  __shared__ unsigned s_woff[kTailWarps + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nwarps = gridDim.x * kTailWarps;
  const int gw = blockIdx.x * kTailWarps + w;
  unsigned long long before = 0;
  for (int j = threadIdx.x; j < blockIdx.x * kTailWarps; j += kTailBlock) before += __ldcg(&wcnt[j]);
  for (int o = 16; o; o >>= 1) before += __shfl_down_sync(0xffffffffu, before, o);
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  if (lane == 0 && before) atomicAdd(&s_base, before);
  if (w == 0) {  // exclusive scan of the block's 32 warp counts
    static_assert(kTailWarps == 32, "one warp count per lane");
    static_assert(kTailWarps * kCompactV >= kTailBlock * kThrScan, "staging holds the windows");
    const unsigned t = __ldcg(&wcnt[blockIdx.x * kTailWarps + lane]);
    unsigned sc = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, sc, o);
      if (lane >= o) sc += y;
    }
    s_woff[lane] = sc - t;
    if (lane == 31) s_woff[32] = sc;
  }
  __syncthreads();
  int64_t base = (int64_t)s_base + s_woff[w];
  const WarpRange R = warp_range(a.n, nwarps, gw);
  int32_t *stg = stage + w * kCompactV;
  uint4 xn = make_uint4(0, 0, 0, 0);
  const uint8_t *memb = a.mis_o ? a.mis_o : a.state;  // InMIS == 1 in both
  if (R.lo + lane * 16 < R.hi)
    xn = __ldcg(reinterpret_cast<const uint4 *>(memb + R.lo + lane * 16));
  for (int64_t t0 = R.lo; t0 < R.hi; t0 += kCompactV) {
    const int64_t v0 = t0 + lane * 16;
    const uint4 x = xn;
    if (v0 + kCompactV < R.hi)
      xn = __ldcg(reinterpret_cast<const uint4 *>(memb + v0 + kCompactV));
    uint32_t m = 0;
    if (v0 < R.hi) {
      // states: InMIS; a relabeled solve's membership plane: 1 (per-round
      // kernels) or 2 (this kernel)
      m = a.mis_o ? (0xffffu & ~eq_mask16(x, 0u)) : eq_mask16(x, TCMIS_IN_MIS);
      const int64_t left = R.hi - v0;
      if (left < 16) m &= (1u << left) - 1u;
    }
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int k = incl - c;
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      stg[k++] = (int32_t)(v0 + bit);
    }
    __syncwarp();
    for (int i = lane; i < total; i += 32) a.mis[base + i] = stg[i];
    base += total;
    __syncwarp();
  }
  if (lane == 0) wnext[gw] = 0;  // the next solve's buffer (this one's is read by other blocks)
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
    const long long total = (long long)s_base + s_woff[kTailWarps];
    *a.mis_count = total;
    if (a.pack) a.pack->mis_count = total;
  }
}

#ifndef TCMIS_TAIL_MINB
#define TCMIS_TAIL_MINB 1
#endif
__global__ void __launch_bounds__(kTailBlock, TCMIS_TAIL_MINB) k_tail(TailArgs a) {
  extern __shared__ int32_t s_stage[];  // kTailDynSmem: compact_mis's staging
  // the block's list: entry k = (id, row extent, q), handled by thread k
  __shared__ int32_t s_v[kTailBlock];
  __shared__ int32_t s_o[kTailBlock];  // the entry's caller id (relabeled graphs; else = s_v)
  __shared__ int64_t s_s[kTailBlock], s_e[kTailBlock];
  __shared__ uint16_t s_q[kTailBlock];
  __shared__ uint8_t s_keep[kTailBlock];  // the entry's verdict: 1 = non-candidate
  // a deferred entry's thread-phase windows: their alive neighbours (bit j of
  // s_live[k] = s_stage[k * kThrScan + j]; the compaction's staging area is
  // free until the rounds end), so the group neither re-gathers them nor
  // rescans them to push
  __shared__ uint32_t s_live[kTailBlock];
  __shared__ int16_t s_def[kTailBlock];   // entries left to the groups
  __shared__ int16_t s_long[kTailLongCap];  // ... and to the whole block
  __shared__ int32_t s_lo[kTailBlock];      // the entry's class lower bound (0: none)
  // candidates whose row below the examined part is still to be pushed: the
  // entries [s_s, s_e) of every listed entry, flattened over the whole block
  // (list and offsets in the staging area's upper half, which s_live's
  // windows leave free during the rounds)
  long long *s_pofs = reinterpret_cast<long long *>(s_stage + kTailBlock * kThrScan);
  int16_t *s_pk = reinterpret_cast<int16_t *>(s_pofs + kTailBlock + 1);
  __shared__ int s_nd, s_nlong, s_nl, s_np;
  __shared__ int32_t s_pend[2][kTailBlock];  // candidates' block columns (seg_mode 1), by round parity
  __shared__ int s_npend[2];
  __shared__ unsigned long long s_acc[4];
  Ctrl *ctrl = a.ctrl;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gl = lane & (kGroup - 1);
  const unsigned gmask = (kGroup == 32 ? 0xffffffffu : ((1u << kGroup) - 1u)) << (lane & ~(kGroup - 1));
  const int grp = threadIdx.x / kGroup;
  constexpr int kW = kGroup * kTU;  // entries per group step
  if (threadIdx.x < 4) s_acc[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    s_nd = 0;
    s_nlong = 0;
    s_nl = 0;
    s_np = 0;
    s_npend[0] = s_npend[1] = 0;
  }
  const uint32_t base0 = __ldcg(&a.tslot[0]);
  const uint32_t solve = __ldcg(&a.tslot[1]);
  const int nwarps = gridDim.x * kTailWarps;
  unsigned *wcnt = a.warpcnt + (solve & 1u) * kTailMaxWarps;
  unsigned *wnext = a.warpcnt + ((solve + 1u) & 1u) * kTailMaxWarps;
  const int32_t wlen = warp_range(a.n, nwarps, 0).len;
  if (*(volatile int *)&ctrl->corrupt) {
    // the per-round kernels flagged corrupt state (update.cuh): no rounds
    // (the list may not fit the blocks), just the control block for the host
    if (blockIdx.x == gridDim.x - 1 && a.pack) {
      const uint32_t *cs = reinterpret_cast<const uint32_t *>(a.ctrl);
      uint32_t *cd = reinterpret_cast<uint32_t *>(&a.pack->ctrl);
      for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += kTailBlock) cd[i] = __ldcg(cs + i);
      __threadfence_system();
    }
    return;
  }
  const int r0 = *(volatile int *)&ctrl->round;
  const bool from1 = r0 == 1;  // the whole solve in this kernel
  const int64_t cnt0 = from1 ? a.nz_count : *(volatile int *)&ctrl->wl_count[r0 & 1];
  if (from1) {
    // round 1's isolated candidates (k_priorities): their count, and for the
    // seg_mode-1 tile counters their block columns, marked as counted in
    // round 1 so that the round's own candidates there add nothing twice
    if (blockIdx.x == 0 && threadIdx.x == 0 && ctrl->sel)
      atomicAdd(slot_field(a, 1, 0), (unsigned long long)ctrl->sel);
    if (a.seg_mode == 1) {
      unsigned long long ev = 0;
      for (int64_t sb = blockIdx.x * (int64_t)kTailBlock + threadIdx.x; sb < a.nseg;
           sb += (int64_t)gridDim.x * kTailBlock)
        if (a.segflag[sb]) {
          a.segmark[sb] = 1u;
          ev += (unsigned long long)__ldg(&a.rowtiles[sb]);
        }
      ev = __reduce_add_sync(0xffffffffu, (unsigned)ev);
      if ((threadIdx.x & 31) == 0 && ev) atomicAdd(slot_field(a, 1, 3), ev);
    }
  }
  TAIL_MARK(1, cnt0);
  // the block's share of the starting list (<= kTailBlock entries: host
  // cap): entries b, b + G, b + 2G, ... -- interleaved, because the list's
  // order is not random (its end holds the rows the round kernels' engines
  // finished last, the longer ones; contiguous slices left the last blocks
  // ~30 % more work at s22)
  int nl = cnt0 > blockIdx.x ? (int)((cnt0 - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  {
    const int32_t *in0 = (r0 & 1) ? a.wl1 : a.wl0;
    if (threadIdx.x < nl) {
      const int64_t idx = blockIdx.x + (int64_t)threadIdx.x * gridDim.x;
      const int32_t v = !from1 ? __ldcg(&in0[idx]) : a.nz_identity ? (int32_t)idx : __ldg(&a.nz[idx]);
      s_v[threadIdx.x] = v;
      s_o[threadIdx.x] = a.perm ? __ldg(&a.perm[v]) : v;
      const int64_t rs = __ldg(&a.off[v]), re = __ldg(&a.off[v + 1]);
      s_s[threadIdx.x] = rs;
      s_e[threadIdx.x] = re;
      s_q[threadIdx.x] = __ldcg(&a.q[v]);
      s_lo[threadIdx.x] = class_bounds(a.cb, re - rs).x;
    }
  }
  // the fused compaction runs in the caller's id order: on the states, or on
  // a relabeled solve's caller-order membership; a relabeled solve without
  // one compacts after the tail (solver.cu, a gather through the permutation)
  const bool compact = !a.perm || a.mis_o;
  if (compact) {  // count pass: the per-round kernels' candidates in this warp's range
     // (next == 1, or the caller-order membership)
    const uint8_t *cand = a.mis_o ? a.mis_o : a.next;
    const WarpRange R = warp_range(a.n, nwarps, blockIdx.x * kTailWarps + w);
    unsigned c = 0;
#pragma unroll 4
    for (int64_t v0 = R.lo + lane * 16; v0 < R.hi; v0 += 32 * 16) {
      uint32_t m = eq_mask16(__ldcg(reinterpret_cast<const uint4 *>(cand + v0)), 1u);
      const int64_t left = R.hi - v0;
      if (left < 16) m &= (1u << left) - 1u;
      c += __popc(m);
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if (lane == 0 && c) atomicAdd(&wcnt[blockIdx.x * kTailWarps + w], c);
  }
  uint32_t base = base0;
  if (base0 >= kTagWrap && cnt0 > 0) {
    // once every ~4e9 rounds: clear the tags of the vertices alive at the
    // start (every later list is a subset) and restart the tags at 1
    __syncthreads();
    if (threadIdx.x < nl) a.xt[s_v[threadIdx.x]] = 0;
    base = 0;
    grid_barrier_sum(a.bar, 1, a.bar_fenced);
  }
  TAIL_MARK(8, 0);
  int round = r0;
  bool done = cnt0 == 0;
  if (done) grid_barrier_sum(a.bar, 0, a.bar_fenced);  // the count pass must be complete before the compaction
  __syncthreads();                       // the list's shared-memory fill
  for (; !done; ++round) {
    if (round - r0 >= kMaxTailRounds) {  // uniform: the ring overflows, the host re-runs step-wise
      if (blockIdx.x == 0 && threadIdx.x == 0) ctrl->overflow = 1;
      break;
    }
    const bool first = round == r0;
    // tail_q's L1 probe: on when the tail takes over from the round kernels
    // (most neighbours are gone by then); a solve run here from round 1 (small
    // graphs: ER 100k keeps a quarter of its vertices alive into round 2) would
    // only pay the probe's extra round trip (ER k_tail 87 -> 94 us with it)
    const bool probe = a.q_l1 && !from1;
#ifdef TCMIS_TAIL_PROF
    if (first && threadIdx.x == 0) g_tail_blk[4][blockIdx.x] = gtimer();
#endif
    const uint32_t tprev = base + 1u + (uint32_t)(round - r0);  // tag(round - 1)
    const uint32_t tcur = tprev + 1u;                           // tag(round)
    if (blockIdx.x == 0 && threadIdx.x == 0)
      a.rounds[(round - 1) % ctrl->max_rounds].t[0] = gtimer_ns();
    unsigned long long sel = 0, ev = 0, rem = 0, alive = 0;
    int32_t *pend = s_pend[round & 1];
    int *npend = &s_npend[round & 1];
    // the previous round's pending block columns: the atomic and the tile
    // count are issued now and consumed at the end of this pass
    const int kp = threadIdx.x;
    const bool have_p = !first && kp < s_npend[(round - 1) & 1];
    unsigned p_old = 0xffffffffu;
    int32_t p_tiles = 0;
    if (have_p) {
      const int32_t sb = s_pend[(round - 1) & 1][kp];
      p_old = atomicMax(&a.segmark[sb], (unsigned)(round - 1));
      p_tiles = __ldg(&a.rowtiles[sb]);
    }
    const int k = threadIdx.x;
    const bool have = k < nl;
    // a handful of entries: one warp per entry, not the thread + group pair
    // (two dependent scans where one suffices for a round of few vertices)
    const bool small = nl <= kTailWarps;
    int32_t v = -1, o = -1, lo = 0;
    int64_t s = 0, e = 0;
    uint32_t qv = 0;
    uint8_t keep = 0;
    if (have) {
      v = s_v[k];
      o = s_o[k];
      s = s_s[k];
      e = s_e[k];
      qv = s_q[k];
      lo = s_lo[k];
    }
    if (small && w < nl) {
      if (lane == 0) {
        s_keep[w] = 0;
        s_live[w] = 0;
      }
      const int32_t wv = s_v[w];
      const int64_t ws = s_s[w], we = s_e[w];
      const uint32_t wq = s_q[w];
      const uint32_t tv = first ? 0u : __ldcg(&a.xt[wv]);
      if (we - ws > kTailLong && !(!first && tv == (uint16_t)tprev)) {
        if (lane == 0) {
          ++alive;
          const int kk = atomicAdd(&s_nlong, 1);  // < kTailWarps <= kTailLongCap
          s_long[kk] = (int16_t)w;
        }
      } else {
        int32_t u[kTU];
#pragma unroll
        for (int j = 0; j < kTU; ++j) {
          const int64_t idx = we - 1 - lane - 32 * j;
          u[j] = idx >= ws ? __ldg(&a.nbr[idx]) : -1;
        }
        if (!first && tv == (uint16_t)tprev) {  // excluded in round - 1
          if (lane == 0) {
            mark_removed(wv, a.state, a.q);
            ++rem;
          }
        } else {
          if (lane == 0) ++alive;
          constexpr int64_t kWW = 32 * kTU;
          bool blocked = false;
          uint32_t live = 0;
          const int32_t wlo = s_lo[w];
          for (int64_t top = we;;) {
            bool b = false, bl = false;
            live = 0;
#pragma unroll
            for (int j = 0; j < kTU; ++j)
              if (u[j] >= 0) {
                bool al;
                b |= tail_blocks(a, u[j], tprev, first, probe, wq, wv, al);
                live |= (uint32_t)al << j;
                bl |= u[j] < wlo;
              }
            blocked = __any_sync(0xffffffffu, b);
            top -= kWW;
            // below the class bound: nothing further down can block
            if (blocked || top <= ws || __any_sync(0xffffffffu, bl)) break;
#pragma unroll
            for (int j = 0; j < kTU; ++j) {
              const int64_t idx = top - 1 - lane - 32 * j;
              u[j] = idx >= ws ? __ldg(&a.nbr[idx]) : -1;
            }
          }
          if (!blocked) {
            if (lane == 0) tail_candidate(a, wv, s_o[w], wcnt, wlen, sel, pend, npend);
            if (we - ws <= kWW) {
#pragma unroll
              for (int j = 0; j < kTU; ++j)
                if ((live >> j) & 1u) a.xt[u[j]] = (uint16_t)tcur;
            } else {
              for (int64_t top = we; top > ws; top -= kWW) {
#pragma unroll
                for (int j = 0; j < kTU; ++j) {
                  const int64_t idx = top - 1 - lane - 32 * j;
                  u[j] = idx >= ws ? __ldg(&a.nbr[idx]) : -1;
                }
#pragma unroll
                for (int j = 0; j < kTU; ++j)
                  if (u[j] >= 0 && tail_alive(a, u[j], tprev, first, probe)) a.xt[u[j]] = (uint16_t)tcur;
              }
            }
          } else if (lane == 0) {
            s_keep[w] = 1;
          }
        }
      }
    }
    if (have && !small) {
      // 1. the entry's tag and the last kThrScan row entries, loaded together
      const uint32_t tv = first ? 0u : __ldcg(&a.xt[v]);  // loaded with the row entries
      // the row's last kThrScan/4 aligned 16-byte windows (13-16 entries):
      // one wavefront per lane and window instead of one per entry
      int32_t u[kThrScan];
      int64_t hi = e;
#pragma unroll
      for (int j = 0; j < kThrScan / 4; ++j) {
        if (hi > s) {
          hi = load_window_down(a.nbr, a.vnnz, s, hi, &u[4 * j]);
        } else {
          u[4 * j] = u[4 * j + 1] = u[4 * j + 2] = u[4 * j + 3] = -1;
        }
      }
      if (!first && tv == (uint16_t)tprev) {  // excluded in round - 1
        mark_removed(v, a.state, a.q);
        ++rem;
      } else {
        ++alive;
        bool b = false, below = false;
        uint32_t live = 0;
        if (first && from1 && a.cb) {
          // a solve's round 1 here: everybody is alive, so an entry at or
          // above the row's upper class bound blocks without a gather
          const int32_t hb = class_bounds(a.cb, e - s).y;
#pragma unroll
          for (int j = 0; j < kThrScan; ++j) b |= u[j] >= hb;
        }
        if (!b) {
#pragma unroll
          for (int j = 0; j < kThrScan; ++j)
            if (u[j] >= 0) {
              bool al;
              b |= tail_blocks(a, u[j], tprev, first, probe, qv, v, al);
              live |= (uint32_t)al << j;
              below |= u[j] < lo;
            }
        }
        if (b) {
          keep = 1;
        } else if (hi <= s || below) {  // the whole row, or all of it that could block
          tail_candidate(a, v, o, wcnt, wlen, sel, pend, npend);
#pragma unroll
          for (int j = 0; j < kThrScan; ++j)
            if ((live >> j) & 1u) a.xt[u[j]] = (uint16_t)tcur;
          if (hi > s) {  // the rest of the row: the block's flat push below
            s_pk[atomicAdd(&s_np, 1)] = (int16_t)k;
            s_e[k] = hi;
          }
        } else {
          s_def[atomicAdd(&s_nd, 1)] = (int16_t)k;
          s_e[k] = hi;  // the group scans [s, hi): [hi, e) was examined here
          s_live[k] = live;
          int32_t *su = s_stage + k * kThrScan;
#pragma unroll
          for (int j = 0; j < kThrScan; ++j)
            if ((live >> j) & 1u) su[j] = u[j];
        }
      }
      s_keep[k] = keep;
    }
    __syncthreads();
    TAIL_MARK(9, s_nd);
#ifdef TCMIS_TAIL_PROF
    if (first && threadIdx.x == 0) {
      g_tail_blk[0][blockIdx.x] = gtimer();
      g_tail_blk[2][blockIdx.x] = (unsigned long long)s_nd;
      g_tail_blk[3][blockIdx.x] = (unsigned long long)nl;
    }
#endif
    // 2. the deferred rows: kGroup lanes each, over the part of the row the
    // thread did not examine (a part of <= kW entries pushes from registers)
    const int nd = s_nd;
    for (int d = grp; d < nd; d += kTailGroups) {
      const int kd = s_def[d];
      const int32_t dv = s_v[kd];
      const int64_t ds = s_s[kd], de = s_e[kd];
      if (de - ds > kTailLong) {
        int listed = 0;
        if (gl == 0) {
          const int kk = atomicAdd(&s_nlong, 1);
          if (kk < kTailLongCap) {
            s_long[kk] = (int16_t)kd;
            listed = 1;
          }
        }
        if (__shfl_sync(gmask, listed, lane & ~(kGroup - 1))) continue;
      }
      const uint32_t dq = s_q[kd];
      const int32_t dlo = s_lo[kd];
      bool blocked = false, stop = false;
      int32_t u[kTU];
      uint32_t live = 0;
      for (int64_t top = de; top > ds && !blocked && !stop; top -= kW) {
#pragma unroll
        for (int j = 0; j < kTU; ++j) {
          const int64_t idx = top - 1 - gl - kGroup * j;
          u[j] = idx >= ds ? __ldg(&a.nbr[idx]) : -1;
        }
        bool b = false, bl = false;
        live = 0;
#pragma unroll
        for (int j = 0; j < kTU; ++j)
          if (u[j] >= 0) {
            bool al;
            b |= tail_blocks(a, u[j], tprev, first, probe, dq, dv, al);
            live |= (uint32_t)al << j;
            bl |= u[j] < dlo;
          }
        blocked = __ballot_sync(gmask, b) != 0;
        stop = __ballot_sync(gmask, bl) != 0;  // below the class bound
      }
      if (!blocked) {
        if (gl == 0) tail_candidate(a, dv, s_o[kd], wcnt, wlen, sel, pend, npend);
        const uint32_t sl = s_live[kd];
        for (int j = gl; j < kThrScan; j += kGroup)
          if ((sl >> j) & 1u) a.xt[s_stage[kd * kThrScan + j]] = (uint16_t)tcur;
        if (de - ds <= kW) {  // one step held the whole part
#pragma unroll
          for (int j = 0; j < kTU; ++j)
            if ((live >> j) & 1u) a.xt[u[j]] = (uint16_t)tcur;
        } else if (gl == 0) {  // [ds, de): the block's flat push below
          s_pk[atomicAdd(&s_np, 1)] = (int16_t)kd;
        }
      } else if (gl == 0) {
        s_keep[kd] = 1;
      }
    }
    __syncthreads();
    TAIL_MARK(10, s_nlong);
    // 3. rows above kTailLong: the whole block, kBU entries per thread and
    // step (a row of <= kBU * kTailBlock entries pushes from registers)
    const int nlong = min(s_nlong, kTailLongCap);
    for (int kk = 0; kk < nlong; ++kk) {
      const int kd = s_long[kk];
      const int32_t dv = s_v[kd];
      const int64_t ds = s_s[kd], de = s_e[kd];
      const uint32_t dq = s_q[kd];
      const int32_t dlo = s_lo[kd];
      constexpr int kBU = 8;
      constexpr int64_t kBW = (int64_t)kBU * kTailBlock;
      bool blocked = false, stop = false;
      int32_t x[kBU];
      uint32_t live = 0;
      for (int64_t top = de; top > ds && !blocked && !stop; top -= kBW) {
#pragma unroll
        for (int j = 0; j < kBU; ++j) {
          const int64_t idx = top - 1 - threadIdx.x - (int64_t)kTailBlock * j;
          x[j] = idx >= ds ? __ldg(&a.nbr[idx]) : -1;
        }
        bool b = false, bl = false;
        live = 0;
#pragma unroll
        for (int j = 0; j < kBU; ++j)
          if (x[j] >= 0) {
            bool al;
            b |= tail_blocks(a, x[j], tprev, first, probe, dq, dv, al);
            live |= (uint32_t)al << j;
            bl |= x[j] < dlo;
          }
        blocked = __syncthreads_or(b) != 0;
        stop = __syncthreads_or(bl) != 0;  // below the class bound
      }
      if (!blocked) {
        if (threadIdx.x == 0) tail_candidate(a, dv, s_o[kd], wcnt, wlen, sel, pend, npend);
        if (threadIdx.x < kThrScan && ((s_live[kd] >> threadIdx.x) & 1u))
          a.xt[s_stage[kd * kThrScan + threadIdx.x]] = (uint16_t)tcur;
        if (de - ds <= kBW) {
#pragma unroll
          for (int j = 0; j < kBU; ++j)
            if ((live >> j) & 1u) a.xt[x[j]] = (uint16_t)tcur;
        } else if (threadIdx.x == 0) {  // [ds, de): the flat push below
          s_pk[atomicAdd(&s_np, 1)] = (int16_t)kd;
        }
      } else if (threadIdx.x == 0) {
        s_keep[kd] = 1;
      }
    }
    __syncthreads();  // the push list is complete
    TAIL_MARK(11, s_np);
    // 4. the candidates' rows beyond their examined part, flattened over the
    // block: each thread takes every kTailBlock-th entry of the concatenation
    // (neighbouring threads read neighbouring row entries), kPU of them per
    // step with their loads in flight together; alive neighbours get tag(round)
    long long ptotal = 0;
    if (const int np = s_np) {
      using Scan = cub::BlockScan<long long, kTailBlock, cub::BLOCK_SCAN_WARP_SCANS>;
      __shared__ typename Scan::TempStorage s_scan;
      const long long len = threadIdx.x < np ? s_e[s_pk[threadIdx.x]] - s_s[s_pk[threadIdx.x]] : 0;
      long long incl;
      Scan(s_scan).InclusiveSum(len, incl);
      s_pofs[threadIdx.x + 1] = incl;
      if (threadIdx.x == 0) s_pofs[0] = 0;
      __syncthreads();
      const long long total = s_pofs[np];
      ptotal = total;
      constexpr int kPU = 8;
      for (long long j0 = threadIdx.x; j0 < total; j0 += (long long)kPU * kTailBlock) {
        int32_t x[kPU];
#pragma unroll
        for (int p = 0; p < kPU; ++p) {
          const long long j = j0 + (long long)p * kTailBlock;
          x[p] = -1;
          // the warp's 32 entries are consecutive: the row of its first entry
          // by a warp-uniform binary search (broadcast reads), then each lane
          // steps over the few row starts between it and its own entry (a
          // per-lane search read 10 scattered 8-byte words per entry: bank
          // conflicts made it the push's cost)
          const long long jw = j - (threadIdx.x & 31);
          if (jw < total) {
            int lo = 0, hi = np - 1;  // the last listed row whose offset <= jw
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (s_pofs[mid] <= jw) lo = mid; else hi = mid - 1;
            }
            if (j < total) {
              while (lo < np - 1 && s_pofs[lo + 1] <= j) ++lo;
              x[p] = __ldg(&a.nbr[s_s[s_pk[lo]] + (j - s_pofs[lo])]);
            }
          }
        }
#pragma unroll
        for (int p = 0; p < kPU; ++p)
          if (x[p] >= 0 && tail_alive(a, x[p], tprev, first, probe)) a.xt[x[p]] = (uint16_t)tcur;
      }
    }
    TAIL_MARK(12, ptotal);
#ifdef TCMIS_TAIL_PROF
    if (first && threadIdx.x == 0) g_tail_blk[1][blockIdx.x] = gtimer();
#endif
    if (have_p && p_old < (unsigned)(round - 1)) ev += (unsigned long long)p_tiles;
    // 4. the round's counters: fire-and-forget atomics into the ring
    // (round: sel; round - 1: rem, alive and -- from the pending columns -- eval)
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
    __syncthreads();  // s_keep, s_acc complete; the entry arrays are read no more
    if (threadIdx.x == 0) {
      if (s_acc[0]) atomicAdd(slot_field(a, round, 0), s_acc[0]);
      if (!first) {
        if (s_acc[1]) atomicAdd(slot_field(a, round - 1, 3), s_acc[1]);
        if (s_acc[2]) atomicAdd(slot_field(a, round - 1, 1), s_acc[2]);
        if (s_acc[3]) atomicAdd(slot_field(a, round - 1, 2), s_acc[3]);
      }
      s_acc[0] = s_acc[1] = s_acc[2] = s_acc[3] = 0;
      s_nd = 0;
      s_nlong = 0;
      s_np = 0;
      s_npend[(round + 1) & 1] = 0;  // the next round's list (round - 1's was read above)
    }
    // 5. the block's survivors (round's non-candidates) stay with it
    if (have && s_keep[k]) {
      const int j = atomicAdd(&s_nl, 1);
      s_v[j] = v;
      s_o[j] = o;
      s_s[j] = s;
      s_e[j] = e;
      s_q[j] = (uint16_t)qv;
      s_lo[j] = lo;
    }
    __syncthreads();
    nl = s_nl;
    TAIL_MARK(2, nl);
    done = grid_barrier_sum(a.bar, (unsigned)nl, a.bar_fenced);
    if (threadIdx.x == 0) s_nl = 0;
    TAIL_MARK(3, round);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const unsigned long long t = gtimer_ns();
      DevRound *r = &a.rounds[(round - 1) % ctrl->max_rounds];
      r->t[1] = r->t[2] = r->t[3] = t;
    }
  }
  // every block has passed the last round's barrier: states and counts are
  // final but for the last pass's pending block columns (seg_mode 1)
  {
    const int np = s_npend[(round - 1) & 1];
    unsigned long long ev = 0;
    if (threadIdx.x < np) {
      const int32_t sb = s_pend[(round - 1) & 1][threadIdx.x];
      if (atomicMax(&a.segmark[sb], (unsigned)(round - 1)) < (unsigned)(round - 1))
        ev = (unsigned long long)__ldg(&a.rowtiles[sb]);
    }
    ev = __reduce_add_sync(0xffffffffu, (unsigned)ev);
    if (lane == 0 && ev) atomicAdd(slot_field(a, round - 1, 3), ev);
    __syncthreads();
    if (threadIdx.x == 0) {  // arrival for the publishing block (below), nobody waits here
      __threadfence();
      atomicAdd(&a.bar[3], 1u);
    }
  }
  TAIL_MARK(4, 0);
  if (compact) {
    compact_mis(a, wcnt, wnext, s_stage);
  } else if (lane == 0) {
    wnext[blockIdx.x * kTailWarps + w] = 0;  // the next solve's count buffer, as compact_mis does
  }
  TAIL_MARK(7, 0);
  // The last block publishes the tail's rounds and packs the control block
  // and the ring for the host, once every block's counters are in.  Pass
  // `round - 1` was the last one run; it was a round of the reference iff it
  // had an alive vertex, i.e. selected one (a pass of only removals closes
  // round - 2).  Its non-candidates were 0, so the ring's zeroed rem / alive
  // of that round are already right.
  if (blockIdx.x != gridDim.x - 1) return;
  if (threadIdx.x == 0) {
    while (*(volatile unsigned *)&a.bar[3] < gridDim.x) __nanosleep(32);
    a.bar[3] = 0;
    __threadfence();
    a.tslot[0] = base + 2u + (uint32_t)(round - r0);  // one past every tag this solve used
    a.tslot[1] = solve + 1u;
    volatile Ctrl *vc = ctrl;
    const int cap = vc->max_rounds;
    int last = round - 1;  // last pass
    if (last >= r0 && ((volatile DevRound *)&a.rounds[(last - 1) % cap])->sel == 0) --last;
    unsigned long long before = (unsigned long long)vc->alive;  // alive at the start of r0
    for (int r = r0; r <= last; ++r) {
      volatile DevRound *pr = &a.rounds[(r - 1) % cap];
      const unsigned long long evp = pr->eval;
      pr->eval = a.seg_mode == 1 ? evp : 0;
      pr->skip = a.seg_mode == 1 ? (unsigned long long)a.total_tiles - evp : 0;
      // engine.cpp:138-160 invariant, as in round_end_tail (update.cuh)
      if (before != pr->sel + pr->rem + pr->alive) vc->corrupt = 1;
      before = pr->alive;
    }
    if (last >= r0) {
      if (last > cap) vc->overflow = 1;
      vc->alive = 0;
      vc->round = last + 1;
    }
    __threadfence();
  }
  __syncthreads();
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
    __threadfence_system();
  }
}

}  // namespace tcmis_b200
