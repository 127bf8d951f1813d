// common.cuh -- device helpers shared by the round kernels.
#pragma once

#include "internal.cuh"

namespace tcmis_b200 {

constexpr int kBlock = 256;    // threads per block of the round kernels
constexpr int kStep = 4;       // row entries per thread-level step
#ifndef TCMIS_THREAD_MAX
#define TCMIS_THREAD_MAX 64
#endif
constexpr int kThreadMax = TCMIS_THREAD_MAX;  // entries a thread examines before handing a row to a warp
// the per-lane scan engines read two 16-byte windows (8 entries) per step
#ifndef TCMIS_SEL_WIN2
#define TCMIS_SEL_WIN2 1
#endif
// 16-byte windows per step of the per-lane scan engines (k_select, k_update_pull)
#ifndef TCMIS_SEL_WIN
#define TCMIS_SEL_WIN (TCMIS_SEL_WIN2 ? 2 : 1)
#endif
constexpr int kSelWin = TCMIS_SEL_WIN;
#ifndef TCMIS_WARP_U
#define TCMIS_WARP_U 8
#endif
constexpr int kWarpU = TCMIS_WARP_U;  // independent loads per lane per step of a warp-wide row scan
#ifndef TCMIS_BLOCK_ROW
#define TCMIS_BLOCK_ROW 65536
#endif
constexpr int64_t kBlockRow = TCMIS_BLOCK_ROW;  // long-row lists: rows beyond this are scanned block-wide
// pull exclusion: rows that outlive the engine are cut into chunks of this
// many entries, which k_round_end's warps take independently (update.cuh)
#ifndef TCMIS_PULL_CHUNK
#define TCMIS_PULL_CHUNK 2048
#endif
constexpr int kPullChunk = TCMIS_PULL_CHUNK;

// Programmatic dependent launch (TCMIS_PDL): the round kernels are launched
// with programmatic stream serialisation, let their successor launch at once
// and wait for their predecessor's completion before touching memory, so a
// kernel boundary costs no launch latency.  Without the launch attribute both
// instructions are no-ops.
#ifndef TCMIS_PDL
#define TCMIS_PDL 0
#endif
__device__ __forceinline__ void pdl_entry() {
#if TCMIS_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// Loads of the CSR (offsets, neighbour ids): read once per phase, so they are
// marked evict-first (ld.global.cs) and do not push the randomly gathered
// priority / state / decision vectors out of L2.
#ifndef TCMIS_STREAM_HINTS
#define TCMIS_STREAM_HINTS 1
#endif
template <typename T>
__device__ __forceinline__ T ld_stream(const T *p) {
#if TCMIS_STREAM_HINTS
  return __ldcs(p);
#else
  return __ldg(p);
#endif
}

// Phase timer of the reference (engine.cpp:253-284): block 0 stamps the
// phase's start into the round's DevRound slot (internal.cuh)
__device__ __forceinline__ void stamp_phase(DevRound *rounds, const Ctrl *ctrl, int round,
                                            int k0, int k1) {
  if (rounds && blockIdx.x == 0 && threadIdx.x == 0) {
    DevRound *r = &rounds[(round - 1) % ctrl->max_rounds];
    const unsigned long long t = gtimer_ns();
    for (int k = k0; k <= k1; ++k) r->t[k] = t;
  }
}

// per-thread work modes of the state-machine kernels
enum : int { kFetch = 0, kScan = 1, kPush = 2, kDone = 3 };

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
  __syncthreads();  // sh reuse by a later call
}

// A candidate joins the MIS (engine.cpp:137-143).  Its key is left in place:
// every neighbour of a candidate leaves in the same round, so no alive vertex
// ever reads it again.  next[v] = 1 is what neighbours test this round (and
// it is never cleared: see update.cuh).
// block column of v for tile dimension T (uniform): a shift for the usual
// power-of-two T instead of a ~20-instruction integer division
__device__ __forceinline__ int32_t seg_of(int32_t v, int T) {
  return (T & (T - 1)) == 0 ? (v >> (__ffs(T) - 1)) : v / T;
}

// The caller's id of solve id v: graphs with an internal vertex order
// (tcmis_graph_reorder) run the kernels on relabeled ids, while keys, hash
// priorities and the tile counters stay defined on the caller's ids
// (priorities.hpp:61-64, spmv.cpp:37-46); perm == null: identity.
__device__ __forceinline__ int32_t orig_id(const int32_t *perm, int32_t v) {
  return perm ? __ldg(&perm[v]) : v;
}

// A relabeled solve of an L2-sized graph also keeps the MIS membership in the
// caller's order (mis_o[caller id] = 1, one fire-and-forget byte store per
// candidate): the final ascending-id compaction then streams it like the
// unrelabeled states instead of gathering every vertex's state through the
// permutation (solver.cu kMisOMax).
__device__ __forceinline__ void mark_candidate(int32_t v, uint8_t *next, uint8_t *state,
                                               uint8_t *segflag, int T,
                                               const int32_t *perm = nullptr,
                                               uint8_t *mis_o = nullptr) {
  next[v] = 1;
  state[v] = TCMIS_IN_MIS;
  const int32_t o = orig_id(perm, v);
  if (mis_o) mis_o[o] = TCMIS_IN_MIS;
  if (segflag) segflag[seg_of(o, T)] = 1;
}

// Multi-GPU: a rank publishes its own range's decisions for the exchange
// (partitioned.cu), either as a bitmap slice (bit v - lo) or, in the late
// rounds, as an id list (list[0] = count, ids from list[1]; the host sizes
// `cap` from an all-reduced alive count that bounds the round's decisions,
// and a count beyond cap is reported as an overflow, never written past).
struct Publish {
  uint32_t *bits;  // dense slice; null on a single GPU
  int32_t lo;
  int32_t *list;   // sparse list (bits == null)
  int32_t cap;
};

__device__ __forceinline__ void publish(const Publish &p, int32_t v) {
  if (p.bits) {
    atomicOr(&p.bits[(uint32_t)(v - p.lo) >> 5], 1u << ((uint32_t)(v - p.lo) & 31u));
  } else if (p.list) {
    const int i = atomicAdd(p.list, 1);
    if (i < p.cap) p.list[1 + i] = v;
  }
}

// publish() for a whole warp (every lane calls it; `have` marks the lanes
// with a decision): bitmap slices take one atomicOr per distinct word (lanes
// grouped by __match_any_sync, their bits OR-reduced with redux.sync), id
// lists one atomicAdd per warp.  The per-decision atomics of publish()
// doubled the cost of round 1's kernels in the partitioned solve (bitmap
// words collecting up to 32 atomics each).
__device__ __forceinline__ void publish_warp(const Publish &p, int32_t v, bool have) {
  if (p.bits) {
    uint32_t w = 0xffffffffu, bit = 0;
    if (have) {
      const uint32_t off = (uint32_t)(v - p.lo);
      w = off >> 5;
      bit = 1u << (off & 31u);
    }
    if (!__any_sync(0xffffffffu, have)) return;
    const unsigned peers = __match_any_sync(0xffffffffu, w);
    if (have) {
      const uint32_t m = __reduce_or_sync(peers, bit);
      if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicOr(&p.bits[w], m);
    }
  } else if (p.list) {
    const unsigned act = __ballot_sync(0xffffffffu, have);
    if (!act) return;
    const int lane = threadIdx.x & 31, leader = __ffs(act) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(p.list, __popc(act));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (have) {
      const int i = base + __popc(act & ((1u << lane) - 1u));
      if (i < p.cap) p.list[1 + i] = v;
    }
  }
}

// The gathered summary of the key order: q[v] = clamp(p[v] >> shift, 1,
// 0xffff) is monotone in p, so q[u] != q[v] decides key(u) > key(v) with a
// 2-byte gather from a vector half the size of p (RGG 24M: 48 MB against
// 96 MB of p, against the 126 MB L2); only q[u] == q[v] needs p[u].  q = 0
// marks a vertex that left the alive set (kNoNeighborKey, priorities.hpp:57),
// so no state gather is needed either.  shift = scale_bits + 1 - 16 for the
// degree-aware priorities (p <= 2^scale_bits for every vertex with an edge,
// priorities.cpp:43-51) and 16 for hash priorities.
__host__ __device__ __forceinline__ uint16_t q_of(uint32_t p, int shift) {
  const uint32_t x = p >> shift;
  return (uint16_t)(x > 0xffffu ? 0xffffu : (x ? x : 1u));
}

// An alive non-candidate with a candidate neighbour is removed
// (engine.cpp:144-147); q = 0 makes it invisible to the alive vertices that
// still neighbour it from the next round on.
__device__ __forceinline__ void mark_removed(int32_t v, uint8_t *state, uint16_t *q) {
  state[v] = TCMIS_REMOVED;
  q[v] = 0;
}

// priority_key (priorities.hpp:61-64): strict (p, id) order, never 0
__device__ __forceinline__ uint64_t key_of(uint32_t p, int32_t v) {
  return ((uint64_t)p << 32) | (uint64_t)(uint32_t)(v + 1);
}

// A neighbour u blocks v (compute_max_np + generate_candidates,
// engine.cpp:86-119) iff u is alive at the start of the round and its key is
// above v's.  Candidates of the running round turn InMIS while the select
// kernels run but keep their q (only removals, written by the update kernels
// after the select kernels, zero it).
// The gathers of q[u] carry an L2 evict_last policy (createpolicy, folded
// into the load's memory descriptor) so the CSR streaming past them (marked
// evict-first, ld_stream) does not push the gathered vector out of L2.
#ifndef TCMIS_GATHER_HINT
#define TCMIS_GATHER_HINT 1
#endif
__device__ __forceinline__ uint32_t ld_gather_q(const uint16_t *p) {
#if TCMIS_GATHER_HINT
  uint16_t r;
  asm("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
      " ld.global.nc.L2::cache_hint.u16 %0, [%1], pol;\n}"
      : "=h"(r)
      : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}

// v's own p is needed only when q ties, so it is loaded then (saves a 4-byte
// stream of p per visited vertex)
__device__ __forceinline__ bool blocks(const uint16_t *__restrict__ q,
                                       const uint32_t *__restrict__ prio, int32_t u,
                                       uint32_t qv, int32_t v, const int32_t *perm = nullptr) {
  const uint32_t qu = ld_gather_q(&q[u]);
  if (qu != qv) return qu > qv;  // qu == 0 (removed) never blocks: qv >= 1
  const uint32_t pu = __ldg(&prio[u]), pv = __ldg(&prio[v]);
  if (pu != pv) return pu > pv;
  return orig_id(perm, u) > orig_id(perm, v);  // the key's id half (priorities.hpp:61-64)
}

// Degree-class bounds (solver.cu k_class_bounds; a degree-ordered graph under
// the H2 priorities): for a vertex of degree d, cb[d] = (lo, hi) with every
// solve id u >= hi of a certainly higher key (p(u) > p(v) whatever the hashes)
// and every u < lo of a certainly lower one.  Rows are sorted ascending, so a
// scan from a row's end that reaches an entry below lo has nothing left that
// could block v or be a candidate above it.  (0, INT_MAX) without bounds:
// every test below then reduces to the plain one.
__device__ __forceinline__ int2 class_bounds(const int2 *cb, int64_t deg) {
  return cb ? __ldg(&cb[deg]) : make_int2(0, 0x7fffffff);
}

__device__ __forceinline__ uint32_t fresh_prio(int32_t v, uint64_t fresh_m) {
  // engine.cpp:324-325: next round's redrawn h1 priority
  return (uint32_t)(vertex_hash_m((uint64_t)v, fresh_m) >> 32);
}

__device__ __forceinline__ void set_fresh(uint32_t *prio, uint16_t *q, int32_t v,
                                          uint64_t fresh_m, const int32_t *perm = nullptr) {
  const uint32_t p = fresh_prio(orig_id(perm, v), fresh_m);
  prio[v] = p;
  q[v] = q_of(p, 16);
}

// Per-warp output buffer in shared memory (64 entries), flushed 32 at a time
// with one atomic on the list tail: lanes of the state-machine kernels emit
// at different loop iterations, so a warp-aggregated atomic per emission
// would serialise on the tail.
struct WarpOut {
  int32_t *buf;
  int fill;  // warp-uniform
};

__device__ __forceinline__ void warp_emit(WarpOut &w, bool have, int32_t v, int32_t *out,
                                          int *tail) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, have);
  if (!m) return;
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

// warp-aggregated append of a rare item (one atomic per warp per call)
__device__ __forceinline__ void warp_append(bool have, int32_t v, int32_t *out, int *tail) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, have);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  int pos = 0;
  if (lane == leader) pos = atomicAdd(tail, __popc(m));
  pos = __shfl_sync(0xffffffffu, pos, leader);
  if (have) out[pos + __popc(m & ((1u << lane) - 1u))] = v;
}

// Block-aggregated list output for kernels whose every thread emits up to
// kPer entries per loop iteration: warp ballots into a shared-memory buffer,
// then ONE global atomic per block and iteration and a coalesced copy (a
// warp-level atomic per emission contends on the tail: 1.25M atomics on one
// word took R-MAT s26's round-1 settle kernel to 376 us).  Block-uniform.
template <int kBlockT, int kPer>
struct BlockOut {
  int32_t buf[kBlockT * kPer];
  int n, base;
  __device__ __forceinline__ void reset() {
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
  }
  __device__ __forceinline__ void put(bool have, int32_t v) {
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, have);
    if (!m) return;
    int pos = 0;
    if (lane == 0) pos = atomicAdd(&n, __popc(m));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (have) buf[pos + __popc(m & ((1u << lane) - 1u))] = v;
  }
  // up to kN entries per lane (have[j] -> v[j]) with ONE warp scan and one
  // shared atomic per warp; call from converged code (no per-entry ballots,
  // which the compiler must emulate when it cannot prove convergence)
  template <int kN>
  __device__ __forceinline__ void put_n(const bool (&have)[kN], const int32_t (&v)[kN]) {
    const int lane = threadIdx.x & 31;
    int c = 0;
#pragma unroll
    for (int j = 0; j < kN; ++j) c += have[j] ? 1 : 0;
    int incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    int base = 0;
    if (lane == 31) base = atomicAdd(&n, total);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - c;
#pragma unroll
    for (int j = 0; j < kN; ++j)
      if (have[j]) buf[base++] = v[j];
  }
  __device__ __forceinline__ void flush(int32_t *out, int *tail) {
    __syncthreads();
    if (threadIdx.x == 0) base = n ? atomicAdd(tail, n) : 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kBlockT) out[base + i] = buf[i];
    __syncthreads();
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
  }
};

// Per-lane reservation of `cnt` (>= 0) consecutive slots at *tail, one atomic
// per warp; returns the lane's first slot.  Warp-uniform call.
__device__ __forceinline__ int warp_reserve(int cnt, int *tail) {
  const int lane = threadIdx.x & 31;
  int x = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  const int total = __shfl_sync(0xffffffffu, x, 31);
  int base = 0;
  if (lane == 31 && total) base = atomicAdd(tail, total);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + x - cnt;
}

}  // namespace tcmis_b200
