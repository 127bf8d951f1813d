// solver.cu -- the TC-MIS round loop on sm_100a.
//
// One round of the reference (engine.cpp:247-291) is two kernels here:
//
//   k_select  Phase 1 + Phase 2 fused.  For every alive vertex v of the
//             worklist, a group of G lanes walks N(v) and asks "is any alive
//             neighbour's key above mine?" (compute_max_np + generate_candidates,
//             engine.cpp:86-119, restated as max(key[u]) < key[v] with dead
//             keys = 0).  A candidate immediately scatters "excluded" to its
//             neighbours (the push form of tiled_spmv's nc > 0, spmv.cpp:18-59):
//             the decision array `next` is never read inside the kernel, so
//             the round's snapshot semantics are preserved.
//   k_update  Phase 3 (engine.cpp:121-160) + worklist compaction + the round's
//             statistics (IterationStats, engine.hpp:24-34) and tile counters.
//
// Rounds stay bulk-synchronous, so the round count and every per-round stat
// equal the reference's (SURVEY 7 "Keep the rounds bulk-synchronous").
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"
#include "common.cuh"
#include "select.cuh"
#include "update.cuh"
#include "tail.cuh"
#include "tile_excl.cuh"
#include "tile_umma.cuh"

namespace tcmis_b200 {

// ------------------------------------------------------------- priorities

// priorities.cpp:43-51, with every IEEE operation spelled out so that no
// contraction or fast-math can change a bit.  floor + the two range checks of
// the reference are one cvt.rmi.u32.f64 (round toward -inf, saturating to
// [0, 0xffffffff]; the argument is never NaN).
__device__ __forceinline__ uint32_t h2_value(double avg, int32_t deg, double eps, double scale) {
  double d = __dadd_rn(__dadd_rn(avg, (double)deg), -eps);
  if (d < 1.0 / 1024.0) d = 1.0 / 1024.0;
  return __double2uint_rd(__dmul_rn(__ddiv_rn(avg, d), scale));
}

// Degree-class bounds of the H2 priorities on a degree-ordered graph
// (common.cuh class_bounds).  In p = h2_value(avg, deg, eps), eps in
// [0, 1 - 2^-53] (hash_to_unit), d = avg + deg - eps falls as eps grows, so p
// is non-decreasing in eps: every vertex of degree k has p in
// [h2(k, 0), h2(k, eps_max)], each IEEE step (add, subtract, clamp, divide,
// multiply, round down) being monotone.  Both ends are non-increasing in k,
// i.e. non-decreasing along the classes (descending degree).  For class c
// (degree k):
//   hi = first id of the first class c' with h2(deg c', 0) > h2(k, eps_max):
//        every u >= hi has p(u) > p(v) for every v of degree k;
//   lo = first id of the first class c'' with h2(deg c'', eps_max) >= h2(k, 0):
//        every u < lo has p(u) < p(v).
// The rest of the ids take the key comparison (ties resolved by the caller's
// ids, priorities.hpp:61-64).  One thread per class, two binary searches.
// lo relies on sorted rows (the early stop), so the unsorted hub rows get 0.
__global__ void k_class_bounds(int32_t ncls, const int32_t *__restrict__ cls,
                               const int64_t *__restrict__ off, double avg, double scale,
                               int2 *__restrict__ cb, int2 *__restrict__ cbc) {
  constexpr double kEpsMax = (double)((1ull << 53) - 1) * 0x1.0p-53;
  auto deg_of = [&](int32_t c) { return (int32_t)(off[cls[c] + 1] - off[cls[c]]); };
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < ncls; c += gridDim.x * blockDim.x) {
    const int32_t k = deg_of(c);
    const uint32_t plo = h2_value(avg, k, 0.0, scale), phi = h2_value(avg, k, kEpsMax, scale);
    int32_t a = 0, b = ncls;  // first c' with h2(deg c', 0) > phi
    while (a < b) {
      const int32_t m = (a + b) >> 1;
      if (h2_value(avg, deg_of(m), 0.0, scale) > phi) b = m; else a = m + 1;
    }
    const int32_t hi = cls[a];
    a = 0;
    b = ncls;  // first c'' with h2(deg c'', eps_max) >= plo
    while (a < b) {
      const int32_t m = (a + b) >> 1;
      if (h2_value(avg, deg_of(m), kEpsMax, scale) >= plo) b = m; else a = m + 1;
    }
    // rows past kSortedMax entries are not sorted (order.cu): no lower bound,
    // so their scans neither skip nor stop early
    cb[k] = make_int2(k > kSortedMax ? 0 : cls[a], hi);
    if (cbc) cbc[c] = cb[k];
  }
}

// K2: priorities (priorities.cpp:33-67) + state / decision initialisation.
// mode 0: h1 / luby-fresh hash priorities from `mseed` (= mix64(seed'));
// mode 1: h2 degree-aware priorities.
// Instruction-bound (ncu: 136 warp instructions per vertex, 62 % issue, 14 %
// of DRAM peak), so each thread takes 4 consecutive vertices: two 16-byte
// offset loads, the (v+1)*golden term of vertex_hash by addition, one 16-byte
// priority store and one 4-byte store each for state and next.
constexpr int kPrioV = 4;

__global__ void __launch_bounds__(256)
    k_priorities(int32_t n, const int64_t *__restrict__ off, int aligned, int mode,
                 uint64_t mseed, double avg, double scale, uint32_t *__restrict__ p_out,
                 uint16_t *__restrict__ q_out, int qshift, uint8_t *__restrict__ state,
                 uint8_t *__restrict__ next, uint8_t *__restrict__ segflag, int T, int tshift,
                 Ctrl *ctrl, Ctrl ctrl0,
                 DevRound *rounds, int32_t nrounds, const int32_t *__restrict__ perm,
                 uint8_t *__restrict__ mis_o) {
  // the solve's control block and (for k_tail, which accumulates into it)
  // the zeroed statistics ring: no separate copy / memset on the stream
  if (ctrl && blockIdx.x == 0 && threadIdx.x == 0) *ctrl = ctrl0;
  if (rounds)
    for (int32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrounds;
         r += gridDim.x * blockDim.x)
      rounds[r] = DevRound{};
  const int32_t quads = (int32_t)(((int64_t)n + kPrioV - 1) / kPrioV);
  for (int32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < quads;
       q += gridDim.x * blockDim.x) {
    const int32_t v0 = q * kPrioV;
    const bool full = v0 + kPrioV <= n;
    int64_t o[kPrioV + 1];
    if (full && aligned) {
      const longlong2 a = __ldg(reinterpret_cast<const longlong2 *>(off + v0));
      const longlong2 b = __ldg(reinterpret_cast<const longlong2 *>(off + v0 + 2));
      o[0] = a.x;
      o[1] = a.y;
      o[2] = b.x;
      o[3] = b.y;
      o[4] = __ldg(&off[v0 + 4]);
    } else {
#pragma unroll
      for (int j = 0; j <= kPrioV; ++j) o[j] = v0 + j <= n ? __ldg(&off[v0 + j]) : 0;
    }
    uint32_t pv[kPrioV];
    uint32_t st4 = 0, nx4 = 0;
    uint64_t x = mseed + (uint64_t)(v0 + 1) * kGolden;  // vertex_hash, priorities.cpp:21-23
#pragma unroll
    for (int j = 0; j < kPrioV; ++j, x += kGolden) {
      // a relabeled graph hashes the caller's id of its vertex (tcmis_graph_reorder)
      const int32_t vid = perm ? (v0 + j < n ? __ldg(&perm[v0 + j]) : 0) : v0 + j;
      if (perm) x = mseed + (uint64_t)(vid + 1) * kGolden;
      const int32_t deg = (int32_t)(o[j + 1] - o[j]);
      // an isolated vertex has no alive neighbour: it is a round-1 candidate
      // (engine.cpp:94-99 leaves max_np at kNoNeighborKey) and round 1's
      // select never has to visit it
      const bool iso = next && deg == 0 && v0 + j < n;
      if (iso) {
        // nobody's neighbour, so its key is never compared: no hash or FP64
        // work (the kernel is instruction-bound; R-MAT's isolated vertices
        // fill whole warps at the high ids).  tcmis_priorities (next == null)
        // still computes every p.
        pv[j] = 0;
      } else {
        const uint64_t h = mix64(x);
        if (mode == 0) {
          pv[j] = (uint32_t)(h >> 32);
        } else {
          const double eps = (double)(h >> 11) * 0x1.0p-53;  // hash_to_unit, priorities.cpp:25-27
          pv[j] = h2_value(avg, deg, eps, scale);
        }
      }
      st4 |= (uint32_t)(iso ? TCMIS_IN_MIS : TCMIS_ALIVE) << (8 * j);
      nx4 |= (uint32_t)(iso ? 1 : 0) << (8 * j);
      if (iso && segflag) segflag[tshift >= 0 ? vid >> tshift : vid / T] = 1;
      if (iso && mis_o) mis_o[vid] = TCMIS_IN_MIS;  // relabeled: caller-order membership
    }
    if (full) {
      if (p_out) *reinterpret_cast<uint4 *>(p_out + v0) = make_uint4(pv[0], pv[1], pv[2], pv[3]);
      if (q_out)
        *reinterpret_cast<uint2 *>(q_out + v0) =
            make_uint2((uint32_t)q_of(pv[0], qshift) | ((uint32_t)q_of(pv[1], qshift) << 16),
                       (uint32_t)q_of(pv[2], qshift) | ((uint32_t)q_of(pv[3], qshift) << 16));
      if (state) *reinterpret_cast<uint32_t *>(state + v0) = st4;
      if (next) *reinterpret_cast<uint32_t *>(next + v0) = nx4;
    } else {
      for (int j = 0; j < kPrioV && v0 + j < n; ++j) {
        if (p_out) p_out[v0 + j] = pv[j];
        if (q_out) q_out[v0 + j] = q_of(pv[j], qshift);
        if (state) state[v0 + j] = (uint8_t)(st4 >> (8 * j));
        if (next) next[v0 + j] = (uint8_t)(nx4 >> (8 * j));
      }
    }
  }
}

// K2 and round 1's Phase 1 in one pass, for a degree-ordered graph under the
// H2 priorities (the class bounds, common.cuh class_bounds): per vertex its
// degree from its class (2 bytes instead of two 8-byte offsets), p and q as
// k_priorities computes them, and -- everybody being alive in round 1 -- the
// round-1 verdict from its largest neighbour id: at or above the class's hi
// blocked (Alive; the pull finds it), below lo a candidate (InMIS, next = 1,
// the tile column and caller-order marks), else listed in wl1 for the probe.
// Isolated vertices (degree 0, the end of the order) are candidates as in
// k_priorities.  The control block and the statistics ring are set by
// k_init_ctrl before (blocks add to the control block here).
struct PrioSettleArgs {
  int32_t n;
  const int32_t *perm;
  const uint16_t *cls;
  const int32_t *cls_deg;
  const int2 *cbc;
  const int32_t *rmax;
  uint64_t mseed;
  double avg, scale;
  int qshift;
  uint32_t *p;
  uint16_t *q;
  uint8_t *state, *next, *segflag;
  int T;
  uint8_t *mis_o;
  int push;
  int32_t *left;
  Ctrl *ctrl;
  DevRound *rounds;  // the statistics ring, zeroed here (nothing stamps it in this kernel)
  int32_t nrounds;
};

__global__ void k_init_ctrl(Ctrl *ctrl, Ctrl c0) {
  if (threadIdx.x == 0) *ctrl = c0;
}

// per-thread inputs of one quad (prefetched one iteration ahead)
struct PsQuad {
  int32_t vid[4], cl[4], mx[4];
};
__device__ __forceinline__ PsQuad ps_load(const PrioSettleArgs &a, int64_t t, int64_t quads) {
  PsQuad d;
  const int64_t v0 = t * 4;
  if (v0 + 4 <= a.n) {
    const int4 p4 = __ldg(reinterpret_cast<const int4 *>(a.perm + v0));
    const uint2 c4 = __ldg(reinterpret_cast<const uint2 *>(a.cls + v0));
    const int4 m4 = __ldg(reinterpret_cast<const int4 *>(a.rmax + v0));
    d.vid[0] = p4.x; d.vid[1] = p4.y; d.vid[2] = p4.z; d.vid[3] = p4.w;
    d.cl[0] = c4.x & 0xffff; d.cl[1] = c4.x >> 16; d.cl[2] = c4.y & 0xffff; d.cl[3] = c4.y >> 16;
    d.mx[0] = m4.x; d.mx[1] = m4.y; d.mx[2] = m4.z; d.mx[3] = m4.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool ok = t < quads && v0 + j < a.n;
      d.vid[j] = ok ? __ldg(&a.perm[v0 + j]) : 0;
      d.cl[j] = ok ? __ldg(&a.cls[v0 + j]) : -1;
      d.mx[j] = ok ? __ldg(&a.rmax[v0 + j]) : -1;
    }
  }
  return d;
}

constexpr int kPsFlush = 4;  // iterations between the residual list's flushes

// The per-vertex inputs (perm, r1_max, class) of a chunk of 1024 vertices
// reach shared memory by TMA bulk copies (cp.async.bulk, completion on an
// mbarrier), kPsStages chunks ahead of the chunk being processed: the loads
// need no registers, so the kernel keeps DRAM busy at its register-limited
// occupancy (ncu, the register-prefetch version: 19 % of the warps' stalls
// sat on the first use of a just-loaded class index).
#ifndef TCMIS_PS_STAGES
#define TCMIS_PS_STAGES 3
#endif
constexpr int kPsChunk = 1024, kPsStages = TCMIS_PS_STAGES;
struct __align__(16) PsStage {
  int32_t perm[kPsChunk];
  int32_t rmax[kPsChunk];
  uint16_t cls[kPsChunk];
};

__device__ __forceinline__ void ps_issue(const PrioSettleArgs &a, PsStage &st, uint64_t &bar,
                                         int64_t c) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  constexpr uint32_t kBytes = sizeof(PsStage);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(kBytes)
               : "memory");
  const int64_t v0 = c * kPsChunk;
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(st.perm)),
      "l"(a.perm + v0), "r"(4u * kPsChunk), "r"(b)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(st.rmax)),
      "l"(a.rmax + v0), "r"(4u * kPsChunk), "r"(b)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(st.cls)),
      "l"(a.cls + v0), "r"(2u * kPsChunk), "r"(b)
      : "memory");
}

__device__ __forceinline__ void ps_wait(uint64_t &bar, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  }
}

__global__ void __launch_bounds__(256) k_prio_settle(PrioSettleArgs a) {
  constexpr int kV = 4;
  static_assert(256 * kV == kPsChunk, "a thread per quad of the chunk");
  __shared__ PsStage stg[kPsStages];
  __shared__ __align__(8) uint64_t bar[kPsStages];
  // the residual list leaves the block every kPsFlush chunks (its barriers
  // stall every warp of the block)
  __shared__ BlockOut<256, kV * kPsFlush> left;
  if (threadIdx.x == 0) {
    for (int st = 0; st < kPsStages; ++st)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(&bar[st])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  left.reset();  // (a block barrier: the barriers are initialised)
  for (int32_t r = blockIdx.x * 256 + threadIdx.x; r < a.nrounds; r += gridDim.x * 256)
    a.rounds[r] = DevRound{};
  unsigned long long sel = 0;
  const int64_t quads = ((int64_t)a.n + kV - 1) / kV;
  const int64_t nchunks = ((int64_t)a.n + kPsChunk - 1) / kPsChunk;
  const int64_t full = (int64_t)a.n / kPsChunk;  // chunks wholly inside [0, n)
  const int64_t G = gridDim.x;
  if (threadIdx.x == 0)
    for (int st = 0; st < kPsStages; ++st) {
      const int64_t c = blockIdx.x + st * G;
      if (c < full) ps_issue(a, stg[st], bar[st], c);
    }
  uint32_t parity = 0;  // bit st: the parity stage st waits for next
  int it = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += G, ++it) {
    const int st = it % kPsStages;
    PsQuad cur;
    if (c < full) {
      ps_wait(bar[st], (parity >> st) & 1u);
      parity ^= 1u << st;
      const int4 p4 = *reinterpret_cast<const int4 *>(stg[st].perm + kV * threadIdx.x);
      const int4 m4 = *reinterpret_cast<const int4 *>(stg[st].rmax + kV * threadIdx.x);
      const uint2 c4 = *reinterpret_cast<const uint2 *>(stg[st].cls + kV * threadIdx.x);
      cur.vid[0] = p4.x; cur.vid[1] = p4.y; cur.vid[2] = p4.z; cur.vid[3] = p4.w;
      cur.mx[0] = m4.x; cur.mx[1] = m4.y; cur.mx[2] = m4.z; cur.mx[3] = m4.w;
      cur.cl[0] = c4.x & 0xffff; cur.cl[1] = c4.x >> 16; cur.cl[2] = c4.y & 0xffff; cur.cl[3] = c4.y >> 16;
      __syncthreads();  // stage st is read: refill it kPsStages chunks ahead
      if (threadIdx.x == 0 && c + kPsStages * G < full) {
        // the block's generic-proxy reads of the stage before the bulk copy's
        // async-proxy writes into it (cross-proxy WAR)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        ps_issue(a, stg[st], bar[st], c + kPsStages * G);
      }
    } else {
      cur = ps_load(a, c * 256 + threadIdx.x, quads);  // the partial last chunk
    }
    const int64_t v0 = c * kPsChunk + kV * threadIdx.x;
    uint32_t pv[kV], st4 = 0, nx4 = 0;
    bool lft[kV];
    int32_t lid[kV];
#pragma unroll
    for (int j = 0; j < kV; ++j) {
      const int32_t deg = cur.cl[j] >= 0 ? __ldg(&a.cls_deg[cur.cl[j]]) : 0;
      const bool iso = deg == 0;
      int r = -1;  // -1 none, 0 left to the probe, 1 blocked, 2 candidate
      if (iso) {
        pv[j] = 0;  // as k_priorities: never compared
      } else {
        const uint64_t h = mix64(a.mseed + (uint64_t)(cur.vid[j] + 1) * kGolden);
        const double eps = (double)(h >> 11) * 0x1.0p-53;  // hash_to_unit, priorities.cpp:25-27
        pv[j] = h2_value(a.avg, deg, eps, a.scale);
        const int2 cb = __ldg(&a.cbc[cur.cl[j]]);
        r = cur.mx[j] >= cb.y ? 1 : (cur.mx[j] < cb.x && !a.push ? 2 : 0);
      }
      const bool in = cur.cl[j] >= 0 && (iso || r == 2);
      st4 |= (uint32_t)(in ? TCMIS_IN_MIS : TCMIS_ALIVE) << (8 * j);
      nx4 |= (uint32_t)(in ? 1 : 0) << (8 * j);
      if (in) {
        if (a.segflag) a.segflag[seg_of(cur.vid[j], a.T)] = 1;
        if (a.mis_o) a.mis_o[cur.vid[j]] = TCMIS_IN_MIS;
      }
      if (r == 2) ++sel;
      lft[j] = r == 0;
      lid[j] = (int32_t)(v0 + j);
    }
    left.put_n<kV>(lft, lid);
    if (v0 + kV <= a.n) {
      *reinterpret_cast<uint4 *>(a.p + v0) = make_uint4(pv[0], pv[1], pv[2], pv[3]);
      *reinterpret_cast<uint2 *>(a.q + v0) =
          make_uint2((uint32_t)q_of(pv[0], a.qshift) | ((uint32_t)q_of(pv[1], a.qshift) << 16),
                     (uint32_t)q_of(pv[2], a.qshift) | ((uint32_t)q_of(pv[3], a.qshift) << 16));
      *reinterpret_cast<uint32_t *>(a.state + v0) = st4;
      *reinterpret_cast<uint32_t *>(a.next + v0) = nx4;
    } else {
      for (int j = 0; j < kV && v0 + j < a.n; ++j) {
        a.p[v0 + j] = pv[j];
        a.q[v0 + j] = q_of(pv[j], a.qshift);
        a.state[v0 + j] = (uint8_t)(st4 >> (8 * j));
        a.next[v0 + j] = (uint8_t)(nx4 >> (8 * j));
      }
    }
    // block-uniform: the block's last chunk, or every kPsFlush
    if ((it + 1) % kPsFlush == 0 || c + G >= nchunks) left.flush(a.left, &a.ctrl->r1_sel_left);
  }
  block_add3(sel, 0, 0, a.ctrl);
}

__global__ void k_max_degree(int32_t n, const int64_t *__restrict__ off,
                             unsigned long long *__restrict__ out) {
  unsigned long long mx = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long d = (unsigned long long)(off[v + 1] - off[v]);
    mx = d > mx ? d : mx;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_down_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

__global__ void k_h1(int32_t n, uint64_t mseed, uint32_t *__restrict__ p) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    p[v] = (uint32_t)(vertex_hash_m((uint64_t)v, mseed) >> 32);  // priorities.cpp:33-41
}

// run_h3_resolution start state: only the alive vertices of `states` take
// part (everyone else is Removed, key 0 = invisible)
__global__ void k_resolve_init(int32_t n, const uint32_t *__restrict__ p,
                               const uint8_t *__restrict__ states, uint32_t *__restrict__ prio,
                               uint16_t *__restrict__ q,
                               uint8_t *__restrict__ state, uint8_t *__restrict__ next) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool alive = states[v] == TCMIS_ALIVE;
    prio[v] = p[v];
    q[v] = alive ? q_of(p[v], 16) : 0;  // any monotone summary works
    state[v] = alive ? TCMIS_ALIVE : TCMIS_REMOVED;
    next[v] = 0;
  }
}

struct IsAliveIn {
  const uint8_t *states;
  __device__ __forceinline__ bool operator()(int32_t v) const { return states[v] == TCMIS_ALIVE; }
};

struct HasEdges {
  const int64_t *off;
  __device__ __forceinline__ bool operator()(int32_t v) const { return off[v + 1] > off[v]; }
};

// ----------------------------------------------------------------- rounds

// The whole-solve graph's last node: control block, MIS count and the first
// 64 rounds' statistics into mapped host memory (HostRes).
__global__ void k_pack(const Ctrl *__restrict__ ctrl, const int64_t *__restrict__ mis_count,
                       const DevRound *__restrict__ rounds, int32_t cap, HostRes *out) {
  if (threadIdx.x == 0) {
    out->ctrl = *ctrl;
    out->mis_count = (long long)*mis_count;
  }
  for (int r = threadIdx.x; r < 64 && r < cap; r += blockDim.x) out->rounds[r] = rounds[r];
  __threadfence_system();
}

// h3: tile counters of the single collapsed iteration (segments that hold
// any MIS vertex).
__global__ void k_seg_total(const uint8_t *__restrict__ segflag,
                            const int32_t *__restrict__ rowtiles, int32_t nseg, Ctrl *ctrl) {
  unsigned long long ev = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nseg;
       b += (int64_t)gridDim.x * blockDim.x)
    if (segflag[b]) ev += (unsigned long long)rowtiles[b];
  block_add3(0, 0, ev, ctrl);
}

// Relabeled solves without the caller-order membership plane (R-MAT s26):
// ascending MIS ids of the caller's order in two passes instead of one cub
// select gathering through inv per id (262 us at s26):
//   1. k_gc_bits: warp per 1024 caller ids, 32 coalesced steps of inv + a
//      gather of the solve-order state (L2-resident), one ballot word each;
//      per-block counts;
//   2. an exclusive sum of the block counts (cub, 8k blocks at s26);
//   3. k_gc_ids: words -> ids, block scan of the words' popcounts.
// DRAM: inv once (4 B/id), 1 bit/id twice, the ids once.
constexpr int kGcBlock = 256;                       // words per block
constexpr int64_t kGcIdsPerBlock = 32ll * kGcBlock;  // caller ids per block

__global__ void __launch_bounds__(kGcBlock) k_gc_bits(int32_t n, const int32_t *__restrict__ inv,
                                                      const uint8_t *__restrict__ state,
                                                      uint32_t *__restrict__ bits,
                                                      int64_t *__restrict__ blk) {
  __shared__ int s_cnt;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // the warp's 32 words: caller ids [base, base + 1024)
  const int64_t base = blockIdx.x * kGcIdsPerBlock + (int64_t)w * 1024;
  uint32_t mine = 0;
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    const int64_t o = base + 32 * k + lane;
    const bool in = o < n && state[__ldg(&inv[o])] == TCMIS_IN_MIS;
    const uint32_t m = __ballot_sync(0xffffffffu, in);
    if (lane == k) mine = m;
  }
  const int64_t word = blockIdx.x * (int64_t)kGcBlock + threadIdx.x;
  if (word * 32 < n) bits[word] = mine;
  const int c = __reduce_add_sync(0xffffffffu, __popc(mine));
  if (lane == 0 && c) atomicAdd(&s_cnt, c);
  __syncthreads();
  if (threadIdx.x == 0) blk[blockIdx.x] = s_cnt;
}

__global__ void __launch_bounds__(kGcBlock) k_gc_ids(int32_t n, const uint32_t *__restrict__ bits,
                                                     const int64_t *__restrict__ blk_off,
                                                     int32_t nblk, int32_t *__restrict__ mis,
                                                     int64_t *__restrict__ mis_count) {
  // each warp expands its 32 words one at a time: lane j writes bit j's id
  // at the word's position + the set bits below j -- every store of a step
  // lands in one contiguous run (no per-thread bit loop, no staging)
  using Scan = cub::BlockScan<int, kGcBlock>;
  __shared__ typename Scan::TempStorage tmp;
  const int lane = threadIdx.x & 31;
  const int64_t word = blockIdx.x * (int64_t)kGcBlock + threadIdx.x;
  const uint32_t m = word * 32 < n ? bits[word] : 0u;
  int pos = 0;
  Scan(tmp).ExclusiveSum(__popc(m), pos);
  const int64_t gpos = blk_off[blockIdx.x] + pos;
  const int64_t w0 = word - lane;
  const uint32_t below = (1u << lane) - 1u;
#pragma unroll 4
  for (int k = 0; k < 32; ++k) {
    const uint32_t wk = __shfl_sync(0xffffffffu, m, k);
    const int64_t pk = __shfl_sync(0xffffffffu, gpos, k);
    if ((wk >> lane) & 1u) mis[pk + __popc(wk & below)] = (int32_t)((w0 + k) * 32 + lane);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *mis_count = blk_off[nblk];
}

int gc_blocks(int32_t n) { return (int)((n + kGcIdsPerBlock - 1) / kGcIdsPerBlock); }

// the buffers (outside any capture)
int gc_prepare(tcmis_graph *g) {
  Workspace &ws = g->ws;
  if (ws.gc_bits) return 0;
  const int nb = gc_blocks((int32_t)ws.n_cap);
  if (int rc = dev_alloc(&ws.gc_bits, (size_t)nb * kGcBlock)) return rc;
  if (int rc = dev_alloc(&ws.gc_blk, 2 * ((size_t)nb + 1))) return rc;
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, ws.gc_blk, ws.gc_blk + nb + 1, nb + 1, g->ctx->stream);
  if (int rc = dev_alloc((char **)&ws.gc_tmp, bytes)) return rc;
  ws.gc_tmp_bytes = bytes;
  return 0;
}

// enqueue the three steps (capturable)
int gc_compact(tcmis_graph *g) {
  Workspace &ws = g->ws;
  cudaStream_t st = g->ctx->stream;
  const int32_t n = g->n;
  const int nb = gc_blocks(n);
  int64_t *cnt = ws.gc_blk, *offs = ws.gc_blk + nb + 1;
  k_gc_bits<<<nb, kGcBlock, 0, st>>>(n, g->d_inv, ws.state, ws.gc_bits, cnt);
  TCMIS_CUDA(cudaMemsetAsync(cnt + nb, 0, 8, st));
  size_t bytes = ws.gc_tmp_bytes;
  TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(ws.gc_tmp, bytes, cnt, offs, nb + 1, st));
  k_gc_ids<<<nb, kGcBlock, 0, st>>>(n, ws.gc_bits, offs, nb, ws.mis, ws.mis_count);
  g->ctx->launches += 4;
  return 0;
}

// relabeled solves: the final states in the caller's order (coalesced
// writes, a gather of the solve-order states)
__global__ void k_unpermute(int32_t n, const int32_t *__restrict__ inv,
                            const uint8_t *__restrict__ state, uint8_t *__restrict__ state_o) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    state_o[v] = state[__ldg(&inv[v])];
}

// a relabeled solve's caller-order membership plane: 1 / 2 = InMIS (tail.cuh)
struct IsMember {
  const uint8_t *plane;
  __device__ __forceinline__ bool operator()(int32_t v) const { return plane[v] != 0; }
};

struct IsInMIS {
  const uint8_t *state;
  __device__ __forceinline__ bool operator()(int32_t v) const { return state[v] == TCMIS_IN_MIS; }
};

// ------------------------------------------------- phase helpers (parity)

__global__ void k_max_np(int32_t n, const int64_t *__restrict__ off,
                         const int32_t *__restrict__ nbr, const uint32_t *__restrict__ p,
                         const uint8_t *__restrict__ st, uint64_t *__restrict__ out) {
  // engine.cpp:86-103, warp per vertex
  const int lane = threadIdx.x & 31;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    unsigned long long best = 0;
    if (st[v] == TCMIS_ALIVE)
      for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) {
        const int32_t u = nbr[e];
        if (st[u] == TCMIS_ALIVE) {
          unsigned long long k = ((unsigned long long)p[u] << 32) | (unsigned long long)(u + 1);
          best = k > best ? k : best;
        }
      }
    for (int o = 16; o; o >>= 1) {
      unsigned long long t = __shfl_down_sync(0xffffffffu, best, o);
      best = t > best ? t : best;
    }
    if (lane == 0) out[v] = best;
  }
}

__global__ void k_neighbor_count(int32_t n, const int64_t *__restrict__ off,
                                 const int32_t *__restrict__ nbr, const uint8_t *__restrict__ c,
                                 int32_t *__restrict__ nc) {
  // spmv.cpp:61-73, warp per vertex
  const int lane = threadIdx.x & 31;
  for (int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int cnt = 0;
    for (int64_t e = off[v] + lane; e < off[v + 1]; e += 32) cnt += c[nbr[e]] != 0;
    for (int o = 16; o; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
    if (lane == 0) nc[v] = cnt;
  }
}

__global__ void k_segflags_from(int32_t n, const uint8_t *__restrict__ c, int T,
                                uint8_t *__restrict__ segflag) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    if (c[v]) segflag[v / T] = 1;
}

// --------------------------------------------------------------- timeline

cudaEvent_t pool_event(tcmis_ctx *ctx) {
  if (ctx->pool_next >= ctx->event_pool.size()) {
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    ctx->event_pool.push_back(ev);
  }
  return ctx->event_pool[ctx->pool_next++];
}

void timeline_begin(tcmis_ctx *ctx) {
  ctx->marks.clear();
  ctx->timeline.clear();
  ctx->recording = true;
  ctx->rec_round = 0;
  ctx->pool_next = 0;
}

void timeline_end(tcmis_ctx *ctx) {
  ctx->recording = false;
  cudaStreamSynchronize(ctx->stream);
  for (const auto &m : ctx->marks) {
    tcmis_kernel_time t{};
    std::snprintf(t.name, sizeof(t.name), "%s", m.name);
    t.round = m.round;
    cudaEventElapsedTime(&t.ms, m.a, m.b);
    ctx->timeline.push_back(t);
  }
  ctx->marks.clear();
}

// -------------------------------------------------------------- workspace

void free_workspace(Workspace &ws) {
  dev_free(ws.prio);
  dev_free(ws.q);
  dev_free(ws.state);
  dev_free(ws.state_o);
  dev_free(ws.mis_o);
  dev_free(ws.next);
  dev_free(ws.xt);
  dev_free(ws.wl[0]);
  dev_free(ws.wl[1]);
  dev_free(ws.segflag);
  dev_free(ws.mis);
  dev_free(ws.gc_bits);
  dev_free(ws.gc_blk);
  dev_free(ws.gc_tmp);
  dev_free(ws.long_list);
  dev_free(ws.prow);
  dev_free(ws.pitems);
  dev_free(ws.vlong);
  dev_free(ws.undec_sel);
  dev_free(ws.undec_pull);
  dev_free(ws.segmark);
  dev_free(ws.bar);
  dev_free(ws.warpcnt);
  dev_free(ws.mis_count);
  dev_free(ws.ctrl);
  cudaFreeHost(ws.h_ctrl);
  cudaFreeHost(ws.h_misc);
  cudaFreeHost(ws.h_res);
  dev_free(ws.rounds);
  cudaFreeHost(ws.h_rounds);
  dev_free(ws.cub_tmp);
  dev_free(ws.cbits);
  dev_free(ws.tile_hit);
  dev_free(ws.alive_bits);
  dev_free(ws.blocked);
  if (ws.exec) cudaGraphExecDestroy(ws.exec);
  ws = Workspace{};
}

int ensure_cub(tcmis_graph *g, size_t bytes) {
  Workspace &ws = g->ws;
  if (bytes <= ws.cub_bytes) return 0;
  dev_free(ws.cub_tmp);
  ws.cub_tmp = nullptr;
  ws.cub_bytes = 0;
  if (int rc = dev_alloc((char **)&ws.cub_tmp, bytes)) return rc;
  ws.cub_bytes = bytes;
  return 0;
}

int ensure_workspace(tcmis_graph *g) {
  Workspace &ws = g->ws;
  const size_t n = (size_t)std::max<int32_t>(g->n, 1);
  Workspace &spare = g->ctx->spare;
  if (!ws.ctrl && spare.ctrl && spare.n_cap >= n && spare.seg_cap >= n) {
    ws = spare;  // adopt a destroyed graph's buffers (tcmis_graph_destroy)
    spare = Workspace{};
  }
  if (ws.n_cap < n) {
    if (ws.exec) {  // the cached round graph points at the old buffers
      cudaGraphExecDestroy(ws.exec);
      ws.exec = nullptr;
    }
    dev_free(ws.prio);
  dev_free(ws.q);
    dev_free(ws.state);
    dev_free(ws.state_o);
    ws.state_o = nullptr;
    dev_free(ws.mis_o);
    ws.mis_o = nullptr;
    dev_free(ws.next);
    dev_free(ws.xt);
    dev_free(ws.wl[0]);
    dev_free(ws.wl[1]);
    dev_free(ws.mis);
    dev_free(ws.gc_bits);
    dev_free(ws.gc_blk);
    dev_free(ws.gc_tmp);
    ws.gc_bits = nullptr;
    ws.gc_blk = nullptr;
    ws.gc_tmp = nullptr;
    dev_free(ws.long_list);
    dev_free(ws.undec_sel);
    dev_free(ws.undec_pull);
    dev_free(ws.segmark);
    dev_free(ws.cbits);
    dev_free(ws.tile_hit);
    dev_free(ws.alive_bits);
    dev_free(ws.blocked);
    ws.n_cap = 0;
    if (int rc = dev_alloc(&ws.prio, n)) return rc;
    if (int rc = dev_alloc(&ws.q, n + 8)) return rc;
    if (int rc = dev_alloc(&ws.state, n + 16)) return rc;  // uint4 reads past n (k_tail)
    if (int rc = dev_alloc(&ws.next, n + 16)) return rc;  // uint4 reads past n (k_tail)
    if (int rc = dev_alloc(&ws.xt, n)) return rc;
    TCMIS_CUDA(cudaMemsetAsync(ws.xt, 0, sizeof(uint16_t) * n, g->ctx->stream));
    if (int rc = dev_alloc(&ws.wl[0], n)) return rc;
    if (int rc = dev_alloc(&ws.wl[1], n)) return rc;
    if (int rc = dev_alloc(&ws.mis, n)) return rc;
    if (int rc = dev_alloc(&ws.long_list, n)) return rc;
    if (int rc = dev_alloc(&ws.undec_sel, n)) return rc;
    if (int rc = dev_alloc(&ws.undec_pull, n)) return rc;
    if (int rc = dev_alloc(&ws.segmark, n)) return rc;
    if (int rc = dev_alloc(&ws.cbits, n / 32 + 2)) return rc;
    if (int rc = dev_alloc(&ws.tile_hit, n / 16 + 2)) return rc;
    if (int rc = dev_alloc(&ws.alive_bits, n / 32 + 2)) return rc;
    if (int rc = dev_alloc(&ws.blocked, n / 16 + 2)) return rc;
    // tile Phase 1 rows blocked: zero between tile rounds (k_tile_mark clears
    // what it reads)
    TCMIS_CUDA(cudaMemsetAsync(ws.blocked, 0, 4 * (n / 16 + 2), g->ctx->stream));
    TCMIS_CUDA(cudaMemsetAsync(ws.next, 0, n + 16, g->ctx->stream));
    ws.n_cap = n;
  }
  {  // at most nnz / kBlockRow rows are longer than kBlockRow (per graph)
    const int64_t need = std::min<int64_t>((int64_t)n, g->nnz / kBlockRow + 1);
    if (ws.vlong_cap < need) {
      if (ws.exec) {  // the cached round graph points at the old lists
        cudaGraphExecDestroy(ws.exec);
        ws.exec = nullptr;
      }
      dev_free(ws.vlong);
      ws.vlong = nullptr;
      ws.vlong_cap = 0;
      if (int rc = dev_alloc(&ws.vlong, (size_t)need)) return rc;
      ws.vlong_cap = need;
    }
  }
  {  // pull rows that outlive the engine are longer than kThreadMax; their
     // chunks number at most rows + nnz / kPullChunk (per graph)
    const int64_t rows = std::min<int64_t>((int64_t)n, g->nnz / kThreadMax + 1);
    if (ws.prow_cap < rows) {
      if (ws.exec) {
        cudaGraphExecDestroy(ws.exec);
        ws.exec = nullptr;
      }
      dev_free(ws.prow);
      dev_free(ws.pitems);
      ws.prow = nullptr;
      ws.pitems = nullptr;
      ws.prow_cap = 0;
      if (int rc = dev_alloc(&ws.prow, (size_t)rows)) return rc;
      if (int rc = dev_alloc(&ws.pitems, (size_t)(rows + g->nnz / kPullChunk + 1))) return rc;
      ws.prow_cap = rows;
    }
  }
  // segment flags for any tile_dim >= 1
  if (ws.seg_cap < n) {
    dev_free(ws.segflag);
    if (int rc = dev_alloc(&ws.segflag, n)) return rc;
    TCMIS_CUDA(cudaMemsetAsync(ws.segflag, 0, n, g->ctx->stream));
    ws.seg_cap = n;
  }
  if (!ws.ctrl) {
    if (int rc = dev_alloc(&ws.ctrl, 1)) return rc;
    if (int rc = dev_alloc(&ws.mis_count, 1)) return rc;
    if (int rc = dev_alloc(&ws.bar, 4)) return rc;
    if (int rc = dev_alloc(&ws.warpcnt, 2 * (size_t)kTailMaxWarps + 2)) return rc;
    TCMIS_CUDA(cudaMemsetAsync(ws.warpcnt, 0, sizeof(unsigned) * (2 * (size_t)kTailMaxWarps + 2),
                               g->ctx->stream));
    TCMIS_CUDA(cudaMemsetAsync(ws.bar, 0, 4 * sizeof(unsigned), g->ctx->stream));
    TCMIS_CUDA(cudaMallocHost((void **)&ws.h_ctrl, sizeof(Ctrl)));
    TCMIS_CUDA(cudaMallocHost((void **)&ws.h_misc, 2 * sizeof(int64_t)));
    TCMIS_CUDA(cudaHostAlloc((void **)&ws.h_res, sizeof(HostRes), cudaHostAllocMapped));
    TCMIS_CUDA(cudaHostGetDevicePointer((void **)&ws.d_res, ws.h_res, 0));
    ws.round_cap = 4096;
    if (int rc = dev_alloc(&ws.rounds, (size_t)ws.round_cap)) return rc;
    TCMIS_CUDA(cudaMallocHost((void **)&ws.h_rounds, sizeof(DevRound) * ws.round_cap));
  }
  size_t need = 0, t = 0;
  thrust::counting_iterator<int32_t> ids(0);
  TCMIS_CUDA(cub::DeviceSelect::If(nullptr, t, ids, ws.mis, ws.mis_count, (int)n,
                                   IsInMIS{ws.state}, g->ctx->stream));
  need = std::max(need, t);
  TCMIS_CUDA(cub::DeviceSelect::If(nullptr, t, ids, ws.mis, ws.mis_count, (int)n,
                                   HasEdges{g->d_off}, g->ctx->stream));
  need = std::max(need, t);
  if (int rc = ensure_cub(g, need)) return rc;
  if (!g->prepared) {
    // once per graph: the round-1 select list (non-isolated ids, ascending)
    // and the degree skew that picks the exclusion form
    cudaStream_t st = g->ctx->stream;
    if (int rc = dev_alloc(&g->d_nz, n)) return rc;
    size_t bytes = ws.cub_bytes;
    TCMIS_CUDA(cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, g->d_nz, ws.mis_count,
                                     (int)g->n, HasEdges{g->d_off}, st));
    unsigned long long *d_mx = nullptr;
    if (int rc = dev_alloc(&d_mx, 1)) return rc;
    cudaMemsetAsync(d_mx, 0, 8, st);
    k_max_degree<<<grid_for(g->ctx, g->n, 256, 8), 256, 0, st>>>(g->n, g->d_off, d_mx);
    g->ctx->launches += 2;
    int64_t nz = 0;
    unsigned long long mx = 0;
    cudaMemcpyAsync(&nz, ws.mis_count, 8, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&mx, d_mx, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    dev_free(d_mx);
    if (e != cudaSuccess) return cuda_error(e, "graph preparation");
    g->nz_count = (int32_t)nz;
    g->max_degree = (int64_t)mx;
    g->prepared = true;
  }
  return 0;
}

// ------------------------------------------------------------------ solve

double avg_degree(const tcmis_graph *g) {
  // priorities.cpp:60 avg = 2.0 * num_edges / n, num_edges = nnz / 2 (of the
  // whole graph, also on a rank that holds only a row partition)
  const int64_t nnz = g->nnz_global >= 0 ? g->nnz_global : g->nnz;
  return 2.0 * (double)(nnz / 2) / (double)g->n;
}

namespace {

}  // namespace

constexpr int64_t kMisOMax = 48ll << 20;  // vertices: caller-order membership plane up to here

// common.cuh q_of: the degree-aware priorities of vertices with an edge are
// <= 2^scale_bits (avg / (avg + deg - eps) <= 1), hash priorities span u32
int q_shift(int heuristic, int scale_bits) {
  if (heuristic == TCMIS_H1 || heuristic == TCMIS_LUBY_FRESH) return 16;
  return scale_bits + 1 > 16 ? scale_bits + 1 - 16 : 0;
}

int launch_priorities(tcmis_graph *g, int heuristic, uint64_t seed, int scale_bits,
                      uint32_t *p_out, uint16_t *q_out, uint8_t *state, uint8_t *next,
                      uint8_t *segflag, int T, Ctrl *ctrl, const Ctrl *ctrl0, DevRound *rounds,
                      int32_t nrounds, const int64_t *solve_off, const int32_t *perm,
                      uint8_t *mis_o) {
  tcmis_ctx *ctx = g->ctx;
  int mode = 1;
  uint64_t mseed = mix64(seed);
  if (heuristic == TCMIS_H1) {
    mode = 0;
  } else if (heuristic == TCMIS_LUBY_FRESH) {
    mode = 0;
    mseed = mix64(combine_seed(seed, 1));  // engine.cpp:324-325, iteration 1
  }
  const double scale = mode ? (double)(1u << scale_bits) : 0.0;
  const int64_t *off = solve_off ? solve_off : (g->d_off_full ? g->d_off_full : g->d_off);
  const int aligned = ((uintptr_t)off & 15) == 0 ? 1 : 0;
  const int tshift = (T & (T - 1)) == 0 ? __builtin_ctz((unsigned)T) : -1;
  const int grid = grid_for(ctx, ((int64_t)g->n + kPrioV - 1) / kPrioV, 256, 8);
  TCMIS_TIMED(ctx, "k_priorities",
              (k_priorities<<<grid, 256, 0, ctx->stream>>>(g->n, off, aligned, mode, mseed,
                                                          mode ? avg_degree(g) : 0.0, scale,
                                                          p_out, q_out, q_shift(heuristic, scale_bits),
                                                          state, next, segflag, T, tshift, ctrl,
                                                          ctrl0 ? *ctrl0 : Ctrl{},
                                                          rounds, nrounds, perm, mis_o)));
  TCMIS_LAUNCHED(ctx);
  return 0;
}

// the fused init + round-1 settle (k_prio_settle) of a degree-ordered H2 solve
int launch_prio_settle(tcmis_graph *g, const RoundArgs &a, uint64_t seed, int scale_bits,
                       int heuristic, uint8_t *segflag, const Ctrl &c0) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  Workspace &ws = g->ws;
  k_init_ctrl<<<1, 32, 0, st>>>(ws.ctrl, c0);
  TCMIS_LAUNCHED(ctx);
  PrioSettleArgs p;
  p.n = g->n;
  p.perm = a.perm;
  p.cls = a.r1_cls;
  p.cls_deg = g->d_cls_deg;
  p.cbc = a.cbc;
  p.rmax = a.r1_max;
  p.mseed = mix64(seed);
  p.avg = avg_degree(g);
  p.scale = (double)(1u << scale_bits);
  p.qshift = q_shift(heuristic, scale_bits);
  p.p = ws.prio;
  p.q = ws.q;
  p.state = ws.state;
  p.next = ws.next;
  p.segflag = segflag;
  p.T = a.T;
  p.mis_o = a.mis_o;
  p.push = a.pull ? 0 : 1;
  p.left = ws.wl[1];
  p.ctrl = ws.ctrl;
  p.rounds = ws.rounds;
  p.nrounds = ws.round_cap;
  const int grid = grid_for(ctx, ((int64_t)g->n + 3) / 4, 256, 4);
  TCMIS_TIMED(ctx, "k_prio_settle", (k_prio_settle<<<grid, 256, 0, st>>>(p)));
  TCMIS_LAUNCHED(ctx);
  return 0;
}

namespace {

int validate(const tcmis_graph *g, const tcmis_config *c) {
  if (c->heuristic < TCMIS_H1 || c->heuristic > TCMIS_LUBY_PERM)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "unknown heuristic id");
  const bool tiled = c->heuristic <= TCMIS_H3;
  // run_tc_mis(g, cfg) tiles first: tile_dim is checked even for n == 0
  // (engine.cpp:297-299 -> tiling.cpp:17-21).
  if (tiled && (c->tile_dim < 1 || c->tile_dim > 64))
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tile_dim must be in [1, 64], got " + std::to_string(c->tile_dim));
  if (g->n == 0) return 0;
  if ((c->heuristic == TCMIS_H2 || c->heuristic == TCMIS_H3 ||
       c->heuristic == TCMIS_LUBY_PERM) &&
      (c->scale_bits < 8 || c->scale_bits > 30))
    return set_error(TCMIS_E_INVALID_ARGUMENT, "scale_bits must be in [8, 30]");
  return 0;
}

}  // namespace


SelectArgs select_args(tcmis_graph *g, const RoundArgs &a) {
  Workspace &ws = g->ws;
  SelectArgs s;
  s.n1 = a.nz_count;
  s.nz = a.nz;
  s.nz_identity = a.nz_count == a.n || a.nz_prefix ? 1 : 0;
  s.off = a.off;
  s.nbr = a.nbr;
  s.vnnz = a.vnnz;
  s.prio = ws.prio;
  s.q = ws.q;
  s.next = ws.next;
  s.state = ws.state;
  s.segflag = a.seg_mode ? ws.segflag : nullptr;
  s.T = a.T;
  s.push = (a.pull || a.tile) ? 0 : 1;
  s.ctrl = ws.ctrl;
  s.wl0 = ws.wl[0];
  s.wl1 = ws.wl[1];
  s.long_list = ws.long_list;
  s.vlong = ws.vlong;
  s.undecided = ws.undec_sel;
  s.pub = Publish{a.pub_cand, a.pub_lo, a.pub_lcand, a.pub_cap};
  if (a.tile) s.pub = Publish{ws.cbits, 0, nullptr, 0};  // the candidate segments of the tile kernels
  s.rounds = ws.rounds;
  s.perm = a.perm;
  s.mis_o = a.mis_o;
  s.cb = a.cb;
  s.r1_max = a.r1_max;
  s.r1_cls = a.r1_cls;
  s.cbc = a.cbc;
  s.tile_gate = a.tile_cand ? a.tile_gate : 0;
  return s;
}

UpdateArgs update_args(tcmis_graph *g, const RoundArgs &a) {
  Workspace &ws = g->ws;
  UpdateArgs u;
  u.n = a.n;
  u.off = a.off;
  u.nbr = a.nbr;
  u.vnnz = a.vnnz;
  u.prio = ws.prio;
  u.q = ws.q;
  u.state = ws.state;
  u.next = ws.next;
  u.ctrl = ws.ctrl;
  u.wl0 = ws.wl[0];
  u.wl1 = ws.wl[1];
  u.fresh = a.fresh;
  u.seed = a.seed;
  u.n1 = a.nz_count;
  u.nz = a.nz;
  u.nz_identity = a.nz_count == a.n || a.nz_prefix ? 1 : 0;
  u.prow = ws.prow;
  u.pitems = ws.pitems;
  u.undecided = ws.undec_pull;
  u.pub = Publish{a.pub_dead, a.pub_lo, a.pub_ldead, a.pub_cap};
  u.segflag = ws.segflag;
  u.tile_hit = a.tile ? ws.tile_hit : nullptr;
  u.rowtiles = a.rowtiles;
  u.nseg = a.nseg;
  u.total_tiles = a.total_tiles;
  u.seg_mode = a.seg_mode;
  u.rounds = ws.rounds;
  u.tail_thr = a.tail_thr;
  u.perm = a.perm;
  u.cb = a.cb;
  u.r1_max = a.r1_max;
  return u;
}

TailArgs tail_args(tcmis_graph *g, const RoundArgs &a) {
  Workspace &ws = g->ws;
  TailArgs t;
  t.off = a.off;
  t.nbr = a.nbr;
  t.vnnz = a.vnnz;
  t.prio = ws.prio;
  t.q = ws.q;
  t.next = ws.next;
  t.xt = ws.xt;
  t.tslot = ws.warpcnt + 2 * (size_t)kTailMaxWarps;
  t.state = ws.state;
  t.segflag = ws.segflag;
  t.segmark = ws.segmark;
  t.rowtiles = a.rowtiles;
  t.nseg = a.nseg;
  t.total_tiles = a.total_tiles;
  t.seg_mode = a.seg_mode;
  t.T = a.T;
  t.ctrl = ws.ctrl;
  t.wl0 = ws.wl[0];
  t.wl1 = ws.wl[1];
  t.rounds = ws.rounds;
  t.bar = ws.bar;
  t.n = a.n;
  t.mis = ws.mis;
  t.mis_count = ws.mis_count;
  t.warpcnt = ws.warpcnt;
  t.pack = nullptr;
  t.perm = a.perm;
  t.mis_o = a.mis_o;
  t.nz = a.nz;
  t.nz_count = a.nz_count;
  t.nz_identity = a.nz_count == a.n || a.nz_prefix ? 1 : 0;
  t.cb = a.cb;
  t.q_l1 = std::getenv("TCMIS_TAIL_Q_L2") ? 0 : 1;
  t.bar_fenced = std::getenv("TCMIS_TAIL_BAR_FENCE") ? 1 : 0;
  t.tag_par = std::getenv("TCMIS_TAIL_TAG_PAR") ? 1 : 0;

  return t;
}

// cooperative launch: the grid barriers of k_tail need every block resident
int launch_tail(tcmis_graph *g, const RoundArgs &a, HostRes *pack = nullptr) {
  TailArgs t = tail_args(g, a);
  t.pack = pack;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(a.tail_grid);
  lc.blockDim = dim3(kTailBlock);
  lc.dynamicSmemBytes = kTailDynSmem;
  lc.stream = g->ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  cudaError_t e = cudaSuccess;
  TCMIS_TIMED(g->ctx, "k_tail", (e = cudaLaunchKernelEx(&lc, k_tail, t)));
  TCMIS_CUDA(e);
  g->ctx->launches++;
  return 0;
}

int tail_grid(tcmis_ctx *ctx) {
  if (ctx->tail_blocks_per_sm == 0) {
    int per_sm = 0;
    cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailDynSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tail, kTailBlock, kTailDynSmem);
    ctx->tail_blocks_per_sm = per_sm > 0 ? per_sm : 1;
  }
  return ctx->num_sms * ctx->tail_blocks_per_sm;
}

// Round kernels (those starting with pdl_entry(), common.cuh) are launched
// with programmatic stream serialisation when TCMIS_PDL is set.
template <typename... KArgs, typename... Args>
cudaError_t launch_round_kernel(void (*k)(KArgs...), int grid, cudaStream_t st, Args... args) {
#if TCMIS_PDL
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(kBlock);
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, k, args...);
#else
  k<<<grid, kBlock, 0, st>>>(args...);
  return cudaSuccess;
#endif
}

int launch_select(tcmis_graph *g, const RoundArgs &a) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const SelectArgs s = select_args(g, a);
  if (a.tile)
    TCMIS_CUDA(cudaMemsetAsync(g->ws.cbits, 0, 4 * ((size_t)a.n / 32 + 1), st));
  if (a.tile_cand) {
    // Phase 1 as a tile product in the rounds that start with >= tile_gate
    // alive vertices (tile_cand.cu): alive bitmap, A-up tiles x alive ->
    // blocked rows, unblocked alive vertices -> candidates; in the other
    // rounds these three idle and the CSR select kernels below run
    Workspace &ws = g->ws;
    const int64_t words = ((int64_t)a.n + 31) / 32;
    TCMIS_TIMED(ctx, "k_alive_bits",
                (k_alive_bits<<<grid_for(ctx, words, 256, 8), 256, 0, st>>>(
                    a.n, ws.state, ws.alive_bits, ws.rounds, ws.ctrl, a.tile_gate)));
    TCMIS_LAUNCHED(ctx);
    if (a.tile_cand == 2) {  // the same product on tcgen05 (tile_umma.cuh)
      UmmaArgs u{a.up_tiles, a.up_trow, a.up_tcol, a.up_tbits, ws.alive_bits, ws.blocked,
                 ws.ctrl, a.tile_gate};
      TCMIS_TIMED(ctx, "k_tile_cand_umma",
                  (k_tile_umma<<<ctx->num_sms * 8, 128, 0, st>>>(u)));
    } else {
      TileExclArgs t{a.up_tiles, a.up_trow, a.up_tcol, a.up_tbits, ws.alive_bits, ws.blocked,
                     ws.ctrl, a.tile_gate};
      TCMIS_TIMED(ctx, "k_tile_cand_bits",
                  (k_tile_excl_bits<<<grid_for(ctx, a.up_tiles, 256, 8), 256, 0, st>>>(t)));
    }
    TCMIS_LAUNCHED(ctx);
    TCMIS_TIMED(ctx, "k_tile_mark",
                (k_tile_mark<<<grid_for(ctx, 32 * words, 256, 8), 256, 0, st>>>(
                    a.n, ws.alive_bits, ws.blocked, ws.cbits, ws.next, ws.state, s.segflag, a.T,
                    ws.ctrl, a.tile_gate, s.push, a.off, a.nbr)));
    TCMIS_LAUNCHED(ctx);
  }
  TCMIS_TIMED(ctx, "k_probe_select", (launch_round_kernel(k_probe_select, a.sel_grid, st, s)));
  TCMIS_LAUNCHED(ctx);
  TCMIS_TIMED(ctx, "k_select",
              (launch_round_kernel(a.n >= kSelWideN ? k_select<4> : k_select<kSelWin>,
                                   a.sel_grid, st, s)));
  TCMIS_LAUNCHED(ctx);
  TCMIS_TIMED(ctx, "k_select_long", (launch_round_kernel(k_select_long, a.sel_grid, st, s)));
  TCMIS_LAUNCHED(ctx);
  return 0;
}

int launch_update(tcmis_graph *g, const RoundArgs &a, cudaGraphConditionalHandle cond,
                  int use_cond) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  const UpdateArgs u = update_args(g, a);
  if (a.pull) {
    if (a.r1_max) {
      TCMIS_TIMED(ctx, "k_r1_pull", (launch_round_kernel(k_r1_pull, a.sel_grid, st, u)));
      TCMIS_LAUNCHED(ctx);
    }
    TCMIS_TIMED(ctx, "k_probe_pull", (launch_round_kernel(k_probe_pull, a.sel_grid, st, u)));
    TCMIS_LAUNCHED(ctx);
    TCMIS_TIMED(ctx, "k_update_pull", (launch_round_kernel(k_update_pull, a.sel_grid, st, u)));
  } else if (a.tile) {
    TCMIS_CUDA(cudaMemsetAsync(g->ws.tile_hit, 0, 4 * ((size_t)a.nb16 + 1), st));
    TileExclArgs t{a.store_tiles, a.trow, a.tcol, a.tbits, g->ws.cbits, g->ws.tile_hit, nullptr, 0};
    const int grid = grid_for(ctx, a.store_tiles, 256, 8);
    if (a.tile == 2)
      TCMIS_TIMED(ctx, "k_tile_excl_mma", (k_tile_excl_mma<<<grid, 256, 0, st>>>(t)));
    else
      TCMIS_TIMED(ctx, "k_tile_excl_bits", (k_tile_excl_bits<<<grid, 256, 0, st>>>(t)));
    TCMIS_LAUNCHED(ctx);
    TCMIS_TIMED(ctx, "k_update",
                (launch_round_kernel(k_update<false>, a.upd_grid, st, u, cond, 0)));
  } else {
    // push: the update kernel ends the round itself
    TCMIS_TIMED(ctx, "k_update",
                (launch_round_kernel(k_update<true>, a.upd_grid, st, u, cond, use_cond)));
    TCMIS_LAUNCHED(ctx);
    return 0;
  }
  TCMIS_LAUNCHED(ctx);
  TCMIS_TIMED(ctx, "k_round_end", (launch_round_kernel(k_round_end, a.upd_grid, st, u, cond, use_cond)));
  TCMIS_LAUNCHED(ctx);
  return 0;
}

inline int launches_per_round(const RoundArgs &a) {
  return ((a.pull || a.tile) ? 6 : 4) + (a.tile_cand ? 3 : 0) + (a.r1_max && a.pull ? 1 : 0);
}

// The parameters of a solve's first kernels (segment-flag clear,
// k_priorities with the control-block init), part of the graph's cache key.
struct SolvePre {
  int H;
  uint64_t seed;
  int scale_bits;
  int T;
  int seg_mode;
  int32_t nseg;
  Ctrl c0;
};

// Instantiate (once per distinct argument set) the whole-solve graph
//   memset(segflag) -> k_priorities -> WHILE(cond) { select ; exclusion ; update }
//     -> k_tail (rounds <= tail_thr + MIS compaction) | cub compaction
//     -> [h3: tile total] -> k_pack (results into mapped host memory)
// over this workspace's buffers.
int ensure_solve_graph(tcmis_graph *g, const RoundArgs &a, const SolvePre &pre) {
  Workspace &ws = g->ws;
  static_assert(sizeof(RoundArgs) + sizeof(SolvePre) <= sizeof(ws.graph_key), "graph key too small");
  unsigned char key[sizeof(ws.graph_key)] = {};
  std::memcpy(key, &a, sizeof(a));
  std::memcpy(key + sizeof(a), &pre, sizeof(pre));
  if (ws.exec && std::memcmp(ws.graph_key, key, sizeof(key)) == 0) return 0;
  if (ws.exec) {
    cudaGraphExecDestroy(ws.exec);
    ws.exec = nullptr;
  }
  tcmis_ctx *ctx = g->ctx;
  const int64_t launches0 = ctx->launches;  // capture is not execution
  cudaStream_t st = ctx->stream;
  cudaGraph_t graph = nullptr;
  TCMIS_CUDA(cudaGraphCreate(&graph, 0));
  int rc = 0;
  cudaError_t e = cudaSuccess;
  cudaGraph_t captured = nullptr;
  // 1. the first kernels
  e = cudaStreamBeginCaptureToGraph(st, graph, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) rc = cuda_error(e, "cudaStreamBeginCaptureToGraph(pre)");
  if (!rc) {
    if (pre.seg_mode) {
      e = cudaMemsetAsync(ws.segflag, 0, (size_t)pre.nseg, st);
      if (e != cudaSuccess) rc = cuda_error(e, "memset(segflag)");
    }
    if (!rc && a.mis_o) {
      e = cudaMemsetAsync(a.mis_o, 0, (size_t)g->n, st);
      if (e != cudaSuccess) rc = cuda_error(e, "memset(mis_o)");
    }
    if (!rc && a.r1_max)  // degree order: init and round 1's settle in one pass
      rc = launch_prio_settle(g, a, pre.seed, pre.scale_bits, pre.H,
                              pre.seg_mode ? ws.segflag : nullptr, pre.c0);
    else if (!rc)
      rc = launch_priorities(g, pre.H, pre.seed, pre.scale_bits, ws.prio, ws.q, ws.state, ws.next,
                             pre.seg_mode ? ws.segflag : nullptr, pre.T, ws.ctrl, &pre.c0,
                             ws.rounds, ws.round_cap, a.off, a.perm, a.mis_o);
    e = cudaStreamEndCapture(st, &captured);
    if (!rc && e != cudaSuccess) rc = cuda_error(e, "cudaStreamEndCapture(pre)");
  }
  // the pre-part's leaf (k_priorities) is the node without dependents
  cudaGraphNode_t leaf = nullptr;
  if (!rc) {
    size_t nn = 0;
    cudaGraphGetNodes(graph, nullptr, &nn);
    std::vector<cudaGraphNode_t> nodes(nn);
    cudaGraphGetNodes(graph, nodes.data(), &nn);
    for (cudaGraphNode_t nd : nodes) {
      size_t nd_out = 0;
      cudaGraphNodeGetDependentNodes(nd, nullptr, &nd_out);
      if (nd_out == 0) leaf = nd;
    }
    if (!leaf) rc = set_error(TCMIS_E_CUDA, "solve graph: no leaf after the first kernels");
  }
  // 2. WHILE(cond) { select ; exclusion ; update }
  cudaGraphConditionalHandle cond;
  cudaGraphNode_t node = nullptr;
  if (!rc) {
    // the loop's first test: round 1 runs in the round kernels unless the
    // whole solve is the tail's
    e = cudaGraphConditionalHandleCreate(&cond, graph, a.tail_from1 ? 0 : 1,
                                         cudaGraphCondAssignDefault);
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = cond;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    if (e == cudaSuccess) e = cudaGraphAddNode(&node, graph, &leaf, 1, &p);
    if (e != cudaSuccess) rc = cuda_error(e, "solve graph: WHILE node");
    cudaGraph_t body = p.conditional.phGraph_out[0];
    if (!rc) {
      e = cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed);
      if (e != cudaSuccess) rc = cuda_error(e, "cudaStreamBeginCaptureToGraph(body)");
    }
    if (!rc) {
      rc = launch_select(g, a);
      if (!rc) rc = launch_update(g, a, cond, 1);
      e = cudaStreamEndCapture(st, &captured);
      if (!rc && e != cudaSuccess) rc = cuda_error(e, "cudaStreamEndCapture(body)");
    }
  }
  // 3. tail + compaction, h3's tile total, and the result pack
  if (!rc) {
    e = cudaStreamBeginCaptureToGraph(st, graph, &node, nullptr, 1, cudaStreamCaptureModeRelaxed);
    if (e != cudaSuccess) rc = cuda_error(e, "cudaStreamBeginCaptureToGraph(post)");
    if (!rc) {
      const bool gather = a.perm && !a.mis_o;  // no fused compaction (tail.cuh)
      const bool tail_packs = a.tail_thr > 0 && pre.seg_mode != 2 && !gather;
      if (a.tail_thr > 0) rc = launch_tail(g, a, tail_packs ? ws.d_res : nullptr);
      if (!rc && gather) {
        rc = gc_compact(g);
      } else if (!rc && a.tail_thr == 0) {
        thrust::counting_iterator<int32_t> ids(0);
        size_t bytes = ws.cub_bytes;
        e = a.mis_o ? cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, ws.mis, ws.mis_count,
                                                     (int)g->n, IsMember{a.mis_o}, st)
                             : cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, ws.mis, ws.mis_count,
                                                     (int)g->n, IsInMIS{ws.state}, st);
        if (e != cudaSuccess) rc = cuda_error(e, "MIS compaction");
      }
      if (!rc && pre.seg_mode == 2) {
        cudaMemsetAsync(&ws.ctrl->eval, 0, sizeof(unsigned long long), st);
        k_seg_total<<<grid_for(ctx, pre.nseg, 256, 4), 256, 0, st>>>(ws.segflag, g->d_rowtiles,
                                                                     pre.nseg, ws.ctrl);
      }
      if (!rc && !tail_packs)
        k_pack<<<1, 64, 0, st>>>(ws.ctrl, ws.mis_count, ws.rounds, ws.round_cap, ws.d_res);
      e = cudaStreamEndCapture(st, &captured);
      if (!rc && e != cudaSuccess) rc = cuda_error(e, "cudaStreamEndCapture(post)");
    }
  }
  if (!rc) {
    e = cudaGraphInstantiate(&ws.exec, graph, 0);
    if (e != cudaSuccess) rc = cuda_error(e, "cudaGraphInstantiate");
  }
  cudaGraphDestroy(graph);
  ctx->launches = launches0;
  if (!rc) std::memcpy(ws.graph_key, key, sizeof(key));
  return rc;
}

// Tiles in the block columns holding any flagged segment (h3's single
// iteration counter, also used per rank by the multi-GPU driver).
int seg_total(tcmis_graph *g, int64_t *ev) {
  tcmis_ctx *ctx = g->ctx;
  Workspace &ws = g->ws;
  unsigned long long h = 0;
  TCMIS_CUDA(cudaMemsetAsync(&ws.ctrl->eval, 0, sizeof(unsigned long long), ctx->stream));
  k_seg_total<<<grid_for(ctx, g->tile_nb, 256, 4), 256, 0, ctx->stream>>>(
      ws.segflag, g->d_rowtiles, g->tile_nb, ws.ctrl);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaMemcpyAsync(&h, &ws.ctrl->eval, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  TCMIS_CUDA(cudaStreamSynchronize(ctx->stream));
  *ev = (int64_t)h;
  return 0;
}

// The setup of a solve (validation, tile counts, priorities, round state and
// the kernel arguments) for the multi-GPU driver (dist.cu): `isolated` is the
// number of round-1 candidates settled by k_priorities on this rank.
int solve_prepare(tcmis_graph *g, const tcmis_config *cfg, RoundArgs &a, int64_t isolated) {
  if (int rc = validate(g, cfg)) return rc;
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (int rc = ensure_workspace(g)) return rc;
  Workspace &ws = g->ws;
  const int H = cfg->heuristic;
  const bool tiled = H <= TCMIS_H3;
  const int T = cfg->tile_dim;
  if (tiled && g->tile_T != T)
    if (int rc = build_tile_counts(g, T)) return rc;
  const int32_t nseg = tiled ? g->tile_nb : 0;
  const int seg_mode = !tiled ? 0 : (H == TCMIS_H3 ? 2 : 1);
  if (seg_mode) TCMIS_CUDA(cudaMemsetAsync(ws.segflag, 0, (size_t)nseg, st));
  if (int rc = launch_priorities(g, H, cfg->seed, cfg->scale_bits, ws.prio, ws.q, ws.state,
                                 ws.next, seg_mode ? ws.segflag : nullptr, T > 0 ? T : 1))
    return rc;
  Ctrl c0{};
  c0.round = 1;
  c0.alive = g->n;
  c0.max_rounds = ws.round_cap;
  c0.sel = (unsigned long long)isolated;
  *ws.h_ctrl = c0;
  TCMIS_CUDA(cudaMemcpyAsync(ws.ctrl, ws.h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
  std::memset(&a, 0, sizeof(a));
  a.n = g->n;
  a.off = g->d_off;
  a.nbr = g->d_nbr;
  a.T = T > 0 ? T : 1;
  a.seg_mode = seg_mode;
  a.nseg = nseg;
  a.total_tiles = g->tile_total;
  a.rowtiles = g->d_rowtiles;
  a.fresh = H == TCMIS_LUBY_FRESH ? 1 : 0;
  a.seed = cfg->seed;
  a.sel_grid = ctx->num_sms * 8;
  a.upd_grid = ctx->num_sms * 4;
  a.nz = g->d_nz;
  a.vnnz = ((uintptr_t)g->d_nbr & 15) == 0 ? g->nnz : -g->nnz;
  a.nz_count = g->nz_count;
  a.pull = 1;
  TCMIS_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int solve_impl(tcmis_graph *g, const tcmis_config *cfg, tcmis_iter_stats *stats,
               int32_t max_stats, int32_t *n_iter, int64_t *mis_count_out) {
  if (int rc = validate(g, cfg)) return rc;
  *n_iter = 0;
  *mis_count_out = 0;
  if (g->n == 0) return 0;  // engine.cpp:240 / 307
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (int rc = ensure_workspace(g)) return rc;
  Workspace &ws = g->ws;
  const int H = cfg->heuristic;
  const bool tiled = H <= TCMIS_H3;
  const bool fresh = H == TCMIS_LUBY_FRESH;
  const int T = cfg->tile_dim;
  if (tiled && g->tile_T != T)
    if (int rc = build_tile_counts(g, T)) return rc;
  const int32_t nseg = tiled ? g->tile_nb : 0;
  const int seg_mode = !tiled ? 0 : (H == TCMIS_H3 ? 2 : 1);
  const bool timing = (cfg->flags & TCMIS_F_TIMING) != 0;
  // run_luby_reference never calls the hook (engine.cpp:301-352)
  tcmis_config cfg_local = *cfg;
  if (!tiled) cfg_local.observer = nullptr;
  cfg = &cfg_local;
  // an internal vertex order (order.cu): the kernels run on the relabeled CSR
  // (not for the observer, whose snapshots are in the caller's order, nor for
  // the tile forms, whose store is built on the caller's CSR)
  const bool tile_cand = (cfg->flags & TCMIS_F_TILE_CAND) != 0;
  if (tile_cand && fresh)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "TCMIS_F_TILE_CAND needs fixed priorities (not luby-fresh)");
  const bool tile_form = cfg->exclusion == TCMIS_EXCL_TILE_BITS ||
                         cfg->exclusion == TCMIS_EXCL_TILE_MMA;
  // (nor for the tile-form Phase 1, whose A-up store is too)
  const bool relabel = g->d_perm && !cfg->observer && !tile_form && !tile_cand;
  const int64_t *s_off = relabel ? g->d_roff : g->d_off;
  const int32_t *s_nbr = relabel ? g->d_rnbr : g->d_nbr;
  const int32_t *s_perm = relabel ? g->d_perm : nullptr;
  // the caller-order membership plane: kept while it stays L2-resident next
  // to the gathered vectors (R-MAT s26's 67 MB plane cost its select kernels
  // more in scattered stores, 3.45 -> 3.56 ms, than the gather compaction)
  int64_t mis_o_max = kMisOMax;
  if (const char *env = std::getenv("TCMIS_MIS_O_MAX")) mis_o_max = std::atoll(env);  // test hook
  const bool use_mis_o = relabel && (int64_t)g->n <= mis_o_max;
  if (use_mis_o && !ws.mis_o)
    // sized by the workspace's capacity, not this graph's n: the workspace is
    // adopted by later graphs up to n_cap vertices (tcmis_graph_destroy)
    if (int rc = dev_alloc(&ws.mis_o, ws.n_cap + 16)) return rc;  // uint4 reads past n
  uint8_t *s_mis_o = use_mis_o ? ws.mis_o : nullptr;
  ws.relabeled = relabel;
  if (relabel && !use_mis_o)
    if (int rc = gc_prepare(g)) return rc;
  // the degree-class bounds: a degree order under the H2 priorities
  // (h2 / h3 / luby-perm), computed once per scale_bits
  const int2 *s_cb = nullptr;
  if (relabel && g->order_mode == TCMIS_ORDER_DEGREE && g->d_cls_start && g->n_cls > 0 &&
      (H == TCMIS_H2 || H == TCMIS_H3 || H == TCMIS_LUBY_PERM) &&
      std::getenv("TCMIS_NO_CLASS_BOUNDS") == nullptr) {
    if (g->cb_scale_bits != cfg->scale_bits) {
      if (!g->d_cb)
        if (int rc = dev_alloc(&g->d_cb, (size_t)g->max_degree + 1)) return rc;
      if (!g->d_cbc)
        if (int rc = dev_alloc(&g->d_cbc, (size_t)g->n_cls)) return rc;
      k_class_bounds<<<grid_for(ctx, g->n_cls, 128, 4), 128, 0, st>>>(
          g->n_cls, g->d_cls_start, g->d_roff, avg_degree(g), (double)(1u << cfg->scale_bits),
          g->d_cb, g->d_cbc);
      TCMIS_LAUNCHED(ctx);
      g->cb_scale_bits = cfg->scale_bits;
    }
    s_cb = g->d_cb;
  }

  if (timing) timeline_begin(ctx);
  uint8_t *seg0 = seg_mode ? ws.segflag : nullptr;
  Ctrl c0{};
  c0.round = 1;
  c0.alive = g->n;
  c0.max_rounds = ws.round_cap;
  c0.sel = (unsigned long long)(g->n - g->nz_count);  // isolated: round-1 candidates
  // test hook: a control block that disagrees with the states, which the
  // round-end invariant check must report as the reference's logic_error
  if (cfg->flags & TCMIS_F_DEBUG_CORRUPT) c0.alive += 1;
  *ws.h_ctrl = c0;
  bool step = cfg->observer || timing || (cfg->flags & TCMIS_F_HOST_LOOP);
  // the solve's first kernels: segment flags cleared, priorities, states, and
  // the control block + zeroed statistics ring (k_tail accumulates into it)
  RoundArgs a;
  std::memset(&a, 0, sizeof(a));
  auto launch_pre = [&]() -> int {
    if (seg_mode) TCMIS_CUDA(cudaMemsetAsync(ws.segflag, 0, (size_t)nseg, st));
    if (s_mis_o) TCMIS_CUDA(cudaMemsetAsync(s_mis_o, 0, (size_t)g->n, st));
    if (a.r1_max)  // degree order: init and round 1's settle in one pass
      return launch_prio_settle(g, a, cfg->seed, cfg->scale_bits, H, seg0, c0);
    return launch_priorities(g, H, cfg->seed, cfg->scale_bits, ws.prio, ws.q, ws.state, ws.next,
                             seg0, T > 0 ? T : 1, ws.ctrl, &c0, ws.rounds, ws.round_cap, s_off,
                             s_perm, s_mis_o);
  };

  a.n = g->n;
  a.off = s_off;
  a.nbr = s_nbr;
  a.perm = s_perm;
  a.mis_o = s_mis_o;
  a.cb = s_cb;
  if (s_cb && g->d_rmax && g->d_vcls && std::getenv("TCMIS_NO_R1_SETTLE") == nullptr) {
    a.cbc = g->d_cbc;
    a.r1_max = g->d_rmax;
    a.r1_cls = g->d_vcls;
  }
  a.nz_prefix = relabel && g->order_mode == TCMIS_ORDER_DEGREE ? 1 : 0;
  a.T = T > 0 ? T : 1;
  a.seg_mode = seg_mode;
  a.nseg = nseg;
  a.total_tiles = g->tile_total;
  a.rowtiles = g->d_rowtiles;
  a.fresh = fresh ? 1 : 0;
  a.seed = cfg->seed;
  a.sel_grid = ctx->num_sms * 8;
  a.upd_grid = ctx->num_sms * 4;
  a.nz = relabel ? g->d_rnz : g->d_nz;
  a.vnnz = ((uintptr_t)s_nbr & 15) == 0 ? g->nnz : -g->nnz;
  a.nz_count = relabel ? g->rnz_count : g->nz_count;
  // exclusion form: pull on degree-skewed graphs, where the
  // neighbours of candidates concentrate on hubs and early-exit pulls are
  // cheap; push elsewhere.  Both produce the same next[] decisions.
  if (cfg->exclusion == TCMIS_EXCL_PUSH) {
    a.pull = 0;
  } else if (cfg->exclusion == TCMIS_EXCL_CSR_PULL) {
    a.pull = 1;
  } else if (tile_form) {
    // the paper's tile form over the compact T = 16 store (tile_excl.cuh);
    // built once per graph, like tile_graph in run_tc_mis(g, cfg)
    if (int rc = build_tile_store(g, 16)) return rc;
    a.pull = 0;
    a.tile = cfg->exclusion == TCMIS_EXCL_TILE_MMA ? 2 : 1;
    a.nb16 = (int32_t)(((int64_t)g->n + 15) / 16);
    a.store_tiles = g->store_tiles;
    a.trow = g->d_trow;
    a.tcol = g->d_tcol;
    a.tbits = static_cast<const uint16_t *>(g->d_tbits);
  } else {
    a.pull = (double)g->max_degree > 64.0 * std::max(1.0, avg_degree(g)) ? 1 : 0;
  }
  if (tile_cand) {
    const int64_t key[3] = {H, (int64_t)cfg->seed, cfg->scale_bits};
    if (int rc = tile_cand_prepare(g, H, cfg->seed, cfg->scale_bits, key, nullptr)) return rc;
    a.tile_cand = (cfg->flags & TCMIS_F_TILE_UMMA) ? 2 : 1;
    a.up_tiles = g->up_tiles;
    a.up_trow = g->d_up_trow;
    a.up_tcol = g->d_up_tcol;
    a.up_tbits = g->d_up_tbits;
    a.nb16 = (int32_t)(((int64_t)g->n + 15) / 16);
    // tile rounds: those starting with at least a quarter of the vertices
    // alive (the tile kernels pay for every tile each round; the CSR scan
    // engines only for the alive rows).  TCMIS_TILE_CAND_GATE overrides.
    a.tile_gate = std::max<int32_t>(1, g->n / 4);
    if (const char *env = std::getenv("TCMIS_TILE_CAND_GATE")) a.tile_gate = std::atoi(env);
  }
  // small late rounds run in the persistent k_tail (not with the per-round
  // observer hook, which needs every round's snapshot)
  a.tail_thr = 0;
  // (luby-fresh redraws every survivor's priority between rounds, which the
  // tail's one-barrier rounds cannot order: it keeps the per-round kernels)
  if (!cfg->observer && !fresh) {
    a.tail_thr = 1 << 16;
    if (const char *env = std::getenv("TCMIS_TAIL_THRESHOLD")) a.tail_thr = std::atoi(env);
    a.tail_grid = tail_grid(ctx);
    // k_tail keeps each block's share of its starting list in shared memory,
    // one vertex per thread (tail.cuh): at most kTailBlock per block
    a.tail_thr = (int32_t)std::min<int64_t>(a.tail_thr, (int64_t)a.tail_grid * kTailBlock);
    // a small graph whose non-isolated vertices all fit the tail's lists
    // runs every round there: no round-kernel launches at all.  On a degree
    // order the fused round-1 verdicts (k_prio_settle, round-kernel work)
    // give way to the plain init, and the tail's scans use the class bounds
    // from round 1 on.  (AUTO exclusion only: an explicit exclusion form or
    // the tile Phase 1 asks for the round kernels; with TCMIS_TAIL_THRESHOLD
    // set, only when the non-isolated vertices are within it)
    const int64_t cap = (int64_t)a.tail_grid * kTailBlock;
    const char *whole = std::getenv("TCMIS_TAIL_WHOLE");
    const bool thr_env = std::getenv("TCMIS_TAIL_THRESHOLD") != nullptr;
    if (a.nz_count > 0 && a.nz_count <= cap && (!thr_env || a.nz_count <= a.tail_thr) && a.tail_thr > 0 &&
        !a.tile_cand && cfg->exclusion == TCMIS_EXCL_AUTO && !(whole && whole[0] == '0')) {
      a.tail_thr = (int32_t)cap;
      a.tail_from1 = 1;
      a.r1_max = nullptr;
      a.r1_cls = nullptr;
      a.cbc = nullptr;
    }
  }
  if (step)
    if (int rc = launch_pre()) return rc;
  if (seg_mode == 1 && a.tail_thr > 0)
    TCMIS_CUDA(cudaMemsetAsync(ws.segmark, 0, sizeof(uint32_t) * (size_t)nseg, st));

  std::vector<DevRound> rounds_h;
  std::vector<uint8_t> h_next, h_state, h_cand;
  std::vector<float> t1, t2, t3;  // per-round phase times (TCMIS_F_TIMING)
  int64_t h_mis_count = 0;
  unsigned long long h3_eval = 0;
  // ascending MIS ids (engine.cpp:293 sorts; ordered compaction needs no sort)
  // and h3's collapsed tile counter, enqueued behind the rounds
  bool tail_compacted = false;  // k_tail ends with the MIS compaction (tail.cuh)
  auto enqueue_finish = [&]() -> int {
    if (!tail_compacted) {
      thrust::counting_iterator<int32_t> ids(0);
      size_t bytes = ws.cub_bytes;
      if (a.perm && !a.mis_o) {
        if (int rc = gc_compact(g)) return rc;
      } else if (a.mis_o)
        TCMIS_CUDA(cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, ws.mis, ws.mis_count,
                                         (int)g->n, IsMember{a.mis_o}, st));
      else
        TCMIS_CUDA(cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, ws.mis, ws.mis_count,
                                         (int)g->n, IsInMIS{ws.state}, st));
      ctx->launches += 1;
    }
    TCMIS_CUDA(cudaMemcpyAsync(&ws.h_misc[0], ws.mis_count, sizeof(int64_t),
                               cudaMemcpyDeviceToHost, st));
    if (seg_mode == 2) {
      TCMIS_CUDA(cudaMemsetAsync(&ws.ctrl->eval, 0, sizeof(unsigned long long), st));
      k_seg_total<<<grid_for(ctx, nseg, 256, 4), 256, 0, st>>>(ws.segflag, g->d_rowtiles, nseg,
                                                               ws.ctrl);
      TCMIS_LAUNCHED(ctx);
      TCMIS_CUDA(cudaMemcpyAsync(&ws.h_misc[1], &ws.ctrl->eval, sizeof(int64_t),
                                 cudaMemcpyDeviceToHost, st));
    }
    return 0;
  };
  auto read_finish = [&]() {  // after the stream synchronisation
    h_mis_count = ws.h_misc[0];
    h3_eval = seg_mode == 2 ? (unsigned long long)ws.h_misc[1] : 0ull;
  };
  bool finished = false;
  if (!step) {
    // the whole solve is one CUDA graph (ensure_solve_graph): priorities,
    // a conditional WHILE node over {select, exclusion, update} whose loop
    // condition k_round_end sets on the device, the persistent tail with the
    // fused MIS compaction, and k_pack, which leaves the control block, the
    // MIS count and the statistics in mapped host memory -- one launch, one
    // synchronisation, no copies.
    SolvePre pre{};
    pre.H = H;
    pre.seed = cfg->seed;
    pre.scale_bits = cfg->scale_bits;
    pre.T = T > 0 ? T : 1;
    pre.seg_mode = seg_mode;
    pre.nseg = nseg;
    pre.c0 = c0;
    if (int rc = ensure_solve_graph(g, a, pre)) return rc;
    TCMIS_CUDA(cudaGraphLaunch(ws.exec, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    const HostRes &hr = *ws.h_res;
    *ws.h_ctrl = hr.ctrl;
    if (hr.ctrl.overflow) {
      // more rounds than the on-device ring holds: redo step-wise, draining
      // the statistics every round (pathological inputs such as long paths)
      step = true;
      a.tail_thr = 0;
      a.tail_from1 = 0;
      tail_compacted = false;
      *ws.h_ctrl = c0;
      if (int rc = launch_pre()) return rc;
    } else {
      const int rr = hr.ctrl.round - 1;
      const int mr = hr.ctrl.main_rounds;
      // k_priorities, the rounds, the tail (or cub's compaction), and k_pack
      // unless the tail packed (h3 adds k_seg_total)
      const bool gather = a.perm && !a.mis_o;
      const bool tail_packs = a.tail_thr > 0 && seg_mode != 2 && !gather;
      ctx->launches += 2 + (a.r1_max ? 1 : 0) + launches_per_round(a) * (int64_t)mr +
                       (seg_mode == 2 ? 1 : 0) + (tail_packs ? 0 : 1) +
                       (gather && a.tail_thr > 0 ? 3 : 0);
      const int pre_n = std::min(rr, std::min(ws.round_cap, 64));
      rounds_h.assign(hr.rounds, hr.rounds + pre_n);
      if (rr > pre_n) {
        rounds_h.resize(rr);
        TCMIS_CUDA(cudaMemcpy(rounds_h.data() + pre_n, ws.rounds + pre_n,
                              sizeof(DevRound) * (rr - pre_n), cudaMemcpyDeviceToHost));
      }
      h_mis_count = hr.mis_count;
      h3_eval = seg_mode == 2 ? hr.ctrl.eval : 0ull;
      finished = true;
    }
  }
  // the rounds after `done` (0 = all of them) in k_tail, their statistics to the host
  auto run_tail_from = [&](int done) -> int {
    ctx->rec_round = done + 1;
    if (int rc = launch_tail(g, a)) return rc;
    tail_compacted = !(a.perm && !a.mis_o);
    TCMIS_CUDA(cudaMemcpyAsync(ws.h_ctrl, ws.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    const int rr = ws.h_ctrl->round - 1;
    if (rr - done > ws.round_cap)
      return set_error(TCMIS_E_RUNTIME, "round statistics capacity exceeded in k_tail");
    for (int r = done; r < rr; ++r) {
      DevRound dr;
      TCMIS_CUDA(cudaMemcpy(&dr, ws.rounds + r % ws.round_cap, sizeof(DevRound),
                            cudaMemcpyDeviceToHost));
      rounds_h.push_back(dr);
    }
    return 0;
  };
  if (step && a.tail_from1) {
    if (int rc = run_tail_from(0)) return rc;
  } else if (step) {
    int round = 0;
    for (;;) {
      ++round;
      if (round > g->n)  // engine.cpp:248-249
        return set_error(TCMIS_E_RUNTIME, "iteration cap exceeded; engine livelock");
      ctx->rec_round = round;
      TCMIS_RANGE("host-loop round");
      if (int rc = launch_select(g, a)) return rc;
      if (cfg->observer && H != TCMIS_H3) {
        // the select kernels already moved this round's candidates to InMIS;
        // the hook gets the states the candidates were generated against
        // (engine.cpp:275-278), i.e. the host copy taken after the last round
        if (h_state.empty()) h_state.assign(g->n, TCMIS_ALIVE);
        h_next.resize(g->n);
        h_cand.resize(g->n);
        TCMIS_CUDA(cudaMemcpyAsync(h_next.data(), ws.next, g->n, cudaMemcpyDeviceToHost, st));
        TCMIS_CUDA(cudaStreamSynchronize(st));
        for (int32_t v = 0; v < g->n; ++v)
          h_cand[v] = h_next[v] == 1 && h_state[v] == TCMIS_ALIVE;
        cfg->observer(cfg->observer_user, round, h_cand.data(), h_state.data(), g->n);
      }
      if (int rc = launch_update(g, a, 0, 0)) return rc;
      if (cfg->observer && H != TCMIS_H3)
        TCMIS_CUDA(cudaMemcpyAsync(h_state.data(), ws.state, g->n, cudaMemcpyDeviceToHost, st));
      TCMIS_CUDA(cudaMemcpyAsync(ws.h_ctrl, ws.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
      DevRound dr;
      TCMIS_CUDA(cudaMemcpyAsync(&dr, ws.rounds + (round - 1) % ws.round_cap, sizeof(DevRound),
                                 cudaMemcpyDeviceToHost, st));
      TCMIS_CUDA(cudaStreamSynchronize(st));
      rounds_h.push_back(dr);
      if (ws.h_ctrl->alive == 0 || ws.h_ctrl->corrupt) break;
      if (a.tail_thr > 0 && ws.h_ctrl->alive <= a.tail_thr) {
        if (int rc = run_tail_from(round)) return rc;
        break;
      }
    }
  }
  const int rounds_run = (int)rounds_h.size();
  if (!finished)
    if (int rc = enqueue_finish()) return rc;
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (!finished) read_finish();
  *mis_count_out = h_mis_count;
  {
    const Ctrl &cf = finished ? ws.h_res->ctrl : *ws.h_ctrl;
    int32_t corrupt = cf.corrupt;
    if (!finished) {  // the host loop's last control block copy may predate the tail
      Ctrl c{};
      TCMIS_CUDA(cudaMemcpy(&c, ws.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
      corrupt = c.corrupt;
    }
    if (corrupt)  // engine.cpp:152-153
      return set_error(TCMIS_E_LOGIC,
                       "candidate flagged on a non-alive vertex (a round's selected + removed + "
                       "alive differs from its alive count before)");
  }
  if (!timing) {
    // the phase stamps the round kernels left in the ring (%globaltimer):
    // Phase 1 = select (push exclusion fused), Phase 2 = pull / tile
    // exclusion, Phase 3 = update and round end; a k_tail round fuses all
    // three and reports its pass + barrier as Phase 1
    auto span_ms = [](unsigned long long a0, unsigned long long a1) {
      return (a0 && a1 && a1 > a0) ? (float)((double)(a1 - a0) * 1e-6) : 0.f;
    };
    t1.assign(rounds_h.size(), 0.f);
    t2.assign(rounds_h.size(), 0.f);
    t3.assign(rounds_h.size(), 0.f);
    for (size_t r = 0; r < rounds_h.size(); ++r) {
      const DevRound &d = rounds_h[r];
      const unsigned long long p2 = d.t[1] ? d.t[1] : d.t[2];
      t1[r] = span_ms(d.t[0], p2 ? p2 : d.t[3]);
      t2[r] = span_ms(d.t[1], d.t[2]);
      t3[r] = span_ms(d.t[2], d.t[3]);
    }
  }
  if (timing) {
    // Phase 1 = the select kernels, Phase 2 = the pull-form exclusion
    // kernels (push-form exclusion is fused into Phase 1), Phase 3 = update;
    // the tail kernel's rounds share one launch (reported on its first round)
    timeline_end(ctx);
    t1.assign(rounds_h.size(), 0.f);
    t2.assign(rounds_h.size(), 0.f);
    t3.assign(rounds_h.size(), 0.f);
    for (const auto &k : ctx->timeline) {
      const int r = k.round - 1;
      if (r < 0 || r >= (int)rounds_h.size()) continue;
      const std::string nm(k.name);
      if (nm == "k_probe_pull" || nm == "k_update_pull" || nm == "k_tile_excl_bits" ||
          nm == "k_tile_excl_mma")
        t2[r] += k.ms;
      else if (nm == "k_update" || nm == "k_round_end") t3[r] += k.ms;
      else t1[r] += k.ms;
    }
  }

  if (H == TCMIS_H3) {
    // engine.cpp:255-258: the h3 candidate vector is already the whole MIS,
    // so the reference reports exactly one iteration.
    if (cfg->observer) {
      h_state.assign(g->n, TCMIS_ALIVE);
      h_cand.resize(g->n);
      std::vector<uint8_t> fin(g->n);
      TCMIS_CUDA(cudaMemcpy(fin.data(), ws.state, g->n, cudaMemcpyDeviceToHost));
      for (int32_t v = 0; v < g->n; ++v) h_cand[v] = fin[v] == TCMIS_IN_MIS;
      cfg->observer(cfg->observer_user, 1, h_cand.data(), h_state.data(), g->n);
    }
    tcmis_iter_stats s{};
    s.iteration = 1;
    s.candidates_selected = h_mis_count;
    s.vertices_removed = g->n - h_mis_count;
    s.alive_remaining = 0;
    s.tiles_evaluated = (int64_t)h3_eval;
    s.tiles_skipped = g->tile_total - (int64_t)h3_eval;
    for (size_t i = 0; i < t1.size(); ++i) {
      s.phase1_ms += t1[i];
      s.phase2_ms += t2[i];
      s.phase3_ms += t3[i];
    }
    if (stats && max_stats > 0) stats[0] = s;
    *n_iter = 1;
    return 0;
  }
  for (int r = 0; r < rounds_run; ++r) {
    if (!stats || r >= max_stats) break;
    const DevRound &d = rounds_h[r];
    tcmis_iter_stats s{};
    s.iteration = r + 1;
    s.candidates_selected = (int64_t)d.sel;
    s.vertices_removed = (int64_t)d.rem;
    s.alive_remaining = (int64_t)d.alive;
    s.tiles_evaluated = (int64_t)d.eval;
    s.tiles_skipped = (int64_t)d.skip;
    if (r < (int)t1.size()) {
      s.phase1_ms = t1[r];
      s.phase2_ms = t2[r];
      s.phase3_ms = t3[r];
    }
    stats[r] = s;
  }
  *n_iter = rounds_run;
  return 0;
}

// the A-up store of the priorities (H, seed, scale_bits), built from the
// priorities of this graph if not cached (tile_cand.cu)
int tile_cand_prepare(tcmis_graph *g, int H, uint64_t seed, int scale_bits, const int64_t key[3],
                      double *build_ms) {
  if (build_ms) *build_ms = 0;
  if (g->d_up_trow && g->up_key[0] == key[0] && g->up_key[1] == key[1] && g->up_key[2] == key[2])
    return 0;
  uint32_t *d_p = nullptr;
  if (int rc = dev_alloc(&d_p, (size_t)g->n)) return rc;
  int rc = launch_priorities(g, H, seed, scale_bits, d_p, nullptr, nullptr, nullptr);
  if (!rc) rc = build_up_store(g, d_p, key, build_ms);
  dev_free(d_p);
  if (!rc && build_ms) g->up_build_ms = *build_ms;
  return rc;
}

int states_in_caller_order(tcmis_graph *g) {
  Workspace &ws = g->ws;
  if (!ws.relabeled || !g->d_inv) return 0;
  if (!ws.state_o)
    if (int rc = dev_alloc(&ws.state_o, ws.n_cap + 16)) return rc;  // capacity, as mis_o
  k_unpermute<<<grid_for(g->ctx, g->n, 256, 8), 256, 0, g->ctx->stream>>>(g->n, g->d_inv,
                                                                          ws.state, ws.state_o);
  TCMIS_LAUNCHED(g->ctx);
  return 0;
}

// ----------------------------------------------- partitioned solve's tail

// the alive subgraph's starting state from the rank's replicated vectors
__global__ void k_sub_init(int32_t A, const int32_t *__restrict__ ids,
                           const uint32_t *__restrict__ prio, const uint16_t *__restrict__ q,
                           uint32_t *__restrict__ sprio, uint16_t *__restrict__ sq,
                           uint8_t *__restrict__ sstate, uint8_t *__restrict__ snext,
                           int32_t *__restrict__ wl) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    sprio[i] = prio[v];
    sq[i] = q[v];
    sstate[i] = TCMIS_ALIVE;
    snext[i] = 0;
    wl[i] = (int32_t)i;
  }
}

__global__ void k_sub_scatter(int32_t A, const int32_t *__restrict__ ids,
                              const uint8_t *__restrict__ sstate, uint8_t *__restrict__ state,
                              uint16_t *__restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < A;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[i];
    const uint8_t s = sstate[i];
    state[v] = s;
    if (s == TCMIS_REMOVED) q[v] = 0;
  }
}

// The late rounds of a partitioned solve on ONE device (partitioned.cu): the
// alive subgraph -- sub vertex i = the caller's vertex ids[i], ids ascending,
// so the key order of (p, id) is kept; rows hold only alive neighbours (a
// vertex with an InMIS neighbour is not alive, removed ones are invisible) --
// gets the rank's priorities and runs all remaining rounds in one k_tail, its
// tile counters flagging the caller's block columns against the GLOBAL
// per-block-row tile counts.  The rounds are the global rounds (every rank
// runs the same tail redundantly); their statistics go to `out`, the final
// states back into the rank's replicated state.  Takes ownership of
// sub_off / sub_nbr.
int partitioned_tail(tcmis_graph *g, const RoundArgs &ra, int32_t round0, const int32_t *ids,
                     int32_t A, int64_t *sub_off, int32_t *sub_nbr, int64_t E,
                     const int32_t *rowtiles_global, int64_t total_tiles_global,
                     std::vector<DevRound> &out) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  tcmis_graph *sub = nullptr;
  if (int rc = wrap_owned(ctx, A, E, sub_off, sub_nbr, &sub)) return rc;
  struct Guard {
    tcmis_graph *h;
    ~Guard() { tcmis_graph_destroy(h); }
  } guard{sub};
  if (int rc = ensure_workspace(sub)) return rc;
  Workspace &ws = sub->ws;
  Workspace &gw = g->ws;
  const int par = round0 & 1;
  k_sub_init<<<grid_for(ctx, A, 256, 8), 256, 0, st>>>(A, ids, gw.prio, gw.q, ws.prio, ws.q,
                                                       ws.state, ws.next, ws.wl[par]);
  TCMIS_LAUNCHED(ctx);
  Ctrl c0{};
  c0.round = round0;
  c0.wl_count[par] = A;
  c0.alive = A;
  c0.max_rounds = ws.round_cap;
  *ws.h_ctrl = c0;
  TCMIS_CUDA(cudaMemcpyAsync(ws.ctrl, ws.h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
  TCMIS_CUDA(cudaMemsetAsync(ws.rounds, 0, sizeof(DevRound) * ws.round_cap, st));
  if (ra.seg_mode == 1) TCMIS_CUDA(cudaMemsetAsync(gw.segmark, 0, 4ull * ra.nseg, st));
  RoundArgs a;
  std::memset(&a, 0, sizeof(a));
  a.n = A;
  a.off = sub->d_off;
  a.nbr = sub->d_nbr;
  a.vnnz = ((uintptr_t)sub->d_nbr & 15) == 0 ? E : -E;
  a.T = ra.T;
  a.seg_mode = ra.seg_mode;
  a.nseg = ra.nseg;
  a.total_tiles = total_tiles_global;
  a.rowtiles = rowtiles_global;
  a.perm = ids;  // sub id -> caller id: ties, tile columns
  a.tail_grid = tail_grid(ctx);
  TailArgs t = tail_args(sub, a);
  t.segflag = gw.segflag;  // the caller's block columns (rank-sized arrays)
  t.segmark = gw.segmark;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(a.tail_grid);
  lc.blockDim = dim3(kTailBlock);
  lc.dynamicSmemBytes = kTailDynSmem;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  TCMIS_CUDA(cudaLaunchKernelEx(&lc, k_tail, t));
  ctx->launches++;
  k_sub_scatter<<<grid_for(ctx, A, 256, 8), 256, 0, st>>>(A, ids, ws.state, gw.state, gw.q);
  TCMIS_LAUNCHED(ctx);
  TCMIS_CUDA(cudaMemcpyAsync(ws.h_ctrl, ws.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  if (ws.h_ctrl->overflow)
    return set_error(TCMIS_E_RUNTIME, "partitioned tail: more rounds than the statistics ring");
  if (ws.h_ctrl->corrupt)
    return set_error(TCMIS_E_LOGIC, "partitioned tail: a round's counts do not add up");
  const int32_t rr = ws.h_ctrl->round - round0;  // the tail's rounds
  out.resize((size_t)std::max(rr, 0));
  if (rr > 0)
    TCMIS_CUDA(cudaMemcpy(out.data(), ws.rounds + (round0 - 1), sizeof(DevRound) * rr,
                          cudaMemcpyDeviceToHost));
  return 0;
}

int priorities_impl(tcmis_graph *g, int heuristic, uint64_t seed, int scale_bits,
                    uint32_t *p_out) {
  if (heuristic == TCMIS_H1) {
    if (g->n < 1) return set_error(TCMIS_E_INVALID_ARGUMENT, "h1_random requires n >= 1");
  } else if (heuristic == TCMIS_H2 || heuristic == TCMIS_H3 || heuristic == TCMIS_LUBY_PERM) {
    if (scale_bits < 8 || scale_bits > 30)
      return set_error(TCMIS_E_INVALID_ARGUMENT, "scale_bits must be in [8, 30]");
    if (g->n == 0) return 0;
  } else {
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "tiled engine only runs h1/h2/h3; use run_luby_reference");
  }
  uint32_t *d_p = nullptr;
  if (int rc = dev_alloc(&d_p, (size_t)g->n)) return rc;
  int rc = launch_priorities(g, heuristic, seed, scale_bits, d_p, nullptr, nullptr, nullptr);
  if (!rc) {
    cudaError_t e = cudaMemcpyAsync(p_out, d_p, sizeof(uint32_t) * g->n, cudaMemcpyDeviceToHost,
                                    g->ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(g->ctx->stream);
    if (e != cudaSuccess) rc = cuda_error(e, "priorities download");
  }
  dev_free(d_p);
  return rc;
}

int max_np_impl(tcmis_graph *g, const uint32_t *p, const uint8_t *states, uint64_t *out) {
  if (g->n == 0) return 0;
  tcmis_ctx *ctx = g->ctx;
  uint32_t *d_p = nullptr;
  uint8_t *d_s = nullptr;
  uint64_t *d_o = nullptr;
  int rc = dev_alloc(&d_p, g->n);
  if (!rc) rc = dev_alloc(&d_s, g->n);
  if (!rc) rc = dev_alloc(&d_o, g->n);
  if (!rc) {
    cudaMemcpyAsync(d_p, p, 4ull * g->n, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemcpyAsync(d_s, states, g->n, cudaMemcpyHostToDevice, ctx->stream);
    k_max_np<<<grid_for(ctx, 32ll * g->n, 256, 8), 256, 0, ctx->stream>>>(g->n, g->d_off,
                                                                           g->d_nbr, d_p, d_s,
                                                                           d_o);
    ctx->launches++;
    cudaError_t e = cudaMemcpyAsync(out, d_o, 8ull * g->n, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) rc = cuda_error(e, "compute_max_np");
  }
  dev_free(d_p);
  dev_free(d_s);
  dev_free(d_o);
  return rc;
}

int neighbor_count_impl(tcmis_graph *g, const uint8_t *c, int32_t *nc, int T, int64_t *ev,
                        int64_t *sk) {
  if (g->n == 0) {
    if (ev) *ev = 0;
    if (sk) *sk = 0;
    return 0;
  }
  tcmis_ctx *ctx = g->ctx;
  uint8_t *d_c = nullptr;
  int32_t *d_nc = nullptr;
  int rc = dev_alloc(&d_c, g->n);
  if (!rc) rc = dev_alloc(&d_nc, g->n);
  if (!rc) {
    cudaMemcpyAsync(d_c, c, g->n, cudaMemcpyHostToDevice, ctx->stream);
    k_neighbor_count<<<grid_for(ctx, 32ll * g->n, 256, 8), 256, 0, ctx->stream>>>(
        g->n, g->d_off, g->d_nbr, d_c, d_nc);
    ctx->launches++;
    cudaMemcpyAsync(nc, d_nc, 4ull * g->n, cudaMemcpyDeviceToHost, ctx->stream);
    if (T > 0) {  // tile counters of tiled_spmv (spmv.cpp:37-46)
      rc = ensure_workspace(g);
      if (!rc && g->tile_T != T) rc = build_tile_counts(g, T);
      if (!rc) {
        Workspace &ws = g->ws;
        cudaMemsetAsync(ws.segflag, 0, g->tile_nb, ctx->stream);
        k_segflags_from<<<grid_for(ctx, g->n, 256, 8), 256, 0, ctx->stream>>>(g->n, d_c, T,
                                                                               ws.segflag);
        cudaMemsetAsync(&ws.ctrl->eval, 0, 8, ctx->stream);
        k_seg_total<<<grid_for(ctx, g->tile_nb, 256, 4), 256, 0, ctx->stream>>>(
            ws.segflag, g->d_rowtiles, g->tile_nb, ws.ctrl);
        ctx->launches += 2;
        unsigned long long e = 0;
        cudaMemcpyAsync(&e, &ws.ctrl->eval, 8, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemsetAsync(ws.segflag, 0, g->tile_nb, ctx->stream);
        cudaError_t ce = cudaStreamSynchronize(ctx->stream);
        if (ce != cudaSuccess) rc = cuda_error(ce, "tiled_spmv counters");
        *ev = (int64_t)e;
        *sk = g->tile_total - (int64_t)e;
      }
    }
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (!rc && e != cudaSuccess) rc = cuda_error(e, "neighbor count");
  }
  dev_free(d_c);
  dev_free(d_nc);
  return rc;
}

}  // namespace tcmis_b200

#ifdef TCMIS_TAIL_PROF
extern "C" __attribute__((visibility("default"))) int tcmis_debug_tail_prof(
    unsigned long long *out, int cap) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, tcmis_b200::g_tail_prof_n, sizeof(int));
  n = n < cap / 2 ? n : cap / 2;
  cudaMemcpyFromSymbol(out, tcmis_b200::g_tail_prof, sizeof(unsigned long long) * 2 * n);
  int z = 0;
  cudaMemcpyToSymbol(tcmis_b200::g_tail_prof_n, &z, sizeof(int));
  return n;
}
extern "C" __attribute__((visibility("default"))) int tcmis_debug_tail_blk(
    unsigned long long *out) {
  return (int)cudaMemcpyFromSymbol(out, tcmis_b200::g_tail_blk, sizeof(unsigned long long) * 5 * 1024);
}
#endif

namespace tcmis_b200 {

int h1_impl(tcmis_ctx *ctx, int32_t n, uint64_t seed, uint32_t *p_out) {
  if (n < 1) return set_error(TCMIS_E_INVALID_ARGUMENT, "h1_random requires n >= 1");
  uint32_t *d_p = nullptr;
  if (int rc = dev_alloc(&d_p, (size_t)n)) return rc;
  k_h1<<<grid_for(ctx, n, 256, 16), 256, 0, ctx->stream>>>(n, mix64(seed), d_p);
  ctx->launches++;
  cudaError_t e = cudaMemcpyAsync(p_out, d_p, 4ull * n, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  dev_free(d_p);
  if (e != cudaSuccess) return cuda_error(e, "h1_random");
  return 0;
}

// engine.cpp:162-229 run_h3_resolution: the rounds of the engine from the
// given alive set, without statistics.  The selected set is the greedy MIS
// of the alive subgraph in (p, id) order.
int h3_resolution_impl(tcmis_graph *g, const uint32_t *p, const uint8_t *states, uint8_t *c) {
  if (g->n == 0) return 0;
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (int rc = ensure_workspace(g)) return rc;
  Workspace &ws = g->ws;
  uint32_t *d_p = nullptr;
  uint8_t *d_s = nullptr;
  int64_t *d_cnt = nullptr;
  int rc = dev_alloc(&d_p, g->n);
  if (!rc) rc = dev_alloc(&d_s, g->n);
  if (!rc) rc = dev_alloc(&d_cnt, 1);
  int64_t alive = 0;
  if (!rc) {
    cudaMemcpyAsync(d_p, p, 4ull * g->n, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_s, states, g->n, cudaMemcpyHostToDevice, st);
    k_resolve_init<<<grid_for(ctx, g->n, 256, 16), 256, 0, st>>>(g->n, d_p, d_s, ws.prio, ws.q, ws.state,
                                                                ws.next);
    ctx->launches++;
    thrust::counting_iterator<int32_t> ids(0);
    size_t bytes = ws.cub_bytes;
    cudaError_t e = cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, ws.wl[0], d_cnt, (int)g->n,
                                          IsAliveIn{d_s}, st);
    ctx->launches++;
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&alive, d_cnt, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_error(e, "h3 resolution setup");
  }
  if (!rc && alive > 0) {
    // start at "round 2" so the first round reads worklist slot 0
    Ctrl c0{};
    c0.round = 2;
    c0.wl_count[0] = (int32_t)alive;
    c0.alive = (int32_t)alive;
    c0.max_rounds = ws.round_cap;
    *ws.h_ctrl = c0;
    cudaMemcpyAsync(ws.ctrl, ws.h_ctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, st);
    RoundArgs a;
    std::memset(&a, 0, sizeof(a));
    a.n = g->n;
    a.off = g->d_off;
    a.nbr = g->d_nbr;
    a.vnnz = ((uintptr_t)g->d_nbr & 15) == 0 ? g->nnz : -g->nnz;
    a.T = 1;
    a.sel_grid = ctx->num_sms * 8;
    a.upd_grid = ctx->num_sms * 4;
    a.nz = g->d_nz;
    a.nz_count = g->nz_count;
    a.pull = (double)g->max_degree > 64.0 * std::max(1.0, avg_degree(g)) ? 1 : 0;
    for (int round = 0; !rc; ++round) {
      if (round > g->n) {
        rc = set_error(TCMIS_E_LOGIC, "pending set stopped shrinking");  // engine.cpp:224-225
        break;
      }
      rc = launch_select(g, a);
      if (!rc) rc = launch_update(g, a, 0, 0);
      if (rc) break;
      cudaMemcpyAsync(ws.h_ctrl, ws.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st);
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = cuda_error(e, "h3 resolution");
      if (ws.h_ctrl->alive == 0 || ws.h_ctrl->corrupt) break;
    }
  }
  if (!rc && ws.h_ctrl->corrupt)
    rc = set_error(TCMIS_E_LOGIC, "pending set stopped shrinking");  // engine.cpp:224-225
  if (!rc) {
    std::vector<uint8_t> fin(g->n);
    cudaError_t e = cudaMemcpy(fin.data(), ws.state, g->n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_error(e, "h3 resolution result");
    for (int32_t v = 0; v < g->n && !rc; ++v) c[v] = fin[v] == TCMIS_IN_MIS ? 1 : 0;
  }
  dev_free(d_p);
  dev_free(d_s);
  dev_free(d_cnt);
  return rc;
}

}  // namespace tcmis_b200
