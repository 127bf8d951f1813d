// partitioned.cu -- the row-partitioned multi-GPU solve, driven natively.
//
// rank r owns the contiguous rows [lo_r, hi_r) (edge-balanced,
// boundaries at multiples of 64 and of tile_dim; dist.cu holds the partial
// CSR and the per-rank device side).  tcmis_solve_partitioned runs the whole
// solve of one rank from C++: no Python in the round, one host thread per
// rank.  One round (the reference's bulk-synchronous round,
// engine.cpp:247-291) is
//
//   select own list            -> own candidates published (bitmap slice or id list)
//   all_gather                 -> remote candidates marked (next = 1, InMIS)
//   pull exclusion + update    -> own removals published
//   all_gather                 -> remote removals applied (Removed, q = 0)
//   all_reduce of the counters -> (sel, rem, alive, eval, skip, overflow) of the round
//   k_ring                     -> the reduced counters into mapped host memory
//
// all stream-ordered on the context stream.  With a capturable exchange
// (NCCL) a round is ONE CUDA graph launch; the host keeps one round in flight
// ahead of the counters it reads (the termination test lags one round, the
// stream never drains between rounds; the extra round after the last runs on
// empty lists).  Every rank sees the same reduced counters, so every rank
// takes the same decisions and enqueues the same collectives.
//
// Exchange format: the first rounds publish n/32-word bitmap slices.  Once the
// all-reduced alive count of round k-1 (known when round k+1 is enqueued)
// bounds round k+1's decisions below the dense slice size, the ranks publish
// id lists of that capacity (a power of two) instead: R-MAT s26's late rounds
// move a few KB per rank instead of 8.4 MB / world, and the apply kernels
// touch only the listed vertices.
//
// Exchanges: NCCL (libnccl.so.2 bound at run time, the process's loaded copy
// first, so a comm created by torch's NCCL can be passed in), or an in-process
// group (one host thread per rank, copies through UVA / NVLink peer access;
// also what the single-GPU test box uses to run 2-4 ranks on one device).
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <thrust/iterator/counting_iterator.h>
#include <nccl.h>  // types only: the library is bound with dlopen

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.cuh"

#define TCMIS_API extern "C" __attribute__((visibility("default")))

namespace tcmis_b200 {

int solve_prepare(tcmis_graph *g, const tcmis_config *cfg, RoundArgs &a, int64_t own_isolated);
int tail_grid(tcmis_ctx *ctx);
constexpr int64_t kTailBlockPart = 1024;  // k_tail's per-block list capacity (tail.cuh kTailBlock)
int seg_total(tcmis_graph *g, int64_t *ev);
int partitioned_tail(tcmis_graph *g, const RoundArgs &ra, int32_t round0, const int32_t *ids,
                     int32_t A, int64_t *sub_off, int32_t *sub_nbr, int64_t E,
                     const int32_t *rowtiles_global, int64_t total_tiles_global,
                     std::vector<DevRound> &out);

// ------------------------------------------------------------------ NCCL

namespace {

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int *) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int *) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                            ncclComm_t, cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {std::getenv("TCMIS_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char *nm : names)  // a copy the process already loaded (torch's) first
      if (nm && !api.h) api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
    for (const char *nm : names)
      if (nm && !api.h) api.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    if (!api.h) {
      api.error = "libnccl.so.2 not found (set TCMIS_NCCL_LIB)";
      return;
    }
#define TCMIS_NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
    TCMIS_NCCL_SYM(GetUniqueId);
    TCMIS_NCCL_SYM(CommInitRank);
    TCMIS_NCCL_SYM(CommDestroy);
    TCMIS_NCCL_SYM(CommCount);
    TCMIS_NCCL_SYM(CommUserRank);
    TCMIS_NCCL_SYM(AllGather);
    TCMIS_NCCL_SYM(AllReduce);
    TCMIS_NCCL_SYM(GetErrorString);
#undef TCMIS_NCCL_SYM
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllGather ||
        !api.AllReduce || !api.CommCount || !api.CommUserRank)
      api.error = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

int nccl_error(ncclResult_t r, const char *what) {
  NcclApi &A = nccl();
  return set_error(TCMIS_E_RUNTIME, std::string("NCCL error in ") + what + ": " +
                                        (A.GetErrorString ? A.GetErrorString(r) : "?"));
}

// an in-process group: world ranks, one host thread each
struct LocalGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<const void *> send;
  std::vector<cudaEvent_t> ready, done;
  std::vector<int> device;
  bool peer_ok = true;  // x_peer_setup's vote
  int peer_votes = 0;
  bool aborted = false;  // a rank failed: its peers leave the barrier with an error
  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) return false;
    const uint64_t g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != g || aborted; });
    }
    return !aborted;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

}  // namespace

}  // namespace tcmis_b200

// The exchange a partitioned solve talks through (one handle per rank).
struct tcmis_exchange {
  // a process-unique id: the per-graph buffers and captured round graphs are
  // keyed on it (a pointer could be re-used by the next exchange object, and
  // a cache hit on some ranks but not on others would desynchronise their
  // collectives)
  uint64_t uid = next_uid();
  static uint64_t next_uid() {
    static std::atomic<uint64_t> c{1};
    return c.fetch_add(1);
  }
  int kind = 0;  // 1 NCCL, 2 in-process group
  int32_t world = 1, rank = 0;
  bool capturable = false;
  // NCCL
  ncclComm_t comm = nullptr;
  bool owns_comm = false;
  // in-process group
  std::shared_ptr<tcmis_b200::LocalGroup> group;
  int64_t *scratch = nullptr;  // all-reduce staging, world x 8 (device of the rank)
  int scratch_dev = -1;
  int peer = -1;  // in-process group: apply kernels read the peers' buffers directly (1)
                  // or through all-gather copies (0); -1 = not yet decided
};

namespace tcmis_b200 {
namespace {

__global__ void k_sum_i64(const int64_t *__restrict__ parts, int32_t world, int32_t count,
                          int64_t *__restrict__ out) {
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    int64_t s = 0;
    for (int r = 0; r < world; ++r) s += parts[(size_t)r * count + i];
    out[i] = s;
  }
}

int x_all_gather(tcmis_exchange *x, const void *send, void *recv, size_t bytes, cudaStream_t st) {
  if (x->kind == 1) {
    ncclResult_t r = nccl().AllGather(send, recv, bytes, ncclUint8, x->comm, st);
    return r == ncclSuccess ? 0 : nccl_error(r, "ncclAllGather");
  }
  LocalGroup &G = *x->group;
  const int me = x->rank;
  G.send[me] = send;
  TCMIS_CUDA(cudaEventRecord(G.ready[me], st));
  if (!G.barrier()) return set_error(TCMIS_E_RUNTIME, "a peer rank of the in-process group failed");
  for (int q = 0; q < G.world; ++q) {
    TCMIS_CUDA(cudaStreamWaitEvent(st, G.ready[q], 0));
    const cudaError_t e = cudaMemcpyAsync(static_cast<char *>(recv) + (size_t)q * bytes,
                                          G.send[q], bytes, cudaMemcpyDefault, st);
    if (e != cudaSuccess) {
      G.abort();
      return set_error(TCMIS_E_CUDA, std::string("in-process all-gather (rank ") +
                                         std::to_string(me) + " <- " + std::to_string(q) +
                                         ", " + std::to_string(bytes) + " bytes): " +
                                         cudaGetErrorString(e));
    }
  }
  TCMIS_CUDA(cudaEventRecord(G.done[me], st));
  // every rank enqueued its copies: the send buffers may be reused after done[]
  if (!G.barrier()) return set_error(TCMIS_E_RUNTIME, "a peer rank of the in-process group failed");
  for (int q = 0; q < G.world; ++q) TCMIS_CUDA(cudaStreamWaitEvent(st, G.done[q], 0));
  return 0;
}

// ---- the fused exchange of an in-process group: no all-gather copies; the
// apply kernels read every rank's published buffer straight from its memory
// (same device, or a peer over NVLink with peer access enabled)
struct PeerSlices {
  const void *p[8];
};
constexpr int kPeerMax = 8;

// decided once per exchange, identically on every rank (after a barrier all
// ranks see every rank's device): peer mode iff every pair of devices can
// access each other (peer access is enabled here) and world <= kPeerMax
int x_peer_setup(tcmis_exchange *x, int device) {
  if (x->peer >= 0) return 0;
  LocalGroup &G = *x->group;
  {
    std::lock_guard<std::mutex> lk(G.mu);
    if (G.device.size() != (size_t)G.world) G.device.assign(G.world, -1);
    G.device[x->rank] = device;
  }
  if (!G.barrier()) return set_error(TCMIS_E_RUNTIME, "a peer rank of the in-process group failed");
  bool ok = G.world <= kPeerMax && std::getenv("TCMIS_PART_NO_PEER") == nullptr;
  for (int q = 0; q < G.world && ok; ++q) {
    const int d = G.device[q];
    if (d == device) continue;
    int can = 0;
    cudaDeviceCanAccessPeer(&can, device, d);
    if (!can) {
      ok = false;
      break;
    }
    const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ok = false;
    cudaGetLastError();
  }
  // every rank must take the same decision: AND over the ranks
  static_assert(sizeof(int) == 4, "");
  {
    std::lock_guard<std::mutex> lk(G.mu);
    G.peer_ok = (G.peer_votes++ == 0 ? ok : (G.peer_ok && ok));
  }
  if (!G.barrier()) return set_error(TCMIS_E_RUNTIME, "a peer rank of the in-process group failed");
  x->peer = G.peer_ok ? 1 : 0;
  return 0;
}

// publish `mine`; when this returns, the stream waits for every rank's
// buffer to be complete, and `out` holds all of them
int x_share(tcmis_exchange *x, const void *mine, cudaStream_t st, PeerSlices &out) {
  LocalGroup &G = *x->group;
  const int me = x->rank;
  G.send[me] = mine;
  TCMIS_CUDA(cudaEventRecord(G.ready[me], st));
  if (!G.barrier()) return set_error(TCMIS_E_RUNTIME, "a peer rank of the in-process group failed");
  for (int q = 0; q < G.world; ++q) {
    TCMIS_CUDA(cudaStreamWaitEvent(st, G.ready[q], 0));
    out.p[q] = G.send[q];
  }
  return 0;
}

// every rank has finished reading every rank's buffer (before any is reused)
int x_release(tcmis_exchange *x, cudaStream_t st) {
  LocalGroup &G = *x->group;
  TCMIS_CUDA(cudaEventRecord(G.done[x->rank], st));
  if (!G.barrier()) return set_error(TCMIS_E_RUNTIME, "a peer rank of the in-process group failed");
  for (int q = 0; q < G.world; ++q) TCMIS_CUDA(cudaStreamWaitEvent(st, G.done[q], 0));
  return 0;
}

int x_all_reduce(tcmis_exchange *x, int64_t *buf, int32_t count, cudaStream_t st) {
  if (x->kind == 1) {
    ncclResult_t r = nccl().AllReduce(buf, buf, (size_t)count, ncclInt64, ncclSum, x->comm, st);
    return r == ncclSuccess ? 0 : nccl_error(r, "ncclAllReduce");
  }
  if (count > 8) return set_error(TCMIS_E_LOGIC, "in-process all-reduce holds at most 8 values");
  int dev = 0;
  TCMIS_CUDA(cudaGetDevice(&dev));
  if (!x->scratch || x->scratch_dev != dev) {
    if (x->scratch) cudaFree(x->scratch);
    x->scratch = nullptr;
    TCMIS_CUDA(cudaMalloc(&x->scratch, sizeof(int64_t) * 8 * (x->world + 1)));
    x->scratch_dev = dev;
  }
  int64_t *mine = x->scratch + 8 * x->world;  // the send copy: `buf` is overwritten by the sum
  TCMIS_CUDA(cudaMemcpyAsync(mine, buf, sizeof(int64_t) * count, cudaMemcpyDeviceToDevice, st));
  if (int rc = x_all_gather(x, mine, x->scratch, sizeof(int64_t) * count, st)) return rc;
  k_sum_i64<<<1, 32, 0, st>>>(x->scratch, x->world, count, buf);
  TCMIS_CUDA(cudaGetLastError());
  return 0;
}

// ------------------------------------------------------------- kernels

// remote decisions from gathered id lists: rank r's list sits at r * stride
// (count, then ids)
__global__ void k_apply_list(const int32_t *__restrict__ gathered, int32_t world, int32_t stride,
                             int32_t me, int what, uint8_t *__restrict__ next,
                             uint8_t *__restrict__ state, uint16_t *__restrict__ q) {
  const int64_t total = (int64_t)world * (stride - 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(i / (stride - 1));
    const int32_t k = (int32_t)(i - (int64_t)r * (stride - 1));
    if (r == me) continue;
    const int32_t *lst = gathered + (int64_t)r * stride;
    if (k >= min(__ldg(lst), stride - 1)) continue;
    const int32_t v = __ldg(lst + 1 + k);
    if (what == 0) {
      next[v] = 1;
      state[v] = TCMIS_IN_MIS;
    } else {
      state[v] = TCMIS_REMOVED;
      q[v] = 0;
    }
  }
}

// remote decisions from gathered bitmap slices (rank r's slice at word r *
// maxw, bit v - lo_r): zero words cost one coalesced load
__global__ void k_apply_words(const uint32_t *__restrict__ gathered,
                              const int32_t *__restrict__ rank_lo, int32_t world, int32_t maxw,
                              int32_t me, int what, uint8_t *__restrict__ next,
                              uint8_t *__restrict__ state, uint16_t *__restrict__ q) {
  const int64_t total = (int64_t)world * maxw;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t bits = __ldg(&gathered[w]);
    if (!bits) continue;
    const int32_t r = (int32_t)(w / maxw);
    if (r == me) continue;
    const int64_t first = rank_lo[r] + (w - (int64_t)r * maxw) * 32;
    const int64_t end = rank_lo[r + 1];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t v = first + b;
      if (v >= end) break;
      if (what == 0) {
        next[v] = 1;
        state[v] = TCMIS_IN_MIS;
      } else {
        state[v] = TCMIS_REMOVED;
        q[v] = 0;
      }
    }
  }
}

// the same two applies reading the publishing ranks' buffers directly
__global__ void k_apply_words_peer(PeerSlices sl, const int32_t *__restrict__ rank_lo,
                                   int32_t world, int32_t maxw, int32_t me, int what,
                                   uint8_t *__restrict__ next, uint8_t *__restrict__ state,
                                   uint16_t *__restrict__ q) {
  const int64_t total = (int64_t)world * maxw;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < total;
       w += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(w / maxw);
    if (r == me) continue;
    const int64_t k = w - (int64_t)r * maxw;
    uint32_t bits = static_cast<const uint32_t *>(sl.p[r])[k];
    if (!bits) continue;
    const int64_t first = rank_lo[r] + k * 32, end = rank_lo[r + 1];
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      const int64_t v = first + b;
      if (v >= end) break;
      if (what == 0) {
        next[v] = 1;
        state[v] = TCMIS_IN_MIS;
      } else {
        state[v] = TCMIS_REMOVED;
        q[v] = 0;
      }
    }
  }
}

__global__ void k_apply_list_peer(PeerSlices sl, int32_t world, int32_t cap, int32_t me,
                                  int what, uint8_t *__restrict__ next,
                                  uint8_t *__restrict__ state, uint16_t *__restrict__ q) {
  const int64_t total = (int64_t)world * cap;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(i / cap);
    if (r == me) continue;
    const int32_t k = (int32_t)(i - (int64_t)r * cap);
    const int32_t *lst = static_cast<const int32_t *>(sl.p[r]);
    if (k >= min(lst[0], cap)) continue;
    const int32_t v = lst[1 + k];
    if (what == 0) {
      next[v] = 1;
      state[v] = TCMIS_IN_MIS;
    } else {
      state[v] = TCMIS_REMOVED;
      q[v] = 0;
    }
  }
}

// the finished round's own counters (DevRound, first 5 x u64) + the sparse
// overflow flag into the all-reduce buffer
__global__ void k_stage_counts(const Ctrl *__restrict__ ctrl, const DevRound *__restrict__ rounds,
                               const int32_t *lcand, const int32_t *ldead, int32_t cap,
                               int64_t *__restrict__ buf) {
  if (threadIdx.x != 0) return;
  const int r = ctrl->round - 1;  // round_end_tail advanced ctrl->round
  const DevRound &d = rounds[(r - 1) % ctrl->max_rounds];
  buf[0] = (int64_t)d.sel;
  buf[1] = (int64_t)d.rem;
  buf[2] = (int64_t)d.alive;
  buf[3] = (int64_t)d.eval;
  buf[4] = (int64_t)d.skip;
  buf[5] = (lcand && *lcand > cap ? 1 : 0) + (ldead && *ldead > cap ? 1 : 0);
}

struct InMIS {
  const uint8_t *s;
  __device__ __forceinline__ bool operator()(int32_t v) const { return s[v] == TCMIS_IN_MIS; }
};

struct RingEntry {
  int64_t round;
  int64_t v[6];
};
constexpr int kRing = 8;

__global__ void k_ring(const int64_t *__restrict__ buf, const Ctrl *__restrict__ ctrl,
                       RingEntry *ring) {
  if (threadIdx.x != 0) return;
  const int r = ctrl->round - 1;
  RingEntry *e = &ring[r % kRing];
  for (int i = 0; i < 6; ++i) e->v[i] = buf[i];
  __threadfence_system();
  *(volatile int64_t *)&e->round = r;
  __threadfence_system();
}

// ---- the tail: the alive subgraph gathered on every rank (partitioned_tail)

struct IsAliveV {
  const uint8_t *s;
  __device__ __forceinline__ bool operator()(int32_t v) const { return s[v] == TCMIS_ALIVE; }
};

// warp per own alive row: its alive neighbours counted (kFill false) or
// written in row order (kFill true)
template <bool kFill>
__global__ void k_alive_rows(int32_t A, const int32_t *__restrict__ ids,
                             const int64_t *__restrict__ off, const int32_t *__restrict__ nbr,
                             const uint8_t *__restrict__ state, int32_t *__restrict__ deg,
                             const int64_t *__restrict__ doff, int32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < A;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int32_t v = ids[i];
    const int64_t s0 = off[v], e0 = off[v + 1];
    int64_t base = kFill ? doff[i] : 0;
    int32_t cnt = 0;
    for (int64_t k0 = s0; k0 < e0; k0 += 32) {
      const int64_t k = k0 + lane;
      const int32_t u = k < e0 ? __ldg(&nbr[k]) : -1;
      const bool keep = u >= 0 && state[u] == TCMIS_ALIVE;
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (kFill && keep) out[base + __popc(m & ((1u << lane) - 1u))] = u;
      base += __popc(m);
      cnt += __popc(m);
    }
    if (!kFill && lane == 0) deg[i] = cnt;
  }
}

__global__ void k_widen(int32_t A, const int32_t *__restrict__ d32, int64_t *__restrict__ d64) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= A;
       i += (int64_t)gridDim.x * blockDim.x)
    d64[i] = i < A ? d32[i] : 0;
}

// rank r's padded slices -> the concatenation (rank order = ascending ids)
__global__ void k_concat(int32_t world, int64_t stride, const int32_t *__restrict__ gathered,
                         const int64_t *__restrict__ pref, int32_t *__restrict__ out) {
  for (int r = 0; r < world; ++r) {
    const int64_t cnt = pref[r + 1] - pref[r];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x)
      out[pref[r] + i] = gathered[(int64_t)r * stride + i];
  }
}

// global ids -> positions in the ascending alive list
__global__ void k_to_sub(int64_t E, int32_t *__restrict__ nbr, const int32_t *__restrict__ ids,
                         int32_t A) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = nbr[k];
    int32_t lo = 0, hi = A;
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (__ldg(&ids[mid]) < u) lo = mid + 1;
      else hi = mid;
    }
    nbr[k] = lo;
  }
}

__global__ void k_sum_slices(int32_t world, int64_t nb, const int32_t *__restrict__ gathered,
                             int32_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t t = 0;
    for (int r = 0; r < world; ++r) t += gathered[(int64_t)r * nb + i];
    out[i] = t;
  }
}

// per-rank buffers of a partitioned solve, kept on the graph's DistState
struct PartBufs {
  int32_t maxw = 0, world = 0;
  uint32_t *mine = nullptr, *gathered = nullptr;  // dense slices
  int32_t cap = 0;                                  // sparse capacity the lists hold
  int32_t *lcand = nullptr, *ldead = nullptr, *lgathered = nullptr;
  int64_t *counts = nullptr;  // all-reduce buffer (8)
  int32_t *d_rank_lo = nullptr;
  RingEntry *h_ring = nullptr, *d_ring = nullptr;
  std::map<int32_t, cudaGraphExec_t> graphs;  // per publish capacity (0 = dense)
  int32_t *rowtiles_global = nullptr;         // the tail's tile counts of every block row
  int64_t total_tiles_global = -1;
  std::vector<unsigned char> key;             // what the graphs were captured for
};

void free_bufs(PartBufs &b) {
  dev_free(b.mine);
  dev_free(b.gathered);
  dev_free(b.lcand);
  dev_free(b.ldead);
  dev_free(b.lgathered);
  dev_free(b.counts);
  dev_free(b.d_rank_lo);
  dev_free(b.rowtiles_global);
  if (b.h_ring) cudaFreeHost(b.h_ring);
  for (auto &kv : b.graphs) cudaGraphExecDestroy(kv.second);
  b = PartBufs{};
}

std::map<const tcmis_graph *, PartBufs> &bufs_of() {
  static auto *m = new std::map<const tcmis_graph *, PartBufs>();
  return *m;
}
std::mutex &bufs_mu() {
  static std::mutex mu;
  return mu;
}

// host-side profile of the last partitioned solve of a graph
struct PartProfile {
  int32_t rounds = 0, sparse_rounds = 0, tail_rounds = 0;
  double enqueue_us = 0, wait_us = 0, rounds_us = 0;
};
std::map<const tcmis_graph *, PartProfile> &profiles() {
  static auto *m = new std::map<const tcmis_graph *, PartProfile>();
  return *m;
}

}  // namespace

void free_partitioned(tcmis_graph *g) {
  {
    std::lock_guard<std::mutex> lk(bufs_mu());
    profiles().erase(g);
  }
  std::lock_guard<std::mutex> lk(bufs_mu());
  auto it = bufs_of().find(g);
  if (it == bufs_of().end()) return;
  free_bufs(it->second);
  bufs_of().erase(it);
}

namespace {

// Enqueue one round on the context stream.  cap == 0: bitmap slices.
int enqueue_round(tcmis_graph *g, tcmis_exchange *x, RoundArgs &a, PartBufs &b, int32_t cap) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  Workspace &ws = g->ws;
  const int world = x->world, me = x->rank;
  const int agrid = grid_for(ctx, cap ? (int64_t)world * cap : (int64_t)world * b.maxw, 256, 4);
  a.pub_cap = cap;
  // 1. select + candidate exchange
  if (cap) {
    TCMIS_CUDA(cudaMemsetAsync(b.lcand, 0, sizeof(int32_t), st));
    a.pub_cand = nullptr;
    a.pub_lcand = b.lcand;
  } else {
    TCMIS_CUDA(cudaMemsetAsync(b.mine, 0, 4ull * b.maxw, st));
    a.pub_cand = b.mine;
    a.pub_lcand = nullptr;
  }
  a.pub_dead = nullptr;
  a.pub_ldead = nullptr;
  if (int rc = launch_select(g, a)) return rc;
  const bool peer = x->kind == 2 && x->peer == 1;
  if (peer) {  // fused: the apply reads the ranks' candidate buffers in place
    PeerSlices sl{};
    if (int rc = x_share(x, cap ? (const void *)b.lcand : (const void *)b.mine, st, sl)) return rc;
    if (cap)
      k_apply_list_peer<<<agrid, 256, 0, st>>>(sl, world, cap, me, 0, ws.next, ws.state, ws.q);
    else
      k_apply_words_peer<<<agrid, 256, 0, st>>>(sl, b.d_rank_lo, world, b.maxw, me, 0, ws.next,
                                                 ws.state, ws.q);
    if (int rc = x_release(x, st)) return rc;
  } else if (cap) {
    if (int rc = x_all_gather(x, b.lcand, b.lgathered, 4ull * (cap + 1), st)) return rc;
    k_apply_list<<<agrid, 256, 0, st>>>(b.lgathered, world, cap + 1, me, 0, ws.next, ws.state,
                                         ws.q);
  } else {
    if (int rc = x_all_gather(x, b.mine, b.gathered, 4ull * b.maxw, st)) return rc;
    k_apply_words<<<agrid, 256, 0, st>>>(b.gathered, b.d_rank_lo, world, b.maxw, me, 0, ws.next,
                                          ws.state, ws.q);
  }
  TCMIS_LAUNCHED(ctx);
  // 2. exclusion + update + removal exchange
  a.pub_lcand = nullptr;
  a.pub_cand = nullptr;
  if (cap) {
    TCMIS_CUDA(cudaMemsetAsync(b.ldead, 0, sizeof(int32_t), st));
    a.pub_ldead = b.ldead;
  } else {
    TCMIS_CUDA(cudaMemsetAsync(b.mine, 0, 4ull * b.maxw, st));
    a.pub_dead = b.mine;
  }
  if (int rc = launch_update(g, a, 0, 0)) return rc;
  if (peer) {
    PeerSlices sl{};
    if (int rc = x_share(x, cap ? (const void *)b.ldead : (const void *)b.mine, st, sl)) return rc;
    if (cap)
      k_apply_list_peer<<<agrid, 256, 0, st>>>(sl, world, cap, me, 1, ws.next, ws.state, ws.q);
    else
      k_apply_words_peer<<<agrid, 256, 0, st>>>(sl, b.d_rank_lo, world, b.maxw, me, 1, ws.next,
                                                 ws.state, ws.q);
    if (int rc = x_release(x, st)) return rc;
  } else if (cap) {
    if (int rc = x_all_gather(x, b.ldead, b.lgathered, 4ull * (cap + 1), st)) return rc;
    k_apply_list<<<agrid, 256, 0, st>>>(b.lgathered, world, cap + 1, me, 1, ws.next, ws.state,
                                         ws.q);
  } else {
    if (int rc = x_all_gather(x, b.mine, b.gathered, 4ull * b.maxw, st)) return rc;
    k_apply_words<<<agrid, 256, 0, st>>>(b.gathered, b.d_rank_lo, world, b.maxw, me, 1, ws.next,
                                          ws.state, ws.q);
  }
  TCMIS_LAUNCHED(ctx);
  // 3. the round's counters: all-reduced, then into the host ring
  k_stage_counts<<<1, 32, 0, st>>>(ws.ctrl, ws.rounds, cap ? b.lcand : nullptr,
                                   cap ? b.ldead : nullptr, cap, b.counts);
  TCMIS_LAUNCHED(ctx);
  if (int rc = x_all_reduce(x, b.counts, 6, st)) return rc;
  k_ring<<<1, 32, 0, st>>>(b.counts, ws.ctrl, b.d_ring);
  TCMIS_LAUNCHED(ctx);
  return 0;
}

constexpr int kKernelsPerRoundExtra = 4;  // apply x2, stage, ring

int launch_round(tcmis_graph *g, tcmis_exchange *x, RoundArgs &a, PartBufs &b, int32_t cap) {
  TCMIS_RANGE(cap ? "partitioned round (id lists)" : "partitioned round (bitmaps)");
  tcmis_ctx *ctx = g->ctx;
  if (!x->capturable) return enqueue_round(g, x, a, b, cap);
  auto it = b.graphs.find(cap);
  if (it == b.graphs.end()) {
    const int64_t launches0 = ctx->launches;
    cudaGraph_t graph = nullptr;
    TCMIS_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeRelaxed));
    int rc = enqueue_round(g, x, a, b, cap);
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    ctx->launches = launches0;
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (e != cudaSuccess) return cuda_error(e, "partitioned round capture");
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return cuda_error(e, "partitioned round instantiate");
    it = b.graphs.emplace(cap, exec).first;
  }
  TCMIS_CUDA(cudaGraphLaunch(it->second, ctx->stream));
  ctx->launches += (a.pull ? 6 : 4) + kKernelsPerRoundExtra;
  return 0;
}

// The late rounds on one device per rank: every rank gathers the alive
// subgraph (each rank contributes its own alive rows, restricted to alive
// neighbours: two all-gathers of padded slices after one of the counts) and
// runs the same k_tail on it (solver.cu partitioned_tail).  round0 is the
// first round the tail runs.
int run_tail(tcmis_graph *g, tcmis_exchange *x, const RoundArgs &a, PartBufs &b,
             int32_t round0, std::vector<DevRound> &tail_rounds) {
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  Workspace &ws = g->ws;
  const int world = x->world;
  const int32_t lo = g->part_lo, own = g->part_hi - g->part_lo;
  // tile counts of every block row and the global tile total (cached)
  if (a.seg_mode == 1 && !b.rowtiles_global) {
    const int64_t nb = g->tile_nb;
    int32_t *gath = nullptr;
    if (int rc = dev_alloc(&gath, (size_t)nb * world + 1)) return rc;
    if (int rc = dev_alloc(&b.rowtiles_global, (size_t)nb + 1)) return rc;
    if (int rc = x_all_gather(x, g->d_rowtiles, gath, 4ull * nb, st)) return rc;
    k_sum_slices<<<grid_for(ctx, nb, 256, 8), 256, 0, st>>>(world, nb, gath, b.rowtiles_global);
    TCMIS_LAUNCHED(ctx);
    TCMIS_CUDA(cudaMemcpyAsync(b.counts, &g->tile_total, 8, cudaMemcpyHostToDevice, st));
    if (int rc = x_all_reduce(x, b.counts, 1, st)) return rc;
    TCMIS_CUDA(cudaMemcpyAsync(&b.total_tiles_global, b.counts, 8, cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    dev_free(gath);
  }
  // own alive rows, restricted to alive neighbours
  int32_t *own_ids = nullptr, *own_deg = nullptr, *own_nbr = nullptr;
  int64_t *own_off = nullptr, *d_cnt = nullptr;
  struct Frees {
    std::vector<void *> p;
    ~Frees() {
      for (void *q : p) dev_free(q);
    }
  } frees;
  if (int rc = dev_alloc(&own_ids, (size_t)own + 1)) return rc;
  frees.p.push_back(own_ids);
  if (int rc = dev_alloc(&d_cnt, 2)) return rc;
  frees.p.push_back(d_cnt);
  {
    thrust::counting_iterator<int32_t> it(lo);
    size_t bytes = ws.cub_bytes;
    TCMIS_CUDA(cub::DeviceSelect::If(ws.cub_tmp, bytes, it, own_ids, d_cnt, (int)own,
                                     IsAliveV{ws.state}, st));
    ctx->launches++;
  }
  int64_t h_a = 0;
  TCMIS_CUDA(cudaMemcpyAsync(&h_a, d_cnt, 8, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  const int32_t a_r = (int32_t)h_a;
  if (int rc = dev_alloc(&own_deg, (size_t)a_r + 1)) return rc;
  frees.p.push_back(own_deg);
  if (int rc = dev_alloc(&own_off, (size_t)a_r + 1)) return rc;
  frees.p.push_back(own_off);
  k_alive_rows<false><<<grid_for(ctx, 32ll * std::max(a_r, 1), 256, 8), 256, 0, st>>>(
      a_r, own_ids, g->d_off, g->d_nbr, ws.state, own_deg, nullptr, nullptr);
  TCMIS_LAUNCHED(ctx);
  k_widen<<<grid_for(ctx, (int64_t)a_r + 1, 256, 8), 256, 0, st>>>(a_r, own_deg, own_off);
  TCMIS_LAUNCHED(ctx);
  {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, own_off, own_off, (int64_t)a_r + 1, st);
    void *tmp = nullptr;
    if (int rc = dev_alloc((char **)&tmp, bytes)) return rc;
    TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, own_off, own_off, (int64_t)a_r + 1, st));
    ctx->launches++;
    dev_free(tmp);
  }
  // counts of every rank (int64 pairs)
  int64_t *cnts = nullptr;
  if (int rc = dev_alloc(&cnts, 2ull * world + 2)) return rc;
  frees.p.push_back(cnts);
  TCMIS_CUDA(cudaMemcpyAsync(d_cnt + 1, own_off + a_r, 8, cudaMemcpyDeviceToDevice, st));
  if (int rc = x_all_gather(x, d_cnt, cnts, 16, st)) return rc;
  std::vector<int64_t> h_cnts(2 * (size_t)world);
  TCMIS_CUDA(cudaMemcpyAsync(h_cnts.data(), cnts, 16ull * world, cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> pa(world + 1, 0), pe(world + 1, 0);
  int64_t maxa = 1, maxe = 1;
  for (int r = 0; r < world; ++r) {
    pa[r + 1] = pa[r] + h_cnts[2 * r];
    pe[r + 1] = pe[r] + h_cnts[2 * r + 1];
    maxa = std::max(maxa, h_cnts[2 * r]);
    maxe = std::max(maxe, h_cnts[2 * r + 1]);
  }
  const int32_t A = (int32_t)pa[world];
  const int64_t E = pe[world];
  const int64_t e_r = h_cnts[2 * x->rank + 1];
  if (int rc = dev_alloc(&own_nbr, (size_t)maxe)) return rc;
  frees.p.push_back(own_nbr);
  k_alive_rows<true><<<grid_for(ctx, 32ll * std::max(a_r, 1), 256, 8), 256, 0, st>>>(
      a_r, own_ids, g->d_off, g->d_nbr, ws.state, nullptr, own_off, own_nbr);
  TCMIS_LAUNCHED(ctx);
  (void)e_r;
  // padded all-gathers of ids, degrees, neighbour lists
  int32_t *send = nullptr, *g_ids = nullptr, *g_deg = nullptr, *g_nbr = nullptr;
  if (int rc = dev_alloc(&send, (size_t)maxa)) return rc;
  frees.p.push_back(send);
  if (int rc = dev_alloc(&g_ids, (size_t)maxa * world)) return rc;
  frees.p.push_back(g_ids);
  if (int rc = dev_alloc(&g_deg, (size_t)maxa * world)) return rc;
  frees.p.push_back(g_deg);
  if (int rc = dev_alloc(&g_nbr, (size_t)maxe * world)) return rc;
  frees.p.push_back(g_nbr);
  if (a_r) TCMIS_CUDA(cudaMemcpyAsync(send, own_ids, 4ull * a_r, cudaMemcpyDeviceToDevice, st));
  if (int rc = x_all_gather(x, send, g_ids, 4ull * maxa, st)) return rc;
  if (a_r) TCMIS_CUDA(cudaMemcpyAsync(send, own_deg, 4ull * a_r, cudaMemcpyDeviceToDevice, st));
  if (int rc = x_all_gather(x, send, g_deg, 4ull * maxa, st)) return rc;
  if (int rc = x_all_gather(x, own_nbr, g_nbr, 4ull * maxe, st)) return rc;
  // the subgraph: ids ascending (rank order), offsets, neighbours as sub ids
  int64_t *d_pref = nullptr;
  if (int rc = dev_alloc(&d_pref, 2ull * (world + 1))) return rc;
  frees.p.push_back(d_pref);
  TCMIS_CUDA(cudaMemcpyAsync(d_pref, pa.data(), 8ull * (world + 1), cudaMemcpyHostToDevice, st));
  TCMIS_CUDA(cudaMemcpyAsync(d_pref + world + 1, pe.data(), 8ull * (world + 1),
                             cudaMemcpyHostToDevice, st));
  int32_t *sub_ids = nullptr, *sub_deg = nullptr, *sub_nbr = nullptr;
  int64_t *sub_off = nullptr;
  if (int rc = dev_alloc(&sub_ids, (size_t)A + 1)) return rc;
  frees.p.push_back(sub_ids);
  if (int rc = dev_alloc(&sub_deg, (size_t)A + 1)) return rc;
  frees.p.push_back(sub_deg);
  if (int rc = dev_alloc(&sub_off, (size_t)A + 1)) return rc;  // owned by the subgraph
  if (int rc = dev_alloc(&sub_nbr, (size_t)std::max<int64_t>(E, 1))) {
    dev_free(sub_off);
    return rc;
  }
  k_concat<<<grid_for(ctx, maxa, 256, 8), 256, 0, st>>>(world, maxa, g_ids, d_pref, sub_ids);
  k_concat<<<grid_for(ctx, maxa, 256, 8), 256, 0, st>>>(world, maxa, g_deg, d_pref, sub_deg);
  k_concat<<<grid_for(ctx, maxe, 256, 8), 256, 0, st>>>(world, maxe, g_nbr, d_pref + world + 1,
                                                       sub_nbr);
  k_widen<<<grid_for(ctx, (int64_t)A + 1, 256, 8), 256, 0, st>>>(A, sub_deg, sub_off);
  k_to_sub<<<grid_for(ctx, std::max<int64_t>(E, 1), 256, 8), 256, 0, st>>>(E, sub_nbr, sub_ids, A);
  ctx->launches += 5;
  {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, sub_off, sub_off, (int64_t)A + 1, st);
    void *tmp = nullptr;
    if (int rc = dev_alloc((char **)&tmp, bytes)) return rc;
    TCMIS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, sub_off, sub_off, (int64_t)A + 1, st));
    ctx->launches++;
    dev_free(tmp);
  }
  TCMIS_CUDA(cudaGetLastError());
  return partitioned_tail(g, a, round0, sub_ids, A, sub_off, sub_nbr, E,
                          a.seg_mode == 1 ? b.rowtiles_global : g->d_rowtiles,
                          a.seg_mode == 1 ? b.total_tiles_global : g->tile_total, tail_rounds);
}

int32_t pow2_at_least(int64_t x) {
  int64_t c = 256;
  while (c < x) c <<= 1;
  return (int32_t)std::min<int64_t>(c, INT32_MAX / 2);
}

}  // namespace

int solve_partitioned_impl(tcmis_graph *g, tcmis_exchange *x, const int32_t *rank_lo,
                           int32_t world, const tcmis_config *cfg, uint8_t *state_out,
                           int32_t *mis_out, int64_t *mis_count, tcmis_iter_stats *stats,
                           int32_t max_stats, int32_t *n_iter) {
  if (g->part_hi < 0) return set_error(TCMIS_E_INVALID_ARGUMENT, "graph is not a row partition");
  if (world != x->world) return set_error(TCMIS_E_INVALID_ARGUMENT, "world differs from the exchange's");
  const int32_t n = g->n, me = x->rank;
  if (rank_lo[0] != 0 || rank_lo[world] != n)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "rank_lo must start at 0 and end at n");
  const int T = cfg->tile_dim;
  for (int r = 0; r < world; ++r) {
    if (rank_lo[r + 1] < rank_lo[r])
      return set_error(TCMIS_E_INVALID_ARGUMENT, "rank_lo must be non-decreasing");
    if (rank_lo[r] != n && ((rank_lo[r] % 64) || (T > 0 && rank_lo[r] % T)))
      return set_error(TCMIS_E_INVALID_ARGUMENT,
                       "partition boundaries must be multiples of 64 and of tile_dim");
  }
  if (rank_lo[me] != g->part_lo || rank_lo[me + 1] != g->part_hi)
    return set_error(TCMIS_E_INVALID_ARGUMENT, "rank_lo disagrees with this rank's rows");
  if (cfg->heuristic == TCMIS_LUBY_FRESH)
    return set_error(TCMIS_E_INVALID_ARGUMENT,
                     "luby-fresh redraws every alive key per round; the partitioned solve runs "
                     "the fixed-priority heuristics (h1, h2, h3, luby-perm)");
  *n_iter = 0;
  if (mis_count) *mis_count = 0;
  if (n == 0) return 0;
  tcmis_ctx *ctx = g->ctx;
  cudaStream_t st = ctx->stream;
  if (int rc = ensure_workspace(g)) return rc;
  RoundArgs a;
  const int64_t own = (int64_t)g->part_hi - g->part_lo;
  if (int rc = solve_prepare(g, cfg, a, own - g->nz_count)) return rc;
  a.pull = 1;  // a push would have to reach remote rows
  a.tail_thr = 0;
  a.pub_lo = g->part_lo;
  Workspace &ws = g->ws;

  std::unique_lock<std::mutex> lk(bufs_mu());
  PartBufs &b = bufs_of()[g];
  lk.unlock();
  int32_t maxw = 1;
  for (int r = 0; r < world; ++r) maxw = std::max(maxw, (rank_lo[r + 1] - rank_lo[r] + 31) / 32);
  // buffers and graphs are per (layout, round arguments, exchange)
  std::vector<unsigned char> key(sizeof(RoundArgs) + sizeof(uint64_t) + 4 * (world + 1));
  std::memcpy(key.data(), &a, sizeof(a));
  std::memcpy(key.data() + sizeof(a), &x->uid, sizeof(uint64_t));
  std::memcpy(key.data() + sizeof(a) + sizeof(uint64_t), rank_lo, 4 * (world + 1));
  if (b.key != key) {
    free_bufs(b);
    b.key = key;
    b.maxw = maxw;
    b.world = world;
    if (int rc = dev_alloc(&b.mine, (size_t)maxw)) return rc;
    if (int rc = dev_alloc(&b.gathered, (size_t)maxw * world)) return rc;
    if (int rc = dev_alloc(&b.counts, 8)) return rc;
    if (int rc = dev_alloc(&b.d_rank_lo, (size_t)world + 1)) return rc;
    TCMIS_CUDA(cudaMemcpyAsync(b.d_rank_lo, rank_lo, 4ull * (world + 1), cudaMemcpyHostToDevice,
                               st));
    TCMIS_CUDA(cudaHostAlloc((void **)&b.h_ring, sizeof(RingEntry) * kRing, cudaHostAllocMapped));
    TCMIS_CUDA(cudaHostGetDevicePointer((void **)&b.d_ring, b.h_ring, 0));
    // the largest list capacity that is still smaller than a dense slice
    int32_t cap = maxw > 512 ? pow2_at_least(maxw / 2) : 0;
    if (const char *env = std::getenv("TCMIS_PART_CAP")) cap = std::atoi(env);  // test hook
    if (cap > 0 && (cap < maxw - 1 || std::getenv("TCMIS_PART_CAP"))) {
      b.cap = cap;
      if (int rc = dev_alloc(&b.lcand, (size_t)cap + 1)) return rc;
      if (int rc = dev_alloc(&b.ldead, (size_t)cap + 1)) return rc;
      if (int rc = dev_alloc(&b.lgathered, (size_t)(cap + 1) * world)) return rc;
    }
  }
  for (int i = 0; i < kRing; ++i) b.h_ring[i].round = -1;
  TCMIS_CUDA(cudaStreamSynchronize(st));

  const int32_t cap_rounds = n;  // engine.cpp:248-249
  std::vector<RingEntry> got;
  int64_t alive_prev[2] = {n, n};  // reduced alive after rounds k-1, k-2 (n before round 1)
  auto choose = [&](int64_t bound) -> int32_t {
    if (!b.cap || bound > b.cap) return 0;
    return std::min(b.cap, pow2_at_least(bound));
  };
  auto wait_ring = [&](int r, RingEntry &out) -> int {
    volatile RingEntry *e = &b.h_ring[r % kRing];
    for (int spin = 0;; ++spin) {
      if (e->round == r) break;
      if ((spin & 1023) == 1023) {
        cudaError_t q = cudaStreamQuery(st);
        if (q != cudaSuccess && q != cudaErrorNotReady) return cuda_error(q, "partitioned round");
        if (e->round == r) break;
        std::this_thread::yield();
      }
    }
    out.round = r;
    for (int i = 0; i < 6; ++i) out.v[i] = e->v[i];
    return 0;
  };
  // round k+1 is enqueued before round k's counters are read; its decisions
  // are bounded by the alive count after round k-1
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  double enqueue_us = 0, wait_us = 0;
  int32_t sparse_rounds = 0;
  auto timed_launch = [&](int32_t cap) -> int {
    const auto t0 = clk::now();
    const int rc = launch_round(g, x, a, b, cap);
    enqueue_us += std::chrono::duration<double, std::micro>(clk::now() - t0).count();
    return rc;
  };
  // the late rounds on one device per rank (run_tail) once the alive count
  // fits k_tail: round it+1 is not enqueued when the alive count after round
  // it-1 (a bound of the one after round it) is that small.  Off by default:
  // gathering the subgraph costs ~0.3 ms of host round trips and
  // allocations, measured on one device (s22 1.17 -> 1.41 ms, s26 8.9 ->
  // 9.2 ms at world 1), which 2-3 late exchange rounds do not cost; it pays
  // for graphs with many late rounds on many GPUs.  TCMIS_PART_TAIL = the
  // alive threshold (capped at k_tail's capacity).
  int64_t tail_thr = 0;
  if (const char *env = std::getenv("TCMIS_PART_TAIL")) tail_thr = std::atoll(env);
  tail_thr = std::min<int64_t>(tail_thr, (int64_t)tail_grid(ctx) * kTailBlockPart);
  std::vector<DevRound> tail_rounds;
  int32_t tail_from = 0;  // first round run by the tail (0: none)
  if (int rc = timed_launch(0)) return rc;
  bool done = false;
  int32_t rounds_run = 0;
  for (int32_t it = 1; !done; ++it) {
    if (it > cap_rounds)
      return set_error(TCMIS_E_RUNTIME, "iteration cap exceeded; engine livelock");
    const bool to_tail = tail_thr > 0 && it >= 2 && alive_prev[0] <= tail_thr;
    if (it < cap_rounds && !to_tail) {
      const int32_t c = choose(alive_prev[0]);
      sparse_rounds += c ? 1 : 0;
      if (int rc = timed_launch(c)) return rc;
    }
    RingEntry e;
    const auto tw = clk::now();
    if (int rc = wait_ring(it, e)) return rc;
    wait_us += std::chrono::duration<double, std::micro>(clk::now() - tw).count();
    if (e.v[5]) return set_error(TCMIS_E_LOGIC, "exchange list overflow (a round decided more "
                                                 "vertices than the alive bound)");
    if (e.v[0] == 0 && e.v[2] > 0)  // the largest alive key is always a candidate
      return set_error(TCMIS_E_LOGIC, "a round selected nothing while vertices are alive");
    got.push_back(e);
    alive_prev[1] = alive_prev[0];
    alive_prev[0] = e.v[2];
    rounds_run = it;
    done = e.v[2] == 0;
    if (!done && to_tail) {
      TCMIS_CUDA(cudaStreamSynchronize(st));
      if (int rc = run_tail(g, x, a, b, it + 1, tail_rounds)) return rc;
      tail_from = it + 1;
      for (const DevRound &d : tail_rounds) {
        RingEntry t{};
        t.round = ++rounds_run;
        t.v[0] = (int64_t)d.sel;
        t.v[1] = (int64_t)d.rem;
        t.v[2] = (int64_t)d.alive;
        t.v[3] = (int64_t)d.eval;
        t.v[4] = (int64_t)d.skip;
        got.push_back(t);
      }
      done = true;
    }
  }
  TCMIS_CUDA(cudaStreamSynchronize(st));  // the extra (empty) round too

  const auto t_rounds = clk::now();
  {
    std::lock_guard<std::mutex> lk2(bufs_mu());
    PartProfile &pf = profiles()[g];
    pf.rounds = rounds_run;
    pf.enqueue_us = enqueue_us;
    pf.wait_us = wait_us;
    pf.rounds_us = std::chrono::duration<double, std::micro>(t_rounds - t_start).count();
    pf.sparse_rounds = sparse_rounds;
    pf.tail_rounds = (int32_t)tail_rounds.size();
  }
  // every rank now holds the final state of all n vertices (own decisions +
  // the applied remote ones): the ascending MIS from one compaction -- of all
  // n, or with TCMIS_F_OWN_RANGE of the own rows only (a distributed result)
  const bool own_only = (cfg->flags & TCMIS_F_OWN_RANGE) != 0;
  const int32_t out_lo = own_only ? g->part_lo : 0, out_hi = own_only ? g->part_hi : n;
  int64_t h_cnt = 0, global_cnt = 0;
  for (const RingEntry &e : got) global_cnt += e.v[0];
  if (mis_out || mis_count) {
    thrust::counting_iterator<int32_t> ids(out_lo);
    size_t bytes = ws.cub_bytes;
    TCMIS_CUDA(cub::DeviceSelect::If(ws.cub_tmp, bytes, ids, ws.mis, ws.mis_count,
                                     (int)(out_hi - out_lo), InMIS{ws.state}, st));
    ctx->launches++;
    TCMIS_CUDA(cudaMemcpyAsync(&h_cnt, ws.mis_count, 8, cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
  }
  if (mis_count) *mis_count = h_cnt;
  if (mis_out && h_cnt)
    TCMIS_CUDA(cudaMemcpyAsync(mis_out, ws.mis, 4ull * h_cnt, cudaMemcpyDeviceToHost, st));
  if (state_out && out_hi > out_lo)
    TCMIS_CUDA(cudaMemcpyAsync(state_out, ws.state + out_lo, (size_t)(out_hi - out_lo),
                               cudaMemcpyDeviceToHost, st));
  // this rank's phase stamps (the reference's timers, engine.cpp:253-284)
  const int32_t own_rounds = tail_from ? tail_from - 1 : rounds_run;
  std::vector<DevRound> stamps((size_t)std::min(own_rounds, ws.round_cap));
  if (!stamps.empty())
    TCMIS_CUDA(cudaMemcpyAsync(stamps.data(), ws.rounds, sizeof(DevRound) * stamps.size(),
                               cudaMemcpyDeviceToHost, st));
  TCMIS_CUDA(cudaStreamSynchronize(st));
  stamps.insert(stamps.end(), tail_rounds.begin(), tail_rounds.end());  // the tail's stamps
  auto span_ms = [](unsigned long long a0, unsigned long long a1) {
    return (a0 && a1 && a1 > a0) ? (double)(a1 - a0) * 1e-6 : 0.0;
  };
  const int H = cfg->heuristic;
  if (H == TCMIS_H3) {
    // engine.cpp:255-258: one collapsed iteration; tiles of the block columns
    // holding any MIS vertex, summed over the ranks
    int64_t ev = 0;
    if (int rc = seg_total(g, &ev)) return rc;
    TCMIS_CUDA(cudaMemcpyAsync(b.counts, &ev, 8, cudaMemcpyHostToDevice, st));
    TCMIS_CUDA(cudaMemcpyAsync(b.counts + 1, &g->tile_total, 8, cudaMemcpyHostToDevice, st));
    if (int rc = x_all_reduce(x, b.counts, 2, st)) return rc;
    int64_t red[2] = {0, 0};
    TCMIS_CUDA(cudaMemcpyAsync(red, b.counts, 16, cudaMemcpyDeviceToHost, st));
    TCMIS_CUDA(cudaStreamSynchronize(st));
    if (stats && max_stats > 0) {
      tcmis_iter_stats s{};
      s.iteration = 1;
      s.candidates_selected = global_cnt;
      s.vertices_removed = n - global_cnt;
      s.alive_remaining = 0;
      s.tiles_evaluated = red[0];
      s.tiles_skipped = red[1] - red[0];
      for (const DevRound &d : stamps) {
        const unsigned long long p2 = d.t[1] ? d.t[1] : d.t[2];
        s.phase1_ms += span_ms(d.t[0], p2 ? p2 : d.t[3]);
        s.phase2_ms += span_ms(d.t[1], d.t[2]);
        s.phase3_ms += span_ms(d.t[2], d.t[3]);
      }
      stats[0] = s;
    }
    *n_iter = 1;
    return 0;
  }
  for (int32_t r = 0; r < rounds_run && stats && r < max_stats; ++r) {
    tcmis_iter_stats s{};
    s.iteration = r + 1;
    s.candidates_selected = got[r].v[0];
    s.vertices_removed = got[r].v[1];
    s.alive_remaining = got[r].v[2];
    s.tiles_evaluated = got[r].v[3];
    s.tiles_skipped = got[r].v[4];
    if (r < (int32_t)stamps.size()) {
      const DevRound &d = stamps[r];
      const unsigned long long p2 = d.t[1] ? d.t[1] : d.t[2];
      s.phase1_ms = span_ms(d.t[0], p2 ? p2 : d.t[3]);
      s.phase2_ms = span_ms(d.t[1], d.t[2]);
      s.phase3_ms = span_ms(d.t[2], d.t[3]);
    }
    stats[r] = s;
  }
  *n_iter = rounds_run;
  return 0;
}

}  // namespace tcmis_b200

using namespace tcmis_b200;

#define NEED(cond, msg) \
  if (!(cond)) return set_error(TCMIS_E_INVALID_ARGUMENT, msg)

TCMIS_API int tcmis_nccl_unique_id(uint8_t id[128]) {
  NEED(id, "null buffer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  NcclApi &A = nccl();
  if (!A.error.empty()) return set_error(TCMIS_E_RUNTIME, A.error);
  ncclUniqueId u;
  ncclResult_t r = A.GetUniqueId(&u);
  if (r != ncclSuccess) return nccl_error(r, "ncclGetUniqueId");
  std::memcpy(id, &u, 128);
  return 0;
}

TCMIS_API int tcmis_exchange_nccl(tcmis_ctx *ctx, int32_t world, int32_t rank, const uint8_t id[128],
                                  tcmis_exchange **out) {
  NEED(ctx && id && out, "null handle");
  NEED(world >= 1 && rank >= 0 && rank < world, "bad rank / world");
  NcclApi &A = nccl();
  if (!A.error.empty()) return set_error(TCMIS_E_RUNTIME, A.error);
  TCMIS_CUDA(cudaSetDevice(ctx->device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t comm = nullptr;
  ncclResult_t r = A.CommInitRank(&comm, world, u, rank);
  if (r != ncclSuccess) return nccl_error(r, "ncclCommInitRank");
  auto *x = new tcmis_exchange();
  x->kind = 1;
  x->world = world;
  x->rank = rank;
  x->capturable = std::getenv("TCMIS_PART_NO_GRAPH") == nullptr;
  x->comm = comm;
  x->owns_comm = true;
  *out = x;
  return 0;
}

TCMIS_API int tcmis_exchange_nccl_comm(void *nccl_comm, tcmis_exchange **out) {
  NEED(nccl_comm && out, "null handle");
  NcclApi &A = nccl();
  if (!A.error.empty()) return set_error(TCMIS_E_RUNTIME, A.error);
  int world = 0, rank = 0;
  ncclResult_t r = A.CommCount(static_cast<ncclComm_t>(nccl_comm), &world);
  if (r == ncclSuccess) r = A.CommUserRank(static_cast<ncclComm_t>(nccl_comm), &rank);
  if (r != ncclSuccess) return nccl_error(r, "ncclCommCount / ncclCommUserRank");
  auto *x = new tcmis_exchange();
  x->kind = 1;
  x->world = world;
  x->rank = rank;
  x->capturable = std::getenv("TCMIS_PART_NO_GRAPH") == nullptr;
  x->comm = static_cast<ncclComm_t>(nccl_comm);
  x->owns_comm = false;
  *out = x;
  return 0;
}

TCMIS_API int tcmis_exchange_local_group(int32_t world, tcmis_exchange **out) {
  NEED(out && world >= 1, "bad arguments");
  auto G = std::make_shared<LocalGroup>();
  G->world = world;
  G->send.assign(world, nullptr);
  G->ready.assign(world, nullptr);
  G->done.assign(world, nullptr);
  for (int r = 0; r < world; ++r) {
    TCMIS_CUDA(cudaEventCreateWithFlags(&G->ready[r], cudaEventDisableTiming));
    TCMIS_CUDA(cudaEventCreateWithFlags(&G->done[r], cudaEventDisableTiming));
  }
  for (int r = 0; r < world; ++r) {
    auto *x = new tcmis_exchange();
    x->kind = 2;
    x->world = world;
    x->rank = r;
    x->capturable = false;  // cross-thread events cannot be captured
    x->group = G;
    out[r] = x;
  }
  return 0;
}

TCMIS_API void tcmis_exchange_destroy(tcmis_exchange *x) {
  if (!x) return;
  if (x->kind == 1 && x->owns_comm && x->comm) nccl().CommDestroy(x->comm);
  if (x->scratch) cudaFree(x->scratch);
  if (x->group && x->group.use_count() == 1) {
    for (cudaEvent_t e : x->group->ready) cudaEventDestroy(e);
    for (cudaEvent_t e : x->group->done) cudaEventDestroy(e);
  }
  delete x;
}

TCMIS_API void tcmis_exchange_abort(tcmis_exchange *x) {
  if (x && x->kind == 2) x->group->abort();
}

TCMIS_API int32_t tcmis_exchange_world(const tcmis_exchange *x) { return x ? x->world : 0; }
TCMIS_API int32_t tcmis_exchange_rank(const tcmis_exchange *x) { return x ? x->rank : -1; }

TCMIS_API int tcmis_solve_partitioned(tcmis_graph *part, tcmis_exchange *x, const int32_t *rank_lo,
                                      int32_t world, const tcmis_config *cfg, uint8_t *state_out,
                                      int32_t *mis_out, int64_t *mis_count,
                                      tcmis_iter_stats *stats, int32_t max_stats,
                                      int32_t *n_iterations) {
  NEED(part && x && rank_lo && cfg && n_iterations, "null handle");
  NEED(world >= 1, "bad world");
  TCMIS_RANGE("tcmis_solve_partitioned");
  TCMIS_CUDA(cudaSetDevice(part->ctx->device));
  t_alloc_stream = part->ctx->stream;
  if (x->kind == 2 && x->peer < 0) {
    if (int rc = x_peer_setup(x, part->ctx->device)) {
      x->group->abort();
      return rc;
    }
  }
  const int rc = solve_partitioned_impl(part, x, rank_lo, world, cfg, state_out, mis_out,
                                        mis_count, stats, max_stats, n_iterations);
  if (rc && x->kind == 2) x->group->abort();  // do not leave the peers in the barrier
  return rc;
}

TCMIS_API int tcmis_partitioned_profile(const tcmis_graph *part, double out[6]) {
  NEED(part && out, "null handle");
  std::lock_guard<std::mutex> lk(bufs_mu());
  auto it = profiles().find(part);
  if (it == profiles().end()) return set_error(TCMIS_E_INVALID_ARGUMENT, "no partitioned solve yet");
  out[0] = it->second.rounds;
  out[1] = it->second.enqueue_us;
  out[2] = it->second.wait_us;
  out[3] = it->second.rounds_us;
  out[4] = it->second.sparse_rounds;
  out[5] = it->second.tail_rounds;
  return 0;
}
