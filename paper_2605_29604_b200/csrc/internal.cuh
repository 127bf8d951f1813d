// internal.cuh -- shared types and device helpers of the B200 TC-MIS engine.
//
// Layout in HBM (per graph):
//   d_off   int64[n+1]   CSR row extents (graph.hpp:20)
//   d_nbr   int32[2m]    sorted neighbour ids (graph.hpp:21)
//   prio    uint32[n]    p[v] (PriorityVector::p, priorities.hpp:33); the key of
//                        v is (p[v] << 32) | (v + 1) (priorities.hpp:61-64), built
//                        in registers; a neighbour u is visible iff state[u] is
//                        not Removed (dead keys = kNoNeighborKey, priorities.hpp:57)
//   state   uint8[n]     VertexState (engine.hpp:17)
//   next    uint8[n]     this round's decision: 1 = candidate, 2 = excluded
//   wl[2]   int32[n]     alive worklists (compacted between rounds)
//   segflag uint8[nb]    "block column b holds a candidate this round"
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "tcmis_b200.h"

namespace tcmis_b200 {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;

// priorities.cpp:15-19
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
// priorities.cpp:21-23, with mix64(seed) hoisted by the caller
__host__ __device__ __forceinline__ uint64_t vertex_hash_m(uint64_t v, uint64_t mixed_seed) {
  return mix64(mixed_seed + (v + 1) * kGolden);
}
// priorities.cpp:29-31
__host__ __device__ __forceinline__ uint64_t combine_seed(uint64_t seed, uint64_t round) {
  return mix64(seed + mix64(round + kGolden));
}

__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Per-round statistics as the device accumulates them.
struct DevRound {
  unsigned long long sel, rem, alive, eval, skip;
  // %globaltimer (ns) at the start of Phase 1, Phase 2, Phase 3 and at the
  // round's end, stamped by the round's kernels (the reference's phase
  // timers, engine.cpp:253-284); 0 where a phase has no kernel of its own
  unsigned long long t[4];
};

// Device control block driving the round loop (one per solve workspace).
struct Ctrl {
  int32_t round;       // 1-based round being executed
  int32_t wl_count[2]; // worklist sizes; round r reads slot r&1 (r >= 2)
  int32_t alive;       // alive vertices after the last completed round
  unsigned long long sel, rem, eval;  // accumulators of the running round
  unsigned int ticket; // last-block election in k_update
  int32_t max_rounds;  // capacity of the DevRound array
  int32_t overflow;    // set when rounds exceeded max_rounds
  int32_t long_count;  // entries of the select long-row list this round
  int32_t pull_count;  // entries of the pull long-row list this round
  int32_t main_rounds; // rounds run by the per-round kernels (the rest ran in k_tail)
  int32_t sel_undec;   // rows k_probe_select left to the k_select engine
  int32_t pull_undec;  // rows k_probe_pull left to the k_update_pull engine
  int32_t sel_vlong;   // select rows longer than kBlockRow (block-wide in k_select_long)
  int32_t pull_items;  // chunks of the pull long rows (k_round_end work items)
  int32_t corrupt;     // a round broke selected + removed + alive == alive before
                       // (engine.cpp:138-141,152-153 logic_error): set on the device
  int32_t r1_sel_left;   // round 1, degree order: vertices k_r1_settle left to the probe
  int32_t r1_pull_left;  // ... and that k_r1_pull left to the pull probe
};

// A pull row that outlived k_update_pull's engine (update.cuh): entries
// [lo, hi) are still to be scanned, as chunks first .. first + chunks - 1 of
// the round's item list; `left` counts the chunks not yet finished and `hit`
// is set by any chunk that finds a candidate neighbour.
struct PullRow {
  int64_t lo, hi;
  int32_t v, first;
  int32_t left, hit;
};

// What the whole-solve graph leaves in mapped pinned host memory (k_pack):
// the host reads it after one stream synchronisation, no copies.
struct HostRes {
  Ctrl ctrl;
  long long mis_count;
  DevRound rounds[64];
};

struct DistState;
struct Staging;

struct Workspace {
  size_t n_cap = 0;
  size_t seg_cap = 0;
  uint32_t *prio = nullptr;
  uint16_t *q = nullptr;          // q_of(prio) (common.cuh), 0 once removed
  uint8_t *state = nullptr;
  uint8_t *state_o = nullptr;     // relabeled solves: the final states in the caller's order (on demand)
  uint8_t *mis_o = nullptr;       // relabeled solves: membership in the caller's order (1 = InMIS)
  bool relabeled = false;         // the last solve ran on a relabeled CSR
  uint8_t *next = nullptr;
  uint16_t *xt = nullptr;         // k_tail round tags (tail.cuh), zeroed at allocation
  int32_t *wl[2] = {nullptr, nullptr};
  uint8_t *segflag = nullptr;
  int32_t *mis = nullptr;
  int32_t *long_list = nullptr;   // select: rows that outlived the thread probe
  PullRow *prow = nullptr;        // pull exclusion: rows that outlived the engine
  int32_t *pitems = nullptr;      // ... their chunks (row index per item), for k_round_end
  int64_t prow_cap = 0;
  int32_t *vlong = nullptr;       // select rows beyond kBlockRow (k_select_long, block-wide)
  int64_t vlong_cap = 0;
  int32_t *undec_sel = nullptr;   // probe leftovers for the select engine
  int32_t *undec_pull = nullptr;  // probe leftovers for the pull engine
  uint32_t *segmark = nullptr;    // tail rounds: round that last counted a block column
  unsigned *bar = nullptr;        // grid barrier of k_tail
  unsigned *warpcnt = nullptr;    // k_tail's fused MIS compaction: 2 x kTailMaxWarps per-warp
                                  // counts by solve parity, then tslot[2] (tag base, solve counter)
  int64_t *mis_count = nullptr;
  // relabeled solves without the caller-order plane: the compaction's
  // membership words (32 caller ids each) and per-block counts -> offsets
  uint32_t *gc_bits = nullptr;
  int64_t *gc_blk = nullptr;
  void *gc_tmp = nullptr;
  size_t gc_tmp_bytes = 0;
  Ctrl *ctrl = nullptr;        // device
  Ctrl *h_ctrl = nullptr;      // pinned host mirror
  int64_t *h_misc = nullptr;   // pinned: [0] MIS count, [1] h3 tiles evaluated
  HostRes *h_res = nullptr;    // mapped pinned (cudaHostAllocMapped)
  HostRes *d_res = nullptr;    // its device alias
  DevRound *rounds = nullptr;  // device, capacity round_cap
  DevRound *h_rounds = nullptr;
  int32_t round_cap = 0;
  void *cub_tmp = nullptr;
  size_t cub_bytes = 0;
  cudaGraphExec_t exec = nullptr;  // cached WHILE{select; update} graph
  uint32_t *cbits = nullptr;      // tile exclusion: this round's candidates, bit per vertex
  uint32_t *tile_hit = nullptr;   // tile exclusion: per T=16 block row, rows with a candidate nbr
  uint32_t *alive_bits = nullptr; // tile Phase 1: the round's alive set, bit per vertex
  uint32_t *blocked = nullptr;    // tile Phase 1: per T=16 block row, rows with an alive higher nbr
  alignas(8) unsigned char graph_key[512] = {};
};

}  // namespace tcmis_b200

struct tcmis_ctx {
  // per-kernel device timeline of the last TCMIS_F_TIMING solve (events
  // recorded around every launch on the context stream)
  struct Mark {
    const char *name;
    int32_t round;
    cudaEvent_t a, b;
  };
  bool recording = false;
  int32_t rec_round = 0;
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> event_pool;
  size_t pool_next = 0;
  std::vector<tcmis_kernel_time> timeline;
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int tail_blocks_per_sm = 0;  // co-resident k_tail blocks per SM (occupancy)
  int64_t launches = 0;
  cudaEvent_t ev[8] = {};
  // side stream + events of upload_tiled (K1 counting overlapped with the upload)
  cudaStream_t side = nullptr;
  cudaEvent_t side_ev[9] = {};  // one per upload chunk (8) + the join
  // the largest solve workspace of a destroyed graph, adopted by the next
  // graph that fits (upload -> solve -> destroy loops re-use buffers, pinned
  // staging and the instantiated round graph)
  tcmis_b200::Workspace spare;
  // pinned staging ring + host copy threads for pageable caller memory (staging.cu)
  tcmis_b200::Staging *staging = nullptr;
};

struct tcmis_graph {
  tcmis_ctx *ctx = nullptr;
  int32_t n = 0;
  int64_t nnz = 0;
  int64_t *d_off = nullptr;
  int32_t *d_nbr = nullptr;
  bool owns = false;
  // tiling cache for the tile counters (one tile_dim at a time)
  int32_t tile_T = 0;
  int32_t tile_nb = 0;
  int32_t *d_rowtiles = nullptr;
  int64_t tile_total = 0;
  // compact device tile store (tiles.cu build_tile_store), T = 8 or 16:
  // block-row offsets, one block column and T*T/8 payload bytes per tile
  int32_t store_T = 0;
  int64_t *d_tbro = nullptr;
  int64_t store_tiles = 0;
  int32_t *d_trow = nullptr;
  int32_t *d_tcol = nullptr;
  void *d_tbits = nullptr;
  // per-graph preparation for the solve (computed once)
  bool prepared = false;
  int32_t *d_nz = nullptr;  // ascending ids of non-isolated vertices (round-1 select list)
  int32_t nz_count = 0;
  int64_t max_degree = 0;
  // row partition of a multi-GPU solve (distributed.py): this rank's CSR
  // holds rows [part_lo, part_hi) only; priorities need the full degrees
  int32_t part_lo = 0, part_hi = -1;  // part_hi < 0: not partitioned
  int64_t *d_off_full = nullptr;
  int64_t nnz_global = -1;
  tcmis_b200::DistState *dist = nullptr;  // partitioned-solve state (dist.cu), freed with the graph
  // internal vertex order (order.cu, tcmis_graph_reorder): the solve kernels
  // run on a relabeled copy of the CSR, solve id i = the caller's d_perm[i]
  int32_t order_mode = 0;
  int32_t *d_perm = nullptr;
  int32_t *d_inv = nullptr;   // its inverse: the solve id of the caller's vertex v
  int64_t *d_roff = nullptr;
  int32_t *d_rnbr = nullptr;
  int32_t *d_rnz = nullptr;   // non-isolated solve ids, ascending
  int32_t rnz_count = 0;
  // TCMIS_ORDER_DEGREE: the degree classes (solve ids [cls_start[c],
  // cls_start[c+1]) share one degree, classes in descending degree;
  // cls_start[n_cls] = n) and, per scale_bits, the class bounds of the H2
  // priorities (class_bounds.cu): cb[d] = (lo, hi) for a vertex of degree d
  int32_t *d_cls_start = nullptr;
  int32_t n_cls = 0;
  int2 *d_cb = nullptr;
  int32_t cb_scale_bits = -1;
  int2 *d_cbc = nullptr;       // the same bounds by class index
  int32_t *d_rmax = nullptr;   // per solve id: its largest neighbour id (-1: isolated)
  uint16_t *d_vcls = nullptr;  // per solve id: its degree class (n_cls <= 65535)
  int32_t *d_cls_deg = nullptr;  // per class: its degree
  int32_t *d_spatial = nullptr;  // tcmis_gen_rgg's points in Z-order of their cells
  // Phase 1 tile form (tile_cand.cu): the A-up store of one priority
  // configuration (heuristic, seed, scale_bits)
  int64_t up_key[3] = {-1, -1, -1};
  int64_t up_tiles = 0;
  int32_t *d_up_trow = nullptr;
  int32_t *d_up_tcol = nullptr;
  uint16_t *d_up_tbits = nullptr;
  double up_build_ms = 0;
  tcmis_b200::Workspace ws;
};

namespace tcmis_b200 {

// order.cu: relabeled rows are kept ascending up to this many entries (the
// select / pull scans stop early on them, common.cuh class_bounds)
constexpr int64_t kSortedMax = 4096;
int sort_rows(tcmis_ctx *ctx, int32_t n, const int64_t *off, int32_t *nbr, int which);

// NVTX ranges around the C-ABI calls and the host-driven rounds (header-only
// NVTX3: free unless a profiler such as nsys / ncu attaches)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};
#define TCMIS_RANGE(name) ::tcmis_b200::NvtxRange tcmis_nvtx_range_(name)

// error plumbing (capi.cu)
int set_error(int code, const std::string &msg);
int cuda_error(cudaError_t e, const char *what);

#define TCMIS_CUDA(expr)                                        \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return ::tcmis_b200::cuda_error(_e, #expr); \
  } while (0)

#define TCMIS_LAUNCHED(ctx)                                        \
  do {                                                             \
    (ctx)->launches++;                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return ::tcmis_b200::cuda_error(_e, "kernel launch"); \
  } while (0)

inline int grid_for(const tcmis_ctx *ctx, int64_t work_threads, int block, int per_sm = 8) {
  int64_t want = (work_threads + block - 1) / block;
  int64_t cap = (int64_t)ctx->num_sms * per_sm;
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

// timeline recording (solver.cu): wraps one launch in an event pair when the
// context is recording
cudaEvent_t pool_event(tcmis_ctx *ctx);
#define TCMIS_TIMED(ctx, kname, launch_stmt)                                   \
  do {                                                                        \
    cudaEvent_t _a = nullptr, _b = nullptr;                                   \
    if ((ctx)->recording) {                                                   \
      _a = ::tcmis_b200::pool_event(ctx);                                     \
      _b = ::tcmis_b200::pool_event(ctx);                                     \
      cudaEventRecord(_a, (ctx)->stream);                                     \
    }                                                                         \
    launch_stmt;                                                              \
    if ((ctx)->recording) {                                                   \
      cudaEventRecord(_b, (ctx)->stream);                                     \
      (ctx)->marks.push_back({kname, (ctx)->rec_round, _a, _b});              \
    }                                                                         \
  } while (0)

// the per-round kernel launches (solver.cu), shared with the multi-GPU driver
struct RoundArgs {
  int32_t n;
  const int64_t *off;
  const int32_t *nbr;
  int T, seg_mode, fresh;
  int32_t nseg;
  int64_t total_tiles;
  const int32_t *rowtiles;
  uint64_t seed;
  int sel_grid, upd_grid;
  int pull;             // exclusion form: 0 push (in k_select), 1 pull (in k_update_pull)
  int32_t nz_count;     // round-1 select list
  const int32_t *nz;
  int32_t tail_thr;     // rounds start in k_tail once alive <= tail_thr
  int tail_from1;       // the whole solve in k_tail (small graphs: every non-isolated
                        // vertex fits the tail's block-resident lists)
  int64_t vnnz;         // nnz, negated when the neighbour array is not 16-byte aligned
  uint32_t *pub_cand;   // multi-GPU publish slices (null on one GPU)
  uint32_t *pub_dead;
  int32_t pub_lo;
  int32_t pub_cap;      // sparse publish lists (late rounds of a partitioned solve)
  int32_t *pub_lcand;
  int32_t *pub_ldead;
  int tail_grid;
  int tile;             // tile exclusion over the compact T = 16 store: 0 off, 1 bits, 2 mma
  int32_t nb16;         // block rows of the store
  int64_t store_tiles;
  const int32_t *trow;
  const int32_t *tcol;
  const uint16_t *tbits;
  int tile_cand;        // Phase 1 as A-up tiles x alive bitmap (tile_cand.cu; 2: tcgen05) ...
  int32_t tile_gate;    // ... in the rounds starting with >= tile_gate alive
  int64_t up_tiles;
  const int32_t *up_trow;
  const int32_t *up_tcol;
  const uint16_t *up_tbits;
  const int32_t *perm;  // solve id -> caller id (relabeled CSR), else null
  uint8_t *mis_o;       // relabeled: caller-order membership kept by the kernels, or null
  const int2 *cb;       // degree-class bounds of the H2 priorities (degree order), or null
  const int2 *cbc;      // ... by class index, with r1_max / r1_cls: round 1's settling
  const int32_t *r1_max;  // per vertex: its largest neighbour id
  const uint16_t *r1_cls; // per vertex: its degree class
  int nz_prefix;        // the round-1 list is 0 .. nz_count-1 (degree order)
  bool operator==(const RoundArgs &o) const { return std::memcmp(this, &o, sizeof(*this)) == 0; }
};

int launch_select(tcmis_graph *g, const RoundArgs &a);
int launch_update(tcmis_graph *g, const RoundArgs &a, cudaGraphConditionalHandle cond, int use_cond);
int launch_priorities(tcmis_graph *g, int heuristic, uint64_t seed, int scale_bits,
                      uint32_t *p_out, uint16_t *q_out, uint8_t *state, uint8_t *next,
                      uint8_t *segflag = nullptr, int T = 1, Ctrl *ctrl = nullptr,
                      const Ctrl *ctrl0 = nullptr, DevRound *rounds = nullptr,
                      int32_t nrounds = 0, const int64_t *solve_off = nullptr,
                      const int32_t *perm = nullptr, uint8_t *mis_o = nullptr);
// workspace management (solver.cu)
int ensure_workspace(tcmis_graph *g);
int ensure_cub(tcmis_graph *g, size_t bytes);
void free_workspace(Workspace &ws);

// copies of caller host memory (staging.cu): pinned memory goes straight to
// the copy engine, pageable memory through a pinned ring filled by host threads
int h2d(tcmis_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st);
int d2h(tcmis_ctx *ctx, void *dst, const void *src, size_t bytes, cudaStream_t st);
bool host_pinned(const void *p);  // page-locked / registered / device-accessible
void free_staging(tcmis_ctx *ctx);

// Phase 1 tile form (tile_cand.cu)
int build_up_store(tcmis_graph *g, const uint32_t *p, const int64_t key[3], double *build_ms);
int tile_cand_prepare(tcmis_graph *g, int H, uint64_t seed, int scale_bits, const int64_t key[3],
                      double *build_ms);
void free_up_store(tcmis_graph *g);

// internal vertex order (order.cu)
int reorder_impl(tcmis_graph *g, int32_t mode, const int32_t *order);
// a relabeled solve's final states in the caller's order (ws.state_o), on demand
int states_in_caller_order(tcmis_graph *g);
void free_order(tcmis_graph *g);

// partitioned-solve state (dist.cu)
void free_dist(tcmis_graph *g);
// native partitioned-solve buffers and round graphs (partitioned.cu)
void free_partitioned(tcmis_graph *g);

// tiling (tiles.cu)
int build_tile_counts(tcmis_graph *g, int T);
int wrap_owned(tcmis_ctx *ctx, int32_t n, int64_t nnz, int64_t *d_off, int32_t *d_nbr,
               tcmis_graph **out);
int upload_tiled(tcmis_ctx *ctx, int32_t n, const int64_t *off, const int32_t *nbr, int T,
                 tcmis_graph **out);
int export_tiles(tcmis_graph *g, int T, int32_t *tile_row, int32_t *tile_col,
                 uint64_t *row_bits, int64_t *bro);
int build_tile_store(tcmis_graph *g, int T);
void free_tile_store(tcmis_graph *g);

// Device memory comes from the device's stream-ordered pool (release
// threshold = unlimited, set in tcmis_ctx_create), allocated and freed in
// order on the stream of the context the current C-ABI call runs on
// (t_alloc_stream, set by every entry point).  A graph upload / solve /
// destroy cycle therefore re-uses pool memory instead of paying cudaMalloc
// and the device-wide synchronisation of cudaFree every time.
extern thread_local cudaStream_t t_alloc_stream;

template <typename T>
int dev_alloc(T **p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMallocAsync((void **)p, count * sizeof(T), t_alloc_stream);
  if (e != cudaSuccess) return cuda_error(e, "cudaMallocAsync");
  return 0;
}

inline void dev_free(void *p) {
  if (p) cudaFreeAsync(p, t_alloc_stream);
}

}  // namespace tcmis_b200
