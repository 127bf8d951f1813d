// engine.cpp -- the C++ drop-in API (include/tcmis/tcmis.hpp) over the C-ABI.
//
// Each call that touches the graph uploads it to the device of a process-wide
// context, runs the sm_100a kernels through tcmis_b200.h and maps the status
// codes back onto the reference's exception types (SURVEY 8(b) "Errors").
#include <algorithm>
#include <numeric>
#include <cmath>
#include <memory>
#include <cstdlib>
#include <mutex>
#include <bit>
#include <istream>
#include <ostream>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <thread>

#include "tcmis/tcmis.hpp"
#include "tcmis_b200.h"

namespace tcmis {
inline namespace b200 {

namespace {

[[noreturn]] void raise(int code) {
  const std::string msg = tcmis_last_error();
  switch (code) {
    case TCMIS_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case TCMIS_E_LOGIC: throw std::logic_error(msg);
    case TCMIS_E_OUT_OF_RANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error(msg);
  }
}

void check(int code) {
  if (code != TCMIS_OK) raise(code);
}

// Device contexts of the drop-in calls.  A context (one stream, one spare
// workspace, the cached round graph) is not re-entrant, while the reference's
// free functions may run concurrently on different graphs; so every call
// leases a context of its own for its whole duration from a process-wide
// pool (created on first use, returned when the call ends, never destroyed:
// the CUDA runtime may already be gone at exit).  One thread at a time re-uses
// the same warm context.
class ContextLease {
 public:
  ContextLease() {
    {
      std::lock_guard<std::mutex> lk(mu());
      if (!pool().empty()) {
        ctx_ = pool().back();
        pool().pop_back();
        return;
      }
    }
    check(tcmis_ctx_create(0, &ctx_));
  }
  ~ContextLease() {
    std::lock_guard<std::mutex> lk(mu());
    pool().push_back(ctx_);
  }
  ContextLease(const ContextLease &) = delete;
  ContextLease &operator=(const ContextLease &) = delete;
  tcmis_ctx *get() const { return ctx_; }

 private:
  static std::mutex &mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<tcmis_ctx *> &pool() {
    static auto *p = new std::vector<tcmis_ctx *>();
    return *p;
  }
  tcmis_ctx *ctx_ = nullptr;
};

// A graph uploaded for one call, on a context leased for that call (the
// lease is declared first, so it outlives the graph).
struct DeviceGraph {
  ContextLease lease;
  tcmis_graph *h = nullptr;
  explicit DeviceGraph(const Graph &g) {
    check(tcmis_graph_upload(lease.get(), g.n, g.offsets.empty() ? nullptr : g.offsets.data(),
                             g.neighbors.empty() ? nullptr : g.neighbors.data(), &h));
  }
  // upload with the K1 tile count of tile_dim overlapped (tcmis_graph_upload_tiled)
  DeviceGraph(const Graph &g, int tile_dim) {
    check(tcmis_graph_upload_tiled(lease.get(), g.n,
                                   g.offsets.empty() ? nullptr : g.offsets.data(),
                                   g.neighbors.empty() ? nullptr : g.neighbors.data(), tile_dim,
                                   &h, nullptr));
  }
  ~DeviceGraph() { tcmis_graph_destroy(h); }
  DeviceGraph(const DeviceGraph &) = delete;
  DeviceGraph &operator=(const DeviceGraph &) = delete;
};

void check_tile_dim(int T) {  // tiling.cpp:17-21
  if (T < 1 || T > 64)
    throw std::invalid_argument("tile_dim must be in [1, 64], got " + std::to_string(T));
}

struct ObserverBridge {
  const EngineConfig *cfg;
  static void call(void *user, int32_t it, const uint8_t *c, const uint8_t *st, int32_t n) {
    auto *self = static_cast<ObserverBridge *>(user);
    self->cfg->iteration_observer(
        it, std::span<const std::uint8_t>(c, static_cast<std::size_t>(n)),
        std::span<const VertexState>(reinterpret_cast<const VertexState *>(st),
                                     static_cast<std::size_t>(n)));
  }
};

// The result's id vector, allocated and page-faulted on a helper thread while
// the upload and the solve run on the device (a fresh 16 MB std::vector costs
// ~2 ms of page faults and zero-fill on the calling thread); the ids are then
// copied straight into it (d2h staging of the C-ABI) and the vector is
// shrunk to |MIS| without reallocating.
class ResultIds {
 public:
  explicit ResultIds(VertexId n)
      : th_([this, n] { ids_.resize(static_cast<std::size_t>(std::max<VertexId>(n, 1))); }) {}
  ~ResultIds() {
    if (th_.joinable()) th_.join();
  }
  std::vector<VertexId> &get() {
    if (th_.joinable()) th_.join();
    return ids_;
  }
  ResultIds(const ResultIds &) = delete;
  ResultIds &operator=(const ResultIds &) = delete;

 private:
  std::vector<VertexId> ids_;
  std::thread th_;
};

MISResult solve(tcmis_graph *g, VertexId n, const EngineConfig &cfg, Heuristic h,
                ResultIds *ids = nullptr) {
  tcmis_config c;
  tcmis_config_init(&c);
  c.heuristic = static_cast<int32_t>(h);
  c.tile_dim = cfg.tile_dim;
  c.seed = cfg.seed;
  c.scale_bits = cfg.scale_bits;
  c.workers = cfg.workers;
  ObserverBridge bridge{&cfg};
  if (cfg.iteration_observer) {
    c.observer = &ObserverBridge::call;
    c.observer_user = &bridge;
  }
  MISResult r;
  r.heuristic = h;
  r.seed = cfg.seed;
  std::vector<tcmis_iter_stats> st(4096);
  std::optional<ResultIds> own;
  if (!ids) ids = &own.emplace(n);
  std::vector<VertexId> &mis = ids->get();
  int64_t cnt = 0;
  int32_t nit = 0;
  check(tcmis_solve(g, &c, nullptr, mis.data(), &cnt, st.data(), static_cast<int32_t>(st.size()),
                    &nit));
  if (nit > static_cast<int32_t>(st.size())) {
    // pathological round counts: ask again for all the statistics (the solve
    // is deterministic); the hook already saw every iteration once
    // (engine.cpp:275-278), so the second run goes without it
    st.resize(static_cast<std::size_t>(nit));
    c.observer = nullptr;
    c.observer_user = nullptr;
    check(tcmis_solve(g, &c, nullptr, mis.data(), &cnt, st.data(), nit, &nit));
  }
  mis.resize(static_cast<std::size_t>(cnt));  // shrinks in place
  r.mis = std::move(mis);
  r.iterations.reserve(static_cast<std::size_t>(nit));
  for (int32_t i = 0; i < nit; ++i) {
    IterationStats s;
    s.iteration = st[i].iteration;
    s.candidates_selected = st[i].candidates_selected;
    s.vertices_removed = st[i].vertices_removed;
    s.alive_remaining = st[i].alive_remaining;
    s.tiles_evaluated = st[i].tiles_evaluated;
    s.tiles_skipped = st[i].tiles_skipped;
    s.phase1_ms = st[i].phase1_ms;
    s.phase2_ms = st[i].phase2_ms;
    s.phase3_ms = st[i].phase3_ms;
    r.iterations.push_back(s);
  }
  return r;
}

}  // namespace

// ------------------------------------------------------------------ graph

bool Graph::has_edge(VertexId u, VertexId v) const {
  auto row = neighbors_of(u);
  return std::binary_search(row.begin(), row.end(), v);
}

// graph.cpp:14-41.  Large edge lists are normalised on the device
// (tcmis_graph_from_edges: radix sort + unique) and the CSR comes back; small
// ones stay on the host, where the copies would cost more than the sort.
// TCMIS_FROM_EDGES_DEVICE_MIN (edges; default 2^20) moves the switch (tests).
static Graph graph_from_edges_device(VertexId n,
                                     std::span<const std::pair<VertexId, VertexId>> edges) {
  const std::size_t m = edges.size();
  std::vector<std::int32_t> u(m), v(m);
  for (std::size_t i = 0; i < m; ++i) {
    u[i] = edges[i].first;
    v[i] = edges[i].second;
  }
  ContextLease lease;
  tcmis_graph *h = nullptr;
  check(tcmis_graph_from_edges(lease.get(), n, static_cast<std::int64_t>(m), u.data(), v.data(),
                               &h));
  Graph g;
  g.n = n;
  g.offsets.assign(static_cast<std::size_t>(n) + 1, 0);
  g.neighbors.resize(static_cast<std::size_t>(tcmis_graph_nnz(h)));
  const int rc = tcmis_graph_download(h, g.offsets.data(),
                                      g.neighbors.empty() ? nullptr : g.neighbors.data());
  tcmis_graph_destroy(h);
  check(rc);
  return g;
}

Graph graph_from_edges(VertexId n, std::span<const std::pair<VertexId, VertexId>> edges) {
  if (n < 0) throw std::invalid_argument("vertex count must be non-negative");
  std::size_t device_min = std::size_t(1) << 20;
  if (const char *env = std::getenv("TCMIS_FROM_EDGES_DEVICE_MIN"))
    device_min = static_cast<std::size_t>(std::atoll(env));
  if (edges.size() >= device_min && !edges.empty()) return graph_from_edges_device(n, edges);
  std::vector<std::uint64_t> keys;
  keys.reserve(edges.size() * 2);
  for (const auto &[u, v] : edges) {
    if (u < 0 || u >= n || v < 0 || v >= n)
      throw std::out_of_range("edge endpoint outside [0, n)");
    if (u == v) continue;
    keys.push_back((static_cast<std::uint64_t>(u) << 32) | static_cast<std::uint32_t>(v));
    keys.push_back((static_cast<std::uint64_t>(v) << 32) | static_cast<std::uint32_t>(u));
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  Graph g;
  g.n = n;
  g.offsets.assign(static_cast<std::size_t>(n) + 1, 0);
  g.neighbors.resize(keys.size());
  for (std::size_t i = 0; i < keys.size(); ++i) {
    g.offsets[(keys[i] >> 32) + 1]++;
    g.neighbors[i] = static_cast<VertexId>(static_cast<std::uint32_t>(keys[i]));
  }
  for (VertexId v = 0; v < n; ++v) g.offsets[v + 1] += g.offsets[v];
  return g;
}

// ------------------------------------------------------------- priorities

std::uint64_t mix64(std::uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
std::uint64_t vertex_hash(std::uint64_t v, std::uint64_t seed) {
  return mix64(mix64(seed) + (v + 1) * 0x9e3779b97f4a7c15ULL);
}
double hash_to_unit(std::uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }
std::uint64_t combine_seed(std::uint64_t seed, std::uint64_t round) {
  return mix64(seed + mix64(round + 0x9e3779b97f4a7c15ULL));
}

PriorityVector h1_random(VertexId n, std::uint64_t seed) {
  if (n < 1) throw std::invalid_argument("h1_random requires n >= 1");
  PriorityVector pv;
  pv.seed = seed;
  pv.p.resize(static_cast<std::size_t>(n));
  ContextLease lease;
  check(tcmis_h1_random(lease.get(), n, seed, pv.p.data()));
  return pv;
}

std::uint32_t h2_priority_value(double avg, VertexId degree, double eps, int scale_bits) {
  // priorities.cpp:43-51 (built with -ffp-contract=off: no fused operations)
  double denom = avg + static_cast<double>(degree) - eps;
  if (denom < 1.0 / 1024.0) denom = 1.0 / 1024.0;
  const double scaled = std::floor(avg / denom * std::ldexp(1.0, scale_bits));
  if (scaled < 0.0) return 0u;
  if (scaled >= 4294967295.0) return 0xffffffffu;
  return static_cast<std::uint32_t>(scaled);
}

PriorityVector h2_degree_aware(const Graph &g, std::uint64_t seed, int scale_bits) {
  if (scale_bits < kMinScaleBits || scale_bits > kMaxScaleBits)
    throw std::invalid_argument("scale_bits must be in [8, 30]");
  PriorityVector pv;
  pv.seed = seed;
  pv.p.resize(static_cast<std::size_t>(g.n));
  if (g.n == 0) return pv;
  DeviceGraph dg(g);
  check(tcmis_priorities(dg.h, TCMIS_H2, seed, scale_bits, pv.p.data()));
  return pv;
}

// ----------------------------------------------------------------- tiling

TiledAdjacency tile_graph(const Graph &g, int tile_dim) {
  check_tile_dim(tile_dim);
  TiledAdjacency a;
  a.tile_dim = tile_dim;
  a.n = g.n;
  const std::int32_t nb = static_cast<std::int32_t>((static_cast<std::int64_t>(g.n) + tile_dim - 1) / tile_dim);
  a.n_padded = nb * tile_dim;
  a.block_row_offsets.assign(static_cast<std::size_t>(nb) + 1, 0);
  if (g.n == 0) return a;
  DeviceGraph dg(g);
  int64_t count = 0;
  check(tcmis_graph_tile(dg.h, tile_dim, &count));
  a.tile_row.resize(static_cast<std::size_t>(count));
  a.tile_col.resize(static_cast<std::size_t>(count));
  a.row_bits.resize(static_cast<std::size_t>(count) * tile_dim);
  check(tcmis_graph_export_tiles(dg.h, tile_dim, a.tile_row.data(), a.tile_col.data(),
                                 a.row_bits.data(), a.block_row_offsets.data()));
  return a;
}

// ------------------------------------------------- tile persistence (f3)
// Host-side utilities over the tiles tile_graph() exported from the device:
// the reference's binary cache format (tiling.hpp:80-86), its roundtrip and
// its statistics (tiling.cpp:103-228), restated from the header contract.

Graph tiled_to_csr_roundtrip(const TiledAdjacency &a) {
  std::vector<std::pair<VertexId, VertexId>> edges;
  const int T = a.tile_dim;
  for (std::int64_t t = 0; t < a.tile_count(); ++t) {
    const VertexId r0 = a.tile_row[t] * T, c0 = a.tile_col[t] * T;
    for (int i = 0; i < T; ++i)
      for (std::uint64_t w = a.row_bits[t * T + i]; w; w &= w - 1) {
        const VertexId v = r0 + i, u = c0 + std::countr_zero(w);
        if (v < u) edges.emplace_back(v, u);  // the symmetric copy is the other tile's
      }
  }
  return graph_from_edges(a.n, edges);
}

TileStats tile_stats(const TiledAdjacency &a) {
  TileStats st;
  const int T = a.tile_dim;
  st.tile_count = a.tile_count();
  st.occupancy_histogram.assign(static_cast<std::size_t>(T) * T + 1, 0);
  for (std::int64_t t = 0; t < st.tile_count; ++t) {
    std::int64_t nz = 0;
    for (int i = 0; i < T; ++i) nz += std::popcount(a.row_bits[t * T + i]);
    st.total_nonzeros += nz;
    ++st.occupancy_histogram[static_cast<std::size_t>(nz)];
  }
  const double np = static_cast<double>(a.n_padded);
  st.density = np > 0 ? static_cast<double>(st.tile_count) * T * T / (np * np) : 0.0;
  return st;
}

namespace {
constexpr char kTiledMagic[8] = {'T', 'C', 'M', 'I', 'S', 'T', 'I', 'L'};
constexpr std::uint32_t kTiledVersion = 1;

template <typename U>
void put_le(std::ostream &out, U x) {
  unsigned char b[sizeof(U)];
  for (std::size_t i = 0; i < sizeof(U); ++i) b[i] = static_cast<unsigned char>(x >> (8 * i));
  out.write(reinterpret_cast<const char *>(b), sizeof(U));
}

template <typename U>
U get_le(std::istream &in) {
  unsigned char b[sizeof(U)];
  if (!in.read(reinterpret_cast<char *>(b), sizeof(U)))
    throw std::runtime_error("truncated tiled file");
  U x = 0;
  for (std::size_t i = 0; i < sizeof(U); ++i) x |= static_cast<U>(b[i]) << (8 * i);
  return x;
}
}  // namespace

void write_tiled(std::ostream &out, const TiledAdjacency &a) {
  const int T = a.tile_dim;
  out.write(kTiledMagic, sizeof(kTiledMagic));
  put_le<std::uint32_t>(out, kTiledVersion);
  put_le<std::uint32_t>(out, static_cast<std::uint32_t>(T));
  put_le<std::uint64_t>(out, static_cast<std::uint64_t>(a.n));
  put_le<std::uint64_t>(out, static_cast<std::uint64_t>(a.tile_count()));
  std::vector<unsigned char> pay(static_cast<std::size_t>((T * T + 7) / 8));
  for (std::int64_t t = 0; t < a.tile_count(); ++t) {
    put_le<std::uint32_t>(out, static_cast<std::uint32_t>(a.tile_row[t]));
    put_le<std::uint32_t>(out, static_cast<std::uint32_t>(a.tile_col[t]));
    std::fill(pay.begin(), pay.end(), 0);
    for (int i = 0; i < T; ++i)
      for (std::uint64_t w = a.row_bits[t * T + i]; w; w &= w - 1) {
        const int k = i * T + std::countr_zero(w);
        pay[k >> 3] |= static_cast<unsigned char>(1u << (k & 7));
      }
    out.write(reinterpret_cast<const char *>(pay.data()), static_cast<std::streamsize>(pay.size()));
  }
  if (!out) throw std::runtime_error("failed writing tiled file");
}

TiledAdjacency read_tiled(std::istream &in) {
  char magic[8];
  if (!in.read(magic, sizeof(magic)) || std::memcmp(magic, kTiledMagic, sizeof(magic)) != 0)
    throw std::runtime_error("not a tiled adjacency file");
  if (get_le<std::uint32_t>(in) != kTiledVersion)
    throw std::runtime_error("unsupported tiled file version");
  const int T = static_cast<int>(get_le<std::uint32_t>(in));
  check_tile_dim(T);
  TiledAdjacency a;
  a.tile_dim = T;
  a.n = static_cast<VertexId>(get_le<std::uint64_t>(in));
  const std::uint64_t tiles = get_le<std::uint64_t>(in);
  const std::int32_t nb = static_cast<std::int32_t>((static_cast<std::int64_t>(a.n) + T - 1) / T);
  a.n_padded = nb * T;
  a.block_row_offsets.assign(static_cast<std::size_t>(nb) + 1, 0);
  std::vector<unsigned char> pay(static_cast<std::size_t>((T * T + 7) / 8));
  std::int32_t pr = -1, pc = -1;
  for (std::uint64_t t = 0; t < tiles; ++t) {
    const auto br = static_cast<std::int32_t>(get_le<std::uint32_t>(in));
    const auto bc = static_cast<std::int32_t>(get_le<std::uint32_t>(in));
    if (br < 0 || bc < 0 || br >= nb || bc >= nb)
      throw std::runtime_error("tile coordinates out of range");
    if (br < pr || (br == pr && bc <= pc))
      throw std::runtime_error("tiles not sorted by (block_row, block_col)");
    pr = br;
    pc = bc;
    if (!in.read(reinterpret_cast<char *>(pay.data()), static_cast<std::streamsize>(pay.size())))
      throw std::runtime_error("truncated tiled file");
    a.tile_row.push_back(br);
    a.tile_col.push_back(bc);
    const std::size_t base = a.row_bits.size();
    a.row_bits.resize(base + static_cast<std::size_t>(T), 0);
    for (int k = 0; k < T * T; ++k)
      if ((pay[k >> 3] >> (k & 7)) & 1u) a.row_bits[base + k / T] |= std::uint64_t{1} << (k % T);
    a.block_row_offsets[static_cast<std::size_t>(br) + 1] = static_cast<std::int64_t>(t) + 1;
  }
  for (std::int32_t b = 0; b < nb; ++b)  // block rows without tiles
    a.block_row_offsets[b + 1] = std::max(a.block_row_offsets[b + 1], a.block_row_offsets[b]);
  return a;
}

std::int64_t tiled_bytes_estimate(const TiledAdjacency &a) {
  return 24 + a.tile_count() * (8 + (a.tile_dim * a.tile_dim + 7) / 8);
}

std::int64_t csr_bytes_estimate(const Graph &g) {
  return static_cast<std::int64_t>((static_cast<std::size_t>(g.n) + 1) * sizeof(EdgeIndex) +
                                   g.neighbors.size() * sizeof(VertexId));
}

TiledVector pack_vector(std::span<const std::uint8_t> values, int tile_dim) {
  check_tile_dim(tile_dim);
  TiledVector c;
  c.tile_dim = tile_dim;
  c.n = static_cast<VertexId>(values.size());
  const std::int32_t ns = static_cast<std::int32_t>((static_cast<std::int64_t>(c.n) + tile_dim - 1) / tile_dim);
  c.n_padded = ns * tile_dim;
  c.values.assign(static_cast<std::size_t>(c.n_padded), 0);
  std::copy(values.begin(), values.end(), c.values.begin());
  c.segment_bits.assign(static_cast<std::size_t>(ns), 0);
  for (VertexId k = 0; k < c.n; ++k)
    if (values[k]) c.segment_bits[k / tile_dim] |= std::uint64_t{1} << (k % tile_dim);
  return c;
}

// ------------------------------------------------------------------- spmv

void tile_mma(std::span<const std::uint64_t> rows, std::uint64_t seg, std::span<std::int32_t> out) {
  for (std::size_t i = 0; i < rows.size(); ++i)
    out[i] += static_cast<std::int32_t>(__builtin_popcountll(rows[i] & seg));
}

std::vector<std::int32_t> tiled_spmv(const TiledAdjacency &a, const TiledVector &c,
                                     const SpmvOptions &options, SpmvStats *stats) {
  if (a.tile_dim != c.tile_dim || a.n_padded != c.n_padded || a.n != c.n)
    throw std::invalid_argument("tiled adjacency and vector disagree on tile layout");
  std::vector<std::int32_t> nc(static_cast<std::size_t>(a.n), 0);
  int64_t ev = 0, sk = 0;
  if (a.n > 0) {
    // K4b on the CUDA cores (it beats the tensor-core form at
    // every measured tile density); an all-zero segment contributes nothing,
    // so without skipping every tile merely counts as evaluated
    ContextLease lease;
    check(tcmis_tiled_spmv_tiles(lease.get(), a.n, a.tile_dim, a.tile_count(), a.tile_col.data(),
                                 a.row_bits.data(), a.block_row_offsets.data(),
                                 c.segment_bits.data(), TCMIS_EXCL_TILE_BITS, nc.data(), &ev,
                                 &sk));
    if (!options.skip_empty_segments) {
      ev += sk;
      sk = 0;
    }
  }
  if (stats) {
    stats->tiles_evaluated = ev;
    stats->tiles_skipped = sk;
  }
  return nc;
}

std::vector<std::int32_t> csr_neighbor_count_oracle(const Graph &g,
                                                    std::span<const std::uint8_t> candidates) {
  if (static_cast<VertexId>(candidates.size()) != g.n)
    throw std::invalid_argument("candidate vector length must equal n");
  std::vector<std::int32_t> nc(static_cast<std::size_t>(g.n), 0);
  if (g.n == 0) return nc;
  DeviceGraph dg(g);
  check(tcmis_neighbor_count(dg.h, candidates.data(), nc.data()));
  return nc;
}

// --------------------------------------------------------------- validate

namespace {
struct SetCheck {
  std::int32_t independent = 0, u = 0, v = 0, maximal = 0, addable = 0;
};
SetCheck check_set(const Graph &g, std::span<const VertexId> set) {
  SetCheck r;
  if (g.n == 0) {  // membership() still rejects any id (validate.cpp:12-22)
    if (!set.empty())
      throw std::invalid_argument("set contains vertex id " + std::to_string(set[0]) +
                                  " outside [0, n)");
    r.independent = r.maximal = 1;
    return r;
  }
  DeviceGraph dg(g);
  check(tcmis_validate(dg.h, set.data(), static_cast<std::int64_t>(set.size()), &r.independent,
                       &r.u, &r.v, &r.maximal, &r.addable));
  return r;
}
}  // namespace

IndependenceReport check_independence(const Graph &g, std::span<const VertexId> set) {
  const SetCheck c = check_set(g, set);
  IndependenceReport r;
  r.independent = c.independent != 0;
  if (!r.independent) r.violating_edge = std::pair<VertexId, VertexId>{c.u, c.v};
  return r;
}

MaximalityReport check_maximality(const Graph &g, std::span<const VertexId> set) {
  const SetCheck c = check_set(g, set);
  if (!c.independent) throw std::invalid_argument("maximality is defined on independent sets");
  MaximalityReport r;
  r.maximal = c.maximal != 0;
  if (!r.maximal) r.addable_vertex = c.addable;
  return r;
}

// ----------------------------------------------------------------- engine

const char *heuristic_name(Heuristic h) {
  switch (h) {
    case Heuristic::H1: return "h1";
    case Heuristic::H2: return "h2";
    case Heuristic::H3: return "h3";
    case Heuristic::LubyFresh: return "luby-fresh";
    case Heuristic::LubyPerm: return "luby-perm";
  }
  return "?";
}

Heuristic heuristic_from_name(const std::string &name) {
  for (Heuristic h : {Heuristic::H1, Heuristic::H2, Heuristic::H3, Heuristic::LubyFresh,
                      Heuristic::LubyPerm})
    if (name == heuristic_name(h)) return h;
  throw std::invalid_argument("unknown heuristic '" + name + "'");
}

double MISResult::phase1_ms() const {
  double t = 0;
  for (const auto &i : iterations) t += i.phase1_ms;
  return t;
}
double MISResult::phase2_ms() const {
  double t = 0;
  for (const auto &i : iterations) t += i.phase2_ms;
  return t;
}
double MISResult::phase3_ms() const {
  double t = 0;
  for (const auto &i : iterations) t += i.phase3_ms;
  return t;
}
double MISResult::total_ms() const { return phase1_ms() + phase2_ms() + phase3_ms(); }
std::int64_t MISResult::tiles_evaluated() const {
  std::int64_t t = 0;
  for (const auto &i : iterations) t += i.tiles_evaluated;
  return t;
}
std::int64_t MISResult::tiles_skipped() const {
  std::int64_t t = 0;
  for (const auto &i : iterations) t += i.tiles_skipped;
  return t;
}

std::vector<std::uint64_t> compute_max_np(const Graph &g, const PriorityVector &pv,
                                          std::span<const VertexState> states, int) {
  std::vector<std::uint64_t> out(static_cast<std::size_t>(g.n), kNoNeighborKey);
  if (g.n == 0) return out;
  DeviceGraph dg(g);
  check(tcmis_compute_max_np(dg.h, pv.p.data(),
                             reinterpret_cast<const std::uint8_t *>(states.data()), out.data()));
  return out;
}

TiledVector generate_candidates(const PriorityVector &pv, std::span<const std::uint64_t> max_np,
                                std::span<const VertexState> states, int tile_dim, int) {
  const VertexId n = static_cast<VertexId>(states.size());
  std::vector<std::uint8_t> c(static_cast<std::size_t>(n), 0);
  for (VertexId v = 0; v < n; ++v)  // engine.cpp:105-119
    c[v] = states[v] == VertexState::Alive && priority_key(pv, v) > max_np[v];
  return pack_vector(c, tile_dim);
}

Phase3Outcome phase3_update(std::span<VertexState> states, std::span<const std::uint8_t> c,
                            std::span<const std::int32_t> nc, std::vector<VertexId> *newly,
                            int) {
  const VertexId n = static_cast<VertexId>(states.size());
  if (static_cast<VertexId>(c.size()) < n || static_cast<VertexId>(nc.size()) != n)
    throw std::invalid_argument("phase3 input lengths must cover n");
  Phase3Outcome o;
  for (VertexId v = 0; v < n; ++v)  // engine.cpp:121-160
    if (c[v] && states[v] != VertexState::Alive)
      throw std::logic_error("candidate flagged on a non-alive vertex");
  for (VertexId v = 0; v < n; ++v) {
    if (c[v]) {
      states[v] = VertexState::InMIS;
      ++o.selected;
      if (newly) newly->push_back(v);
    } else if (states[v] == VertexState::Alive && nc[v] > 0) {
      states[v] = VertexState::Removed;
      ++o.removed;
    }
  }
  return o;
}

std::vector<std::uint8_t> run_h3_resolution(const Graph &g, const PriorityVector &pv,
                                            std::span<const VertexState> states, int) {
  std::vector<std::uint8_t> c(static_cast<std::size_t>(g.n), 0);
  if (g.n == 0) return c;
  DeviceGraph dg(g);
  check(tcmis_h3_resolution(dg.h, pv.p.data(),
                            reinterpret_cast<const std::uint8_t *>(states.data()), c.data()));
  return c;
}

MISResult run_tc_mis(const Graph &g, const TiledAdjacency &tiled, const EngineConfig &cfg) {
  if (tiled.n != g.n)  // engine.cpp:233-234
    throw std::invalid_argument("tiled adjacency built for a different graph");
  MISResult r;
  r.heuristic = cfg.heuristic;
  r.seed = cfg.seed;
  if (g.n == 0) return r;  // engine.cpp:240
  if (cfg.heuristic != Heuristic::H1 && cfg.heuristic != Heuristic::H2 &&
      cfg.heuristic != Heuristic::H3)  // engine.cpp:29-31
    throw std::invalid_argument("tiled engine only runs h1/h2/h3; use run_luby_reference");
  if (cfg.heuristic != Heuristic::H1 &&
      (cfg.scale_bits < kMinScaleBits || cfg.scale_bits > kMaxScaleBits))
    throw std::invalid_argument("scale_bits must be in [8, 30]");
  check_tile_dim(cfg.tile_dim);  // pack_vector(cfg.tile_dim)
  if (tiled.tile_dim != cfg.tile_dim)  // spmv.cpp:22-24, raised in round 1
    throw std::invalid_argument("tiled adjacency and vector disagree on tile layout");
  DeviceGraph dg(g);
  check(tcmis_graph_set_tiling(dg.h, tiled.tile_dim, tiled.block_row_offsets.data(),
                               tiled.n_block_rows(), tiled.tile_col.data(), tiled.tile_count()));
  return solve(dg.h, g.n, cfg, cfg.heuristic);
}

MISResult run_tc_mis(const Graph &g, const EngineConfig &cfg) {
  check_tile_dim(cfg.tile_dim);  // tile_graph runs first (engine.cpp:297-299)
  MISResult r;
  r.heuristic = cfg.heuristic;
  r.seed = cfg.seed;
  if (g.n == 0) return r;
  if (cfg.heuristic != Heuristic::H1 && cfg.heuristic != Heuristic::H2 &&
      cfg.heuristic != Heuristic::H3)
    throw std::invalid_argument("tiled engine only runs h1/h2/h3; use run_luby_reference");
  ResultIds ids(g.n);               // faulted in while the device works
  DeviceGraph dg(g, cfg.tile_dim);  // tile_graph on the device, overlapped with the upload
  return solve(dg.h, g.n, cfg, cfg.heuristic, &ids);
}

MISResult run_luby_reference(const Graph &g, std::uint64_t seed, LubyMode mode, int scale_bits,
                             int workers) {
  EngineConfig cfg;
  cfg.seed = seed;
  cfg.scale_bits = scale_bits;
  cfg.workers = workers;
  const Heuristic h = mode == LubyMode::Fresh ? Heuristic::LubyFresh : Heuristic::LubyPerm;
  cfg.heuristic = h;
  MISResult r;
  r.heuristic = h;
  r.seed = seed;
  if (g.n == 0) return r;  // engine.cpp:307
  ResultIds ids(g.n);
  DeviceGraph dg(g);
  return solve(dg.h, g.n, cfg, h, &ids);
}

MISResult run_mis(const Graph &g, const EngineConfig &cfg) {  // engine.cpp:354-365
  switch (cfg.heuristic) {
    case Heuristic::LubyFresh:
      return run_luby_reference(g, cfg.seed, LubyMode::Fresh, cfg.scale_bits, cfg.workers);
    case Heuristic::LubyPerm:
      return run_luby_reference(g, cfg.seed, LubyMode::Permutation, cfg.scale_bits,
                                cfg.workers);
    default:
      return run_tc_mis(g, cfg);
  }
}

// ---------------------------------------------------------- multi-GPU

std::vector<VertexId> partition_rows(const Graph &g, int world, int tile_dim) {
  if (world < 1) throw std::invalid_argument("world must be >= 1");
  check_tile_dim(tile_dim);
  const int64_t align = std::lcm<int64_t>(64, tile_dim);
  const int64_t n = g.n;
  const int64_t total = g.offsets.empty() ? 0 : g.offsets.back();
  std::vector<VertexId> lo{0};
  for (int r = 1; r < world; ++r) {
    const int64_t target = total * r / world;
    int64_t v = std::lower_bound(g.offsets.begin(), g.offsets.end(), target) - g.offsets.begin();
    v = std::min(n / align * align, std::max<int64_t>(lo.back(), (v + align / 2) / align * align));
    lo.push_back(static_cast<VertexId>(v));
  }
  lo.push_back(g.n);
  return lo;
}

NcclUniqueId nccl_unique_id() {
  NcclUniqueId id{};
  check(tcmis_nccl_unique_id(id.data()));
  return id;
}

namespace {

struct OwnedCtx {
  tcmis_ctx *h = nullptr;
  explicit OwnedCtx(int device) { check(tcmis_ctx_create(device, &h)); }
  ~OwnedCtx() { tcmis_ctx_destroy(h); }
  OwnedCtx(const OwnedCtx &) = delete;
  OwnedCtx &operator=(const OwnedCtx &) = delete;
};

struct OwnedGraph {
  tcmis_graph *h = nullptr;
  ~OwnedGraph() { tcmis_graph_destroy(h); }
};

struct OwnedExchange {
  tcmis_exchange *h = nullptr;
  ~OwnedExchange() { tcmis_exchange_destroy(h); }
};

void check_partitioned(const Graph &g, const EngineConfig &cfg) {
  check_tile_dim(cfg.tile_dim);
  if (cfg.heuristic == Heuristic::LubyFresh)
    throw std::invalid_argument(
        "luby-fresh redraws every alive key per round; the partitioned solve runs h1, h2, h3 "
        "and luby-perm");
  if (cfg.heuristic != Heuristic::H1 &&
      (cfg.scale_bits < kMinScaleBits || cfg.scale_bits > kMaxScaleBits))
    throw std::invalid_argument("scale_bits must be in [8, 30]");
  (void)g;
}

// one rank: upload its rows, solve through the exchange, the whole result
int solve_rank(const Graph &g, const EngineConfig &cfg, tcmis_ctx *ctx, tcmis_exchange *x,
               const std::vector<VertexId> &lo, int rank, MISResult *out) {
  OwnedGraph part;
  const int64_t a = g.offsets[lo[rank]], b = g.offsets[lo[rank + 1]];
  if (int rc = tcmis_graph_upload_partition(ctx, g.n, lo[rank], lo[rank + 1], g.offsets.data(),
                                            b > a ? g.neighbors.data() + a : nullptr, &part.h))
    return rc;
  tcmis_config c;
  tcmis_config_init(&c);
  c.heuristic = static_cast<int32_t>(cfg.heuristic);
  c.tile_dim = cfg.tile_dim;
  c.seed = cfg.seed;
  c.scale_bits = cfg.scale_bits;
  std::vector<int32_t> mis(static_cast<std::size_t>(std::max<VertexId>(g.n, 1)));
  std::vector<tcmis_iter_stats> st(static_cast<std::size_t>(std::max<VertexId>(g.n, 1)));
  int64_t cnt = 0;
  int32_t nit = 0;
  if (int rc = tcmis_solve_partitioned(part.h, x, lo.data(), static_cast<int32_t>(lo.size() - 1),
                                       &c, nullptr, mis.data(), &cnt, st.data(),
                                       static_cast<int32_t>(st.size()), &nit))
    return rc;
  out->heuristic = cfg.heuristic;
  out->seed = cfg.seed;
  out->mis.assign(mis.begin(), mis.begin() + cnt);
  for (int32_t i = 0; i < nit; ++i) {
    IterationStats s;
    s.iteration = st[i].iteration;
    s.candidates_selected = st[i].candidates_selected;
    s.vertices_removed = st[i].vertices_removed;
    s.alive_remaining = st[i].alive_remaining;
    s.tiles_evaluated = st[i].tiles_evaluated;
    s.tiles_skipped = st[i].tiles_skipped;
    s.phase1_ms = st[i].phase1_ms;
    s.phase2_ms = st[i].phase2_ms;
    s.phase3_ms = st[i].phase3_ms;
    out->iterations.push_back(s);
  }
  return 0;
}

}  // namespace

MISResult run_mis_partitioned(const Graph &g, const EngineConfig &cfg, int world, int rank,
                              const NcclUniqueId &id, int device) {
  check_partitioned(g, cfg);
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank / world");
  MISResult r;
  r.heuristic = cfg.heuristic;
  r.seed = cfg.seed;
  const std::vector<VertexId> lo = partition_rows(g, world, cfg.tile_dim);
  OwnedCtx ctx(device);
  OwnedExchange x;
  check(tcmis_exchange_nccl(ctx.h, world, rank, id.data(), &x.h));
  if (g.n == 0) return r;
  check(solve_rank(g, cfg, ctx.h, x.h, lo, rank, &r));
  return r;
}

MISResult run_mis_partitioned(const Graph &g, const EngineConfig &cfg,
                              const std::vector<int> &devices) {
  check_partitioned(g, cfg);
  const int world = static_cast<int>(devices.size());
  if (world < 1) throw std::invalid_argument("no devices");
  MISResult r;
  r.heuristic = cfg.heuristic;
  r.seed = cfg.seed;
  if (g.n == 0) return r;
  const std::vector<VertexId> lo = partition_rows(g, world, cfg.tile_dim);
  std::vector<std::unique_ptr<OwnedCtx>> ctxs;
  for (int d : devices) ctxs.push_back(std::make_unique<OwnedCtx>(d));
  std::vector<tcmis_exchange *> xs(static_cast<std::size_t>(world), nullptr);
  check(tcmis_exchange_local_group(world, xs.data()));
  std::vector<MISResult> res(static_cast<std::size_t>(world));
  std::vector<int> rcs(static_cast<std::size_t>(world), 0);
  std::vector<std::string> errs(static_cast<std::size_t>(world));
  std::vector<std::thread> th;
  for (int k = 0; k < world; ++k)
    th.emplace_back([&, k] {
      rcs[k] = solve_rank(g, cfg, ctxs[k]->h, xs[k], lo, k, &res[k]);
      if (rcs[k]) {
        errs[k] = tcmis_last_error();  // thread-local
        tcmis_exchange_abort(xs[k]);   // the peers must not wait for this rank
      }
    });
  for (auto &t : th) t.join();
  for (tcmis_exchange *x : xs) tcmis_exchange_destroy(x);
  for (int k = 0; k < world; ++k)
    if (rcs[k]) {
      const std::string msg = errs[k];
      switch (rcs[k]) {
        case TCMIS_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TCMIS_E_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
      }
    }
  return std::move(res[0]);
}

std::string csv_header() {
  return "graph,n,m,heuristic,seed,mis_size,iterations,total_ms,phase1_ms,phase2_ms,phase3_ms,"
         "tiles_evaluated,tiles_skipped";
}

std::string csv_row(const std::string &graph_name, const Graph &g, const MISResult &r) {
  if (graph_name.find_first_of(",\n\"") != std::string::npos)
    throw std::invalid_argument("csv_row: graph name must not contain ',', '\"' or a newline");
  char ms[4][32];
  const double t[4] = {r.total_ms(), r.phase1_ms(), r.phase2_ms(), r.phase3_ms()};
  for (int i = 0; i < 4; ++i) std::snprintf(ms[i], sizeof(ms[i]), "%.3f", t[i]);
  std::string row = graph_name;
  auto put = [&row](const std::string &x) {
    row += ',';
    row += x;
  };
  put(std::to_string(g.n));
  put(std::to_string(g.num_edges()));
  put(heuristic_name(r.heuristic));
  put(std::to_string(r.seed));
  put(std::to_string(r.cardinality()));
  put(std::to_string(r.iterations.size()));
  for (const char *x : ms) put(x);
  put(std::to_string(r.tiles_evaluated()));
  put(std::to_string(r.tiles_skipped()));
  return row;
}

}  // namespace b200
}  // namespace tcmis
