// tcmis/tcmis.hpp -- the C++ drop-in API of the B200 engine.
//
// Source-compatible with the reference's public headers for the MIS path
// (/root/reference/proj/include/tcmis/{graph,priorities,tiling,spmv,engine}.hpp):
// the same names, types, argument meaning and exception types.  A program
// written against the reference switches by including these headers and
// linking libtcmis.so (+ libtcmis_b200.so) instead of libtcmis_core.a.
//
// Everything that walks the graph runs on the GPU through the C-ABI of
// tcmis_b200.h; the few elementwise helpers that touch no graph
// (pack_vector, tile_mma, generate_candidates, phase3_update, the hash
// functions) are plain host code, exactly as small as their definitions.
// Symbols live in the inline namespace tcmis::b200, so a binary can hold
// both this library and the reference without ODR clashes.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <iosfwd>
#include <optional>
#include <span>
#include <utility>
#include <string>
#include <utility>
#include <vector>

namespace tcmis {
inline namespace b200 {

// ------------------------------------------------------------------ graph
// graph.hpp:11-39

using VertexId = std::int32_t;
using EdgeIndex = std::int64_t;

struct Graph {
  VertexId n = 0;
  std::vector<EdgeIndex> offsets;   // n + 1 entries, offsets[0] == 0
  std::vector<VertexId> neighbors;  // 2m entries, rows sorted, no loops/duplicates

  EdgeIndex num_edges() const { return static_cast<EdgeIndex>(neighbors.size()) / 2; }
  VertexId degree(VertexId v) const {
    return static_cast<VertexId>(offsets[v + 1] - offsets[v]);
  }
  std::span<const VertexId> neighbors_of(VertexId v) const {
    return {neighbors.data() + offsets[v], static_cast<std::size_t>(degree(v))};
  }
  bool has_edge(VertexId u, VertexId v) const;
  bool operator==(const Graph &) const = default;
};

// graph.cpp:14-41 semantics: loops dropped, reverse edges added, duplicates
// merged; std::out_of_range for endpoints outside [0, n).
Graph graph_from_edges(VertexId n, std::span<const std::pair<VertexId, VertexId>> edges);

// ------------------------------------------------------------- priorities
// priorities.hpp:11-69

std::uint64_t mix64(std::uint64_t x);
std::uint64_t vertex_hash(std::uint64_t v, std::uint64_t seed);
double hash_to_unit(std::uint64_t h);
std::uint64_t combine_seed(std::uint64_t seed, std::uint64_t round);

inline constexpr int kDefaultScaleBits = 20;
inline constexpr int kMinScaleBits = 8;
inline constexpr int kMaxScaleBits = 30;

struct PriorityVector {
  std::vector<std::uint32_t> p;
  std::uint64_t seed = 0;
  VertexId size() const { return static_cast<VertexId>(p.size()); }
};

// Computed on the GPU (k_priorities); bit-identical to the reference.
PriorityVector h1_random(VertexId n, std::uint64_t seed);
std::uint32_t h2_priority_value(double avg_degree, VertexId degree, double eps, int scale_bits);
PriorityVector h2_degree_aware(const Graph &g, std::uint64_t seed,
                               int scale_bits = kDefaultScaleBits);

inline constexpr std::uint64_t kNoNeighborKey = 0;

inline std::uint64_t priority_key(const PriorityVector &pv, VertexId v) {
  return (static_cast<std::uint64_t>(pv.p[v]) << 32) |
         (static_cast<std::uint64_t>(static_cast<std::uint32_t>(v)) + 1);
}
inline bool priority_gt(const PriorityVector &pv, VertexId u, VertexId v) {
  return priority_key(pv, v) > priority_key(pv, u);
}

// ----------------------------------------------------------------- tiling
// tiling.hpp:17-64

struct TiledAdjacency {
  int tile_dim = 16;
  VertexId n = 0;
  VertexId n_padded = 0;
  std::vector<std::int32_t> tile_row;
  std::vector<std::int32_t> tile_col;
  std::vector<std::uint64_t> row_bits;  // tile_dim words per tile
  std::vector<std::int64_t> block_row_offsets;

  std::int64_t tile_count() const { return static_cast<std::int64_t>(tile_col.size()); }
  std::int32_t n_block_rows() const {
    return block_row_offsets.empty() ? 0
                                     : static_cast<std::int32_t>(block_row_offsets.size() - 1);
  }
  std::span<const std::uint64_t> tile_payload(std::int64_t t) const {
    return {row_bits.data() + t * tile_dim, static_cast<std::size_t>(tile_dim)};
  }
  bool payload_bit(std::int64_t t, int i, int j) const {
    return (row_bits[t * tile_dim + i] >> j) & 1u;
  }
};

// K1 on the GPU (warp-per-block-row merge, tiles.cu); std::invalid_argument
// unless 1 <= tile_dim <= 64.
TiledAdjacency tile_graph(const Graph &g, int tile_dim);

/// tiling.hpp:69 -- inverse of tile_graph: the source graph back from its tiles.
Graph tiled_to_csr_roundtrip(const TiledAdjacency &a);

/// tiling.hpp:71-78
struct TileStats {
  std::int64_t tile_count = 0;
  std::int64_t total_nonzeros = 0;
  std::vector<std::int64_t> occupancy_histogram;  // index = non-zeros per tile
  double density = 0.0;                           // tile_count*T^2 / n_padded^2
};
TileStats tile_stats(const TiledAdjacency &a);

/// tiling.hpp:80-86 -- the binary cache "TCMISTIL" (little endian): 8-byte
/// magic, u32 version 1, u32 tile_dim, u64 n, u64 tile_count, then per tile
/// u32 block_row, u32 block_col and ceil(T*T/8) payload bytes, row-major,
/// bit k = entry (k/T, k%T), LSB-first.  read_tiled throws std::runtime_error
/// on a bad magic / version / truncated or unsorted file.
void write_tiled(std::ostream &out, const TiledAdjacency &a);
TiledAdjacency read_tiled(std::istream &in);
std::int64_t tiled_bytes_estimate(const TiledAdjacency &a);
std::int64_t csr_bytes_estimate(const Graph &g);

struct TiledVector {
  int tile_dim = 16;
  VertexId n = 0;
  VertexId n_padded = 0;
  std::vector<std::uint8_t> values;
  std::vector<std::uint64_t> segment_bits;
  std::int32_t n_segments() const { return static_cast<std::int32_t>(segment_bits.size()); }
  bool segment_nonzero(std::int32_t s) const { return segment_bits[s] != 0; }
};

TiledVector pack_vector(std::span<const std::uint8_t> values, int tile_dim);

// ------------------------------------------------------------------- spmv
// spmv.hpp:15-42

void tile_mma(std::span<const std::uint64_t> payload_rows, std::uint64_t segment_bits,
              std::span<std::int32_t> out);

struct SpmvStats {
  std::int64_t tiles_evaluated = 0;
  std::int64_t tiles_skipped = 0;
};

struct SpmvOptions {
  int workers = 0;                  // accepted, ignored (GPU)
  bool skip_empty_segments = true;
};

// nc = A * c on the GPU.  The counts are the CSR neighbour counts (identical
// to the tile products by definition); tiles_evaluated / tiles_skipped are
// the given tiling's counters.
std::vector<std::int32_t> tiled_spmv(const TiledAdjacency &a, const TiledVector &c,
                                     const SpmvOptions &options = {},
                                     SpmvStats *stats = nullptr);

std::vector<std::int32_t> csr_neighbor_count_oracle(const Graph &g,
                                                    std::span<const std::uint8_t> candidates);

// ----------------------------------------------------------------- engine
// engine.hpp:15-131

enum class VertexState : std::uint8_t { Alive = 0, InMIS = 1, Removed = 2 };
enum class Heuristic { H1, H2, H3, LubyFresh, LubyPerm };

const char *heuristic_name(Heuristic h);
Heuristic heuristic_from_name(const std::string &name);

struct IterationStats {
  int iteration = 0;
  std::int64_t candidates_selected = 0;
  std::int64_t vertices_removed = 0;
  std::int64_t alive_remaining = 0;
  std::int64_t tiles_evaluated = 0;
  std::int64_t tiles_skipped = 0;
  double phase1_ms = 0.0;  // device time of the select kernels
  double phase2_ms = 0.0;  // device time of the pull-form exclusion kernels
  double phase3_ms = 0.0;  // device time of the update kernels
};

struct MISResult {
  std::vector<VertexId> mis;
  std::vector<IterationStats> iterations;
  Heuristic heuristic = Heuristic::H3;
  std::uint64_t seed = 0;

  std::int64_t cardinality() const { return static_cast<std::int64_t>(mis.size()); }
  double phase1_ms() const;
  double phase2_ms() const;
  double phase3_ms() const;
  double total_ms() const;
  std::int64_t tiles_evaluated() const;
  std::int64_t tiles_skipped() const;
};

struct EngineConfig {
  Heuristic heuristic = Heuristic::H3;
  std::uint64_t seed = 1;
  int tile_dim = 16;
  int workers = 0;  // accepted, ignored: the CUDA grid replaces the thread pool
  int scale_bits = kDefaultScaleBits;
  std::function<void(int iteration, std::span<const std::uint8_t> candidates,
                     std::span<const VertexState> states)>
      iteration_observer;
};

std::vector<std::uint64_t> compute_max_np(const Graph &g, const PriorityVector &priorities,
                                          std::span<const VertexState> states, int workers = 1);

TiledVector generate_candidates(const PriorityVector &priorities,
                                std::span<const std::uint64_t> max_np,
                                std::span<const VertexState> states, int tile_dim,
                                int workers = 1);

struct Phase3Outcome {
  std::int64_t selected = 0;
  std::int64_t removed = 0;
};

Phase3Outcome phase3_update(std::span<VertexState> states,
                            std::span<const std::uint8_t> candidates,
                            std::span<const std::int32_t> neighbor_counts,
                            std::vector<VertexId> *newly_selected = nullptr, int workers = 1);

// GPU: the rounds of the engine started from the given alive set.
std::vector<std::uint8_t> run_h3_resolution(const Graph &g, const PriorityVector &priorities,
                                            std::span<const VertexState> states,
                                            int workers = 1);

MISResult run_tc_mis(const Graph &g, const TiledAdjacency &tiled, const EngineConfig &config);
MISResult run_tc_mis(const Graph &g, const EngineConfig &config);

enum class LubyMode { Fresh, Permutation };

MISResult run_luby_reference(const Graph &g, std::uint64_t seed, LubyMode mode,
                             int scale_bits = kDefaultScaleBits, int workers = 1);

MISResult run_mis(const Graph &g, const EngineConfig &config);

// ----------------------------------------------- multi-GPU
// Not in the reference (a single-process CPU engine): the row-partitioned
// solve over several B200s (csrc/partitioned.cu, tcmis_solve_partitioned).
// For h1 / h2 / h3 / luby-perm the result (mis, iterations, every counter)
// equals run_mis(g, cfg) at any world size; luby-fresh throws
// std::invalid_argument.  Phase times are the calling rank's.

/// Edge-balanced contiguous row ranges rank_lo[world + 1] (rank_lo[0] = 0,
/// rank_lo[world] = n), inner boundaries at multiples of lcm(64, tile_dim).
std::vector<VertexId> partition_rows(const Graph &g, int world, int tile_dim = 16);

using NcclUniqueId = std::array<std::uint8_t, 128>;
/// Rank 0 creates it; the caller broadcasts it to the other ranks (MPI, a
/// file, torch.distributed, ...).
NcclUniqueId nccl_unique_id();

/// One process per GPU: this rank uploads its rows of g to `device` and
/// solves with its world - 1 peers over NCCL.
MISResult run_mis_partitioned(const Graph &g, const EngineConfig &config, int world, int rank,
                              const NcclUniqueId &id, int device);

/// One process: one rank per entry of `devices` (repeats allowed), each
/// driven by its own host thread, exchanging through UVA / peer copies.
MISResult run_mis_partitioned(const Graph &g, const EngineConfig &config,
                              const std::vector<int> &devices);

/// The result row of the reference's `cmd_run` (the absent
/// CLI): graph, n, m, heuristic, seed, |MIS|, iterations, total ms, phase 1/2/3
/// ms, tiles evaluated, tiles skipped -- comma-separated, no trailing newline.
/// Phase times are the device times the result carries (the round kernels'
/// %globaltimer stamps on every solve path).
std::string csv_header();
std::string csv_row(const std::string &graph_name, const Graph &g, const MISResult &r);

// ------------------------------------------------------------- validate.hpp
// validate.hpp:12-31 check_independence / check_maximality, evaluated on the
// device (tcmis_validate); same witnesses and exception types.
struct IndependenceReport {
  bool independent = false;
  std::optional<std::pair<VertexId, VertexId>> violating_edge;
};

IndependenceReport check_independence(const Graph &g, std::span<const VertexId> set);

struct MaximalityReport {
  bool maximal = false;
  std::optional<VertexId> addable_vertex;
};

/// Requires an independent input set; throws std::invalid_argument otherwise.
MaximalityReport check_maximality(const Graph &g, std::span<const VertexId> set);

}  // namespace b200
}  // namespace tcmis
