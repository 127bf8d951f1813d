// dropin_main.cpp -- a C++ program written against the reference's public
// API (tcmis/engine.hpp & co.), linked against the B200 drop-in libtcmis.so.
// Reads a CSR graph (binary: int32 n, int64 nnz, int64 offsets[n+1], int32
// neighbors[nnz]) and prints one JSON object per (heuristic, seed) run plus
// the exception checks, for tests/test_gpu_dropin.py to compare with the
// oracle.
#include <cstdio>
#include <fstream>
#include <stdexcept>
#include <sstream>
#include <string>

#include "tcmis/engine.hpp"
#include "tcmis/tiling.hpp"
#include "tcmis/validate.hpp"

using namespace tcmis;

static Graph read_graph(const char *path) {
  std::ifstream in(path, std::ios::binary);
  Graph g;
  int64_t nnz = 0;
  in.read(reinterpret_cast<char *>(&g.n), 4);
  in.read(reinterpret_cast<char *>(&nnz), 8);
  g.offsets.resize(static_cast<size_t>(g.n) + 1);
  g.neighbors.resize(static_cast<size_t>(nnz));
  in.read(reinterpret_cast<char *>(g.offsets.data()), 8 * (g.n + 1));
  in.read(reinterpret_cast<char *>(g.neighbors.data()), 4 * nnz);
  return g;
}

static uint64_t fnv(const std::vector<VertexId> &v) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (VertexId x : v) {
    h ^= static_cast<uint32_t>(x);
    h *= 0x100000001b3ULL;
  }
  return h;
}

template <typename E, typename F>
static const char *throws(F f) {
  try {
    f();
  } catch (const E &) {
    return "yes";
  } catch (...) {
    return "other";
  }
  return "no";
}

int main(int argc, char **argv) {
  Graph g = read_graph(argv[1]);
  for (const char *name : {"h1", "h2", "h3", "luby-fresh", "luby-perm"}) {
    for (uint64_t seed : {1ull, 7ull}) {
      EngineConfig cfg;
      cfg.heuristic = heuristic_from_name(name);
      cfg.seed = seed;
      int observed = 0;
      cfg.iteration_observer = [&](int, std::span<const std::uint8_t>,
                                   std::span<const VertexState>) { ++observed; };
      MISResult r = run_mis(g, cfg);
      std::printf("{\"heuristic\": \"%s\", \"seed\": %llu, \"size\": %lld, \"mis_fnv\": %llu, "
                  "\"observed\": %d, \"rounds\": [",
                  name, (unsigned long long)seed, (long long)r.cardinality(),
                  (unsigned long long)fnv(r.mis), observed);
      for (size_t i = 0; i < r.iterations.size(); ++i) {
        const auto &it = r.iterations[i];
        std::printf("%s[%lld, %lld, %lld, %lld, %lld]", i ? ", " : "",
                    (long long)it.candidates_selected, (long long)it.vertices_removed,
                    (long long)it.alive_remaining, (long long)it.tiles_evaluated,
                    (long long)it.tiles_skipped);
      }
      std::printf("]}\n");
    }
  }
  // prebuilt-tiles overload with T = 8
  TiledAdjacency t8 = tile_graph(g, 8);
  EngineConfig c8;
  c8.heuristic = Heuristic::H2;
  c8.tile_dim = 8;
  MISResult r8 = run_tc_mis(g, t8, c8);
  std::printf("{\"tiles8\": %lld, \"t8_rounds\": %zu, \"t8_eval1\": %lld}\n",
              (long long)t8.tile_count(), r8.iterations.size(),
              (long long)(r8.iterations.empty() ? 0 : r8.iterations[0].tiles_evaluated));
  // tiling.hpp persistence: binary cache write -> read,
  // roundtrip to CSR, statistics
  {
    TiledAdjacency t16 = tile_graph(g, 16);
    const std::string path = std::string(argv[1]) + ".t16";
    {
      std::ofstream f(path, std::ios::binary);
      write_tiled(f, t16);
    }
    std::ifstream f(path, std::ios::binary);
    TiledAdjacency back = read_tiled(f);
    const bool same = back.tile_row == t16.tile_row && back.tile_col == t16.tile_col &&
                      back.row_bits == t16.row_bits &&
                      back.block_row_offsets == t16.block_row_offsets && back.n == t16.n;
    Graph rt = tiled_to_csr_roundtrip(t16);
    const bool rt_ok = rt.offsets == g.offsets && rt.neighbors == g.neighbors;
    TileStats ts = tile_stats(t16);
    std::printf("{\"tiled_io\": %d, \"roundtrip\": %d, \"nonzeros\": %lld, \"hist0\": %lld, "
                "\"bytes_est\": %lld, \"csr_est\": %lld}\n",
                same ? 1 : 0, rt_ok ? 1 : 0, (long long)ts.total_nonzeros,
                (long long)ts.occupancy_histogram[0], (long long)tiled_bytes_estimate(t16),
                (long long)csr_bytes_estimate(g));
    std::stringstream bad("NOTTILED........");
    std::printf("{\"bad_magic\": \"%s\"}\n",
                throws<std::runtime_error>([&] { read_tiled(bad); }));
  }
  // validate.hpp on the device: the H2 result, and the result minus its
  // first vertex (no longer maximal)
  {
    EngineConfig c2;
    c2.heuristic = Heuristic::H2;
    MISResult r2 = run_mis(g, c2);
    IndependenceReport ir = check_independence(g, r2.mis);
    MaximalityReport mr = check_maximality(g, r2.mis);
    std::span<const VertexId> tail(r2.mis.data() + 1, r2.mis.size() - 1);
    MaximalityReport mr2 = check_maximality(g, tail);
    std::printf("{\"valid_ind\": %d, \"valid_max\": %d, \"minus_first_max\": %d, "
                "\"addable\": %d}\n",
                ir.independent ? 1 : 0, mr.maximal ? 1 : 0, mr2.maximal ? 1 : 0,
                mr2.addable_vertex ? (int)*mr2.addable_vertex : -1);
  }
  // cmd_run's CSV row
  {
    EngineConfig c2;
    c2.heuristic = Heuristic::H2;
    MISResult r2 = run_mis(g, c2);
    std::printf("{\"csv_header\": \"%s\", \"csv_row\": \"%s\", \"csv_bad_name\": \"%s\"}\n",
                csv_header().c_str(), csv_row("g", g, r2).c_str(),
                throws<std::invalid_argument>([&] { csv_row("a,b", g, r2); }));
  }
  // reference error behaviour
  EngineConfig bad;
  bad.tile_dim = 0;
  EngineConfig luby;
  luby.heuristic = Heuristic::LubyPerm;
  EngineConfig sb;
  sb.heuristic = Heuristic::H2;
  sb.scale_bits = 31;
  std::printf("{\"bad_tile\": \"%s\", \"luby_tiled\": \"%s\", \"bad_scale\": \"%s\", "
              "\"bad_name\": \"%s\", \"edge_range\": \"%s\"}\n",
              throws<std::invalid_argument>([&] { run_mis(g, bad); }),
              throws<std::invalid_argument>([&] { run_tc_mis(g, luby); }),
              throws<std::invalid_argument>([&] { run_mis(g, sb); }),
              throws<std::invalid_argument>([&] { heuristic_from_name("h9"); }),
              throws<std::out_of_range>([&] {
                std::pair<VertexId, VertexId> e[1] = {{0, g.n}};
                graph_from_edges(g.n, e);
              }));
  return 0;
}
