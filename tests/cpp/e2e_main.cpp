// e2e_main.cpp -- the reference user's MIS call, timed end to end: a program
// written against the reference's public API (tcmis/engine.hpp) calls
// tcmis::run_mis(const Graph &, const EngineConfig &) on a Graph held in plain
// std::vector (pageable) storage, linked against the B200 drop-in libtcmis.so.
// The call uploads the CSR, tiles it, solves and returns the MISResult --
// exactly what the reference's run_mis does on its CPU (engine.cpp:354-365).
//
// usage: e2e_main <graph.bin> [reps] [heuristic]
// graph.bin: int32 n, int64 nnz, int64 offsets[n+1], int32 neighbors[nnz]
// prints one JSON object: per-call wall times (ms), |MIS|, iterations and an
// FNV hash of the MIS for the caller to check against the device solve.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "tcmis/engine.hpp"
#include "tcmis_b200.h"

using namespace tcmis;

static Graph read_graph(const char *path) {
  std::ifstream in(path, std::ios::binary);
  Graph g;
  int64_t nnz = 0;
  in.read(reinterpret_cast<char *>(&g.n), 4);
  in.read(reinterpret_cast<char *>(&nnz), 8);
  g.offsets.resize(static_cast<size_t>(g.n) + 1);
  g.neighbors.resize(static_cast<size_t>(nnz));
  in.read(reinterpret_cast<char *>(g.offsets.data()), 8 * (static_cast<int64_t>(g.n) + 1));
  in.read(reinterpret_cast<char *>(g.neighbors.data()), 4 * nnz);
  return g;
}

int main(int argc, char **argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s graph.bin [reps] [heuristic]\n", argv[0]);
    return 2;
  }
  const Graph g = read_graph(argv[1]);
  const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
  EngineConfig cfg;
  cfg.heuristic = heuristic_from_name(argc > 3 ? argv[3] : "h2");
  cfg.seed = 1;
  cfg.tile_dim = 16;
  MISResult r = run_mis(g, cfg);  // warm-up: contexts, pools, the solve graph
  std::vector<double> ms;
  for (int k = 0; k < reps; ++k) {
    const auto t0 = std::chrono::steady_clock::now();
    r = run_mis(g, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
  }
  // the same call split at the C-ABI (upload + tile count / solve with the ids
  // into a pre-allocated std::vector / destroy), for the breakdown
  double br[4] = {0, 0, 0, 0};
  {
    tcmis_ctx *ctx = nullptr;
    tcmis_ctx_create(0, &ctx);
    std::vector<int32_t> ids(static_cast<size_t>(g.n));
    std::vector<tcmis_iter_stats> st(4096);
    for (int k = 0; k < reps + 1; ++k) {
      const auto t0 = std::chrono::steady_clock::now();
      tcmis_graph *dg = nullptr;
      tcmis_graph_upload_tiled(ctx, g.n, g.offsets.data(), g.neighbors.data(), 16, &dg, nullptr);
      const auto t1 = std::chrono::steady_clock::now();
      tcmis_config c;
      tcmis_config_init(&c);
      c.heuristic = static_cast<int32_t>(cfg.heuristic);
      int64_t cnt = 0;
      int32_t nit = 0;
      tcmis_solve(dg, &c, nullptr, ids.data(), &cnt, st.data(), 4096, &nit);
      const auto t2 = std::chrono::steady_clock::now();
      std::vector<VertexId> out(ids.begin(), ids.begin() + cnt);  // MISResult::mis
      const auto t3 = std::chrono::steady_clock::now();
      tcmis_graph_destroy(dg);
      const auto t4 = std::chrono::steady_clock::now();
      if (k) {
        br[0] += std::chrono::duration<double, std::milli>(t1 - t0).count() / reps;
        br[1] += std::chrono::duration<double, std::milli>(t2 - t1).count() / reps;
        br[2] += std::chrono::duration<double, std::milli>(t3 - t2).count() / reps;
        br[3] += std::chrono::duration<double, std::milli>(t4 - t3).count() / reps;
      }
    }
    tcmis_ctx_destroy(ctx);
  }
  std::vector<double> sorted = ms;
  std::sort(sorted.begin(), sorted.end());
  uint64_t h = 0xcbf29ce484222325ULL;
  for (VertexId x : r.mis) {
    h ^= static_cast<uint32_t>(x);
    h *= 0x100000001b3ULL;
  }
  std::printf("{\"n\": %d, \"m\": %lld, \"mis_size\": %lld, \"iterations\": %zu, "
              "\"mis_fnv\": %llu, \"median_ms\": %.4f, \"ms\": [",
              g.n, static_cast<long long>(g.num_edges()), static_cast<long long>(r.cardinality()),
              r.iterations.size(), static_cast<unsigned long long>(h), sorted[sorted.size() / 2]);
  for (size_t i = 0; i < ms.size(); ++i) std::printf("%s%.4f", i ? ", " : "", ms[i]);
  std::printf("], \"capi_breakdown_ms\": {\"upload_tiled\": %.4f, \"solve_ids_to_vector\": %.4f, "
              "\"result_vector\": %.4f, \"destroy\": %.4f}}\n",
              br[0], br[1], br[2], br[3]);
  return 0;
}
