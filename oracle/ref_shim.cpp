// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference library, compiled from the
// reference's own sources in /root/reference/proj/src (see oracle/Makefile)
// into oracle/_ref/libtcmis_ref.so.  It lets the Python tests and the
// cpu_baseline leg of bench.py call the reference exactly as a C++ user would
// (tcmis::run_mis & co.).  No reference source is copied into this repo.
#include <chrono>
#include <fstream>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "support/oracles.hpp"
#include "tcmis/engine.hpp"
#include "tcmis/generate.hpp"
#include "tcmis/graph.hpp"
#include "tcmis/priorities.hpp"
#include "tcmis/spmv.hpp"
#include "tcmis/tiling.hpp"
#include "tcmis/validate.hpp"

namespace {

thread_local std::string g_err;

int code_of(const std::exception_ptr& ep) {
  try {
    std::rethrow_exception(ep);
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 5;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct RoundOut {
  int64_t sel, rem, alive, tiles_eval, tiles_skip;
  double p1, p2, p3;
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int fill_result(const tcmis::MISResult& r, int32_t n, uint8_t* member, int32_t* mis,
                int64_t* mis_count, RoundOut* rounds, int max_rounds, int* n_rounds) {
  if (member) {
    std::memset(member, 0, static_cast<size_t>(n));
    for (auto v : r.mis) member[v] = 1;
  }
  if (mis) std::memcpy(mis, r.mis.data(), r.mis.size() * sizeof(int32_t));
  if (mis_count) *mis_count = static_cast<int64_t>(r.mis.size());
  *n_rounds = static_cast<int>(r.iterations.size());
  for (size_t i = 0; i < r.iterations.size() && static_cast<int>(i) < max_rounds; ++i) {
    const auto& it = r.iterations[i];
    rounds[i] = {it.candidates_selected, it.vertices_removed, it.alive_remaining,
                 it.tiles_evaluated, it.tiles_skipped, it.phase1_ms, it.phase2_ms,
                 it.phase3_ms};
  }
  return 0;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_graph_create(int32_t n, const int64_t* off, const int32_t* nbr) {
  auto* g = new tcmis::Graph();
  g->n = n;
  g->offsets.assign(off, off + n + 1);
  g->neighbors.assign(nbr, nbr + off[n]);
  return g;
}
void ref_graph_free(void* g) { delete static_cast<tcmis::Graph*>(g); }
int32_t ref_graph_n(void* g) { return static_cast<tcmis::Graph*>(g)->n; }
int64_t ref_graph_nnz(void* g) {
  return static_cast<int64_t>(static_cast<tcmis::Graph*>(g)->neighbors.size());
}
void ref_graph_copy(void* gp, int64_t* off, int32_t* nbr) {
  auto* g = static_cast<tcmis::Graph*>(gp);
  std::memcpy(off, g->offsets.data(), g->offsets.size() * sizeof(int64_t));
  std::memcpy(nbr, g->neighbors.data(), g->neighbors.size() * sizeof(int32_t));
}

// generate.hpp
void* ref_gen_rmat(int scale, int ef, uint64_t seed) {
  try {
    return new tcmis::Graph(tcmis::rmat_graph(scale, ef, seed));
  } catch (...) {
    code_of(std::current_exception());
    return nullptr;
  }
}
void* ref_gen_gnp_avg(int32_t n, double avg, uint64_t seed) {
  return new tcmis::Graph(tcmis::gnp_graph_avg_degree(n, avg, seed));
}
void* ref_gen_named(const char* name, int32_t k) {
  std::string s(name);
  if (s == "petersen") return new tcmis::Graph(tcmis::petersen_graph());
  if (s == "path") return new tcmis::Graph(tcmis::path_graph(k));
  if (s == "cycle") return new tcmis::Graph(tcmis::cycle_graph(k));
  if (s == "complete") return new tcmis::Graph(tcmis::complete_graph(k));
  if (s == "star") return new tcmis::Graph(tcmis::star_graph(k));
  if (s == "edgeless") return new tcmis::Graph(tcmis::edgeless_graph(k));
  return nullptr;
}
void* ref_graph_from_edges(int32_t n, int64_t m, const int32_t* eu, const int32_t* ev) {
  std::vector<std::pair<tcmis::VertexId, tcmis::VertexId>> e(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) e[i] = {eu[i], ev[i]};
  try {
    return new tcmis::Graph(tcmis::graph_from_edges(n, e));
  } catch (...) {
    code_of(std::current_exception());
    return nullptr;
  }
}

// priorities.hpp
uint64_t ref_mix64(uint64_t x) { return tcmis::mix64(x); }
uint64_t ref_vertex_hash(uint64_t v, uint64_t s) { return tcmis::vertex_hash(v, s); }
uint64_t ref_combine_seed(uint64_t s, uint64_t r) { return tcmis::combine_seed(s, r); }
double ref_hash_to_unit(uint64_t h) { return tcmis::hash_to_unit(h); }
uint32_t ref_h2_priority_value(double avg, int32_t deg, double eps, int sb) {
  return tcmis::h2_priority_value(avg, deg, eps, sb);
}
int ref_h1_random(int32_t n, uint64_t seed, uint32_t* p) {
  try {
    auto pv = tcmis::h1_random(n, seed);
    std::memcpy(p, pv.p.data(), pv.p.size() * 4);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}
int ref_h2_degree_aware(void* g, uint64_t seed, int sb, uint32_t* p) {
  try {
    auto pv = tcmis::h2_degree_aware(*static_cast<tcmis::Graph*>(g), seed, sb);
    std::memcpy(p, pv.p.data(), pv.p.size() * 4);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// tiling.hpp
void* ref_tile_graph(void* g, int T, double* ms) {
  try {
    double t0 = now_ms();
    auto* a = new tcmis::TiledAdjacency(tcmis::tile_graph(*static_cast<tcmis::Graph*>(g), T));
    if (ms) *ms = now_ms() - t0;
    return a;
  } catch (...) {
    code_of(std::current_exception());
    return nullptr;
  }
}
void ref_tiled_free(void* a) { delete static_cast<tcmis::TiledAdjacency*>(a); }
int64_t ref_tiled_count(void* a) { return static_cast<tcmis::TiledAdjacency*>(a)->tile_count(); }
int ref_tiled_dim(void* a) { return static_cast<tcmis::TiledAdjacency*>(a)->tile_dim; }
void ref_tiled_copy(void* ap, int32_t* tile_row, int32_t* tile_col, uint64_t* row_bits,
                    int64_t* bro) {
  auto* a = static_cast<tcmis::TiledAdjacency*>(ap);
  std::memcpy(tile_row, a->tile_row.data(), a->tile_row.size() * 4);
  std::memcpy(tile_col, a->tile_col.data(), a->tile_col.size() * 4);
  std::memcpy(row_bits, a->row_bits.data(), a->row_bits.size() * 8);
  std::memcpy(bro, a->block_row_offsets.data(), a->block_row_offsets.size() * 8);
}
int ref_tiled_spmv(void* ap, const uint8_t* c, int32_t n, int32_t* nc, int64_t* ev,
                   int64_t* sk) {
  try {
    auto* a = static_cast<tcmis::TiledAdjacency*>(ap);
    auto tv = tcmis::pack_vector({c, static_cast<size_t>(n)}, a->tile_dim);
    tcmis::SpmvStats st;
    auto out = tcmis::tiled_spmv(*a, tv, {}, &st);
    std::memcpy(nc, out.data(), out.size() * 4);
    *ev = st.tiles_evaluated;
    *sk = st.tiles_skipped;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// engine.hpp -- heuristic ids follow engine.hpp:19 declaration order
int ref_run_mis(void* g, int heuristic, uint64_t seed, int tile_dim, int workers,
                int scale_bits, uint8_t* member, int32_t* mis, int64_t* mis_count,
                RoundOut* rounds, int max_rounds, int* n_rounds, double* wall_ms) {
  try {
    tcmis::EngineConfig cfg;
    cfg.heuristic = static_cast<tcmis::Heuristic>(heuristic);
    cfg.seed = seed;
    cfg.tile_dim = tile_dim;
    cfg.workers = workers;
    cfg.scale_bits = scale_bits;
    double t0 = now_ms();
    auto r = tcmis::run_mis(*static_cast<tcmis::Graph*>(g), cfg);
    if (wall_ms) *wall_ms = now_ms() - t0;
    return fill_result(r, static_cast<tcmis::Graph*>(g)->n, member, mis, mis_count, rounds,
                       max_rounds, n_rounds);
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_run_tc_mis_tiled(void* g, void* tiled, int heuristic, uint64_t seed, int tile_dim,
                         int workers, int scale_bits, uint8_t* member, int64_t* mis_count,
                         RoundOut* rounds, int max_rounds, int* n_rounds, double* wall_ms) {
  try {
    tcmis::EngineConfig cfg;
    cfg.heuristic = static_cast<tcmis::Heuristic>(heuristic);
    cfg.seed = seed;
    cfg.tile_dim = tile_dim;
    cfg.workers = workers;
    cfg.scale_bits = scale_bits;
    double t0 = now_ms();
    auto r = tcmis::run_tc_mis(*static_cast<tcmis::Graph*>(g),
                               *static_cast<tcmis::TiledAdjacency*>(tiled), cfg);
    if (wall_ms) *wall_ms = now_ms() - t0;
    return fill_result(r, static_cast<tcmis::Graph*>(g)->n, member, nullptr, mis_count, rounds,
                       max_rounds, n_rounds);
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_run_luby(void* g, uint64_t seed, int fresh, int scale_bits, int workers,
                 uint8_t* member, int64_t* mis_count, RoundOut* rounds, int max_rounds,
                 int* n_rounds, double* wall_ms) {
  try {
    double t0 = now_ms();
    auto r = tcmis::run_luby_reference(*static_cast<tcmis::Graph*>(g), seed,
                                       fresh ? tcmis::LubyMode::Fresh
                                             : tcmis::LubyMode::Permutation,
                                       scale_bits, workers);
    if (wall_ms) *wall_ms = now_ms() - t0;
    return fill_result(r, static_cast<tcmis::Graph*>(g)->n, member, nullptr, mis_count, rounds,
                       max_rounds, n_rounds);
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// tests/support/oracles.hpp
int64_t ref_sequential_greedy(void* g, const uint32_t* p, uint8_t* member) {
  auto* gr = static_cast<tcmis::Graph*>(g);
  tcmis::PriorityVector pv;
  pv.p.assign(p, p + gr->n);
  auto mis = tcmis::testing::sequential_greedy_mis(*gr, pv);
  std::memset(member, 0, static_cast<size_t>(gr->n));
  for (auto v : mis) member[v] = 1;
  return static_cast<int64_t>(mis.size());
}

int ref_compute_max_np(void* g, const uint32_t* p, const uint8_t* states, uint64_t* out) {
  auto* gr = static_cast<tcmis::Graph*>(g);
  tcmis::PriorityVector pv;
  pv.p.assign(p, p + gr->n);
  std::vector<tcmis::VertexState> st(gr->n);
  for (int32_t v = 0; v < gr->n; ++v) st[v] = static_cast<tcmis::VertexState>(states[v]);
  auto r = tcmis::compute_max_np(*gr, pv, st, 1);
  std::memcpy(out, r.data(), r.size() * 8);
  return 0;
}

int ref_h3_resolution(void* g, const uint32_t* p, const uint8_t* states, uint8_t* c) {
  auto* gr = static_cast<tcmis::Graph*>(g);
  tcmis::PriorityVector pv;
  pv.p.assign(p, p + gr->n);
  std::vector<tcmis::VertexState> st(gr->n);
  for (int32_t v = 0; v < gr->n; ++v) st[v] = static_cast<tcmis::VertexState>(states[v]);
  auto r = tcmis::run_h3_resolution(*gr, pv, st, 1);
  std::memcpy(c, r.data(), r.size());
  return 0;
}

// validate.cpp:45-75 -- the reference's own validators (pins the oracle's)
int ref_check_independence(void* gh, const int32_t* set, int64_t cnt, int32_t* independent,
                           int32_t* wu, int32_t* wv) {
  try {
    const auto& g = *static_cast<tcmis::Graph*>(gh);
    auto r = tcmis::check_independence(g, std::span<const tcmis::VertexId>(set, (size_t)cnt));
    *independent = r.independent ? 1 : 0;
    if (r.violating_edge) {
      *wu = r.violating_edge->first;
      *wv = r.violating_edge->second;
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_check_maximality(void* gh, const int32_t* set, int64_t cnt, int32_t* maximal,
                         int32_t* addable) {
  try {
    const auto& g = *static_cast<tcmis::Graph*>(gh);
    auto r = tcmis::check_maximality(g, std::span<const tcmis::VertexId>(set, (size_t)cnt));
    *maximal = r.maximal ? 1 : 0;
    if (r.addable_vertex) *addable = *r.addable_vertex;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// tiling.cpp write_tiled of tile_graph(g, T) into `path` (format pin)
int ref_write_tiled(void* gh, int32_t T, const char* path) {
  try {
    const auto& g = *static_cast<tcmis::Graph*>(gh);
    auto a = tcmis::tile_graph(g, T);
    std::ofstream f(path, std::ios::binary);
    tcmis::write_tiled(f, a);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

}  // extern "C"
