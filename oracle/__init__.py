"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TC-MIS hot path.

Two checkers live here, both loaded through ctypes:

* ``liboracle.so`` -- the plain-C restatement in ``tcmis_oracle.c`` (every
  function cites the reference file:line it restates);
* ``_ref/libtcmis_ref.so`` -- the UNMODIFIED reference library compiled from
  ``/root/reference/proj/src`` by ``oracle/Makefile`` plus a C shim
  (``ref_shim.cpp``).  It exists wherever ``make -C oracle ref`` ran (in the
  build container; the prebuilt file travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_2605_29604_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtcmis_ref.so")

_lib = None
_ref = None

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


class OrcGraph(C.Structure):
    _fields_ = [("n", C.c_int32), ("nnz", C.c_int64),
                ("off", C.POINTER(C.c_int64)), ("nbr", C.POINTER(C.c_int32))]


class OrcRound(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "sel", "rem", "alive", "tiles_eval", "tiles_skip", "alive_start",
        "nnz_alive", "noncand", "nnz_noncand", "nnz_cand")]


class RefRound(C.Structure):
    _fields_ = [("sel", C.c_int64), ("rem", C.c_int64), ("alive", C.c_int64),
                ("tiles_eval", C.c_int64), ("tiles_skip", C.c_int64),
                ("p1", C.c_double), ("p2", C.c_double), ("p3", C.c_double)]


@dataclass
class Graph:
    """CSR in the reference layout (graph.hpp:18-39)."""
    n: int
    off: np.ndarray  # int64[n+1]
    nbr: np.ndarray  # int32[2m]

    @property
    def num_edges(self) -> int:
        return int(self.nbr.size) // 2


def build() -> None:
    """Build liboracle.so (and the reference shim when the sources exist)."""
    import subprocess
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_vertex_hash.restype = C.c_uint64
        L.orc_vertex_hash.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_hash_to_unit.restype = C.c_double
        L.orc_hash_to_unit.argtypes = [C.c_uint64]
        L.orc_combine_seed.restype = C.c_uint64
        L.orc_combine_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_h1_random.argtypes = [C.c_int32, C.c_uint64, u32p]
        L.orc_h2_priority_value.restype = C.c_uint32
        L.orc_h2_priority_value.argtypes = [C.c_double, C.c_int32, C.c_double, C.c_int]
        L.orc_h2_degree_aware.argtypes = [C.c_int32, i64p, C.c_uint64, C.c_int, u32p]
        L.orc_luby_rounds.argtypes = [C.c_int32, i64p, i32p, C.c_void_p, C.c_int, C.c_uint64,
                                      C.c_void_p, C.c_int, u8p, C.POINTER(OrcRound), C.c_int]
        L.orc_h3_resolution.argtypes = [C.c_int32, i64p, i32p, u32p, u8p, u8p]
        L.orc_greedy_mis.restype = C.c_int64
        L.orc_greedy_mis.argtypes = [C.c_int32, i64p, i32p, u32p, u8p]
        L.orc_compute_max_np.argtypes = [C.c_int32, i64p, i32p, u32p, u8p, u64p]
        L.orc_phase3_update.argtypes = [C.c_int32, u8p, u8p, i32p, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64)]
        L.orc_csr_neighbor_count.argtypes = [C.c_int32, i64p, i32p, u8p, i32p]
        L.orc_tile_graph.restype = C.c_int64
        L.orc_tile_graph.argtypes = [C.c_int32, i64p, i32p, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p]
        L.orc_tile_row_counts.restype = C.c_int64
        L.orc_tile_row_counts.argtypes = [C.c_int32, i64p, i32p, C.c_int, i64p]
        L.orc_pack_segments.argtypes = [C.c_int32, u8p, C.c_int, u64p]
        L.orc_tiled_spmv.argtypes = [C.c_int32, C.c_int, C.c_int64, i32p, u64p, i64p, u64p,
                                     i32p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        for name, args in (("orc_gnp", [C.c_int32, C.c_double, C.c_uint64]),
                           ("orc_gnp_avg_degree", [C.c_int32, C.c_double, C.c_uint64]),
                           ("orc_rmat", [C.c_int, C.c_int, C.c_uint64]),
                           ("orc_grid", [C.c_int32]),
                           ("orc_rgg", [C.c_int32, C.c_double, C.c_uint64]),
                           ("orc_petersen", []),
                           ("orc_graph_from_edges", [C.c_int32, C.c_int64, i32p, i32p])):
            fn = getattr(L, name)
            fn.restype = C.POINTER(OrcGraph)
            fn.argtypes = args
        L.orc_rgg_radius.restype = C.c_uint64
        L.orc_rgg_radius.argtypes = [C.c_int32, C.c_double]
        L.orc_check_independence.argtypes = [C.c_int32, i64p, i32p, i32p, C.c_int64,
                                             C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.orc_check_maximality.argtypes = [C.c_int32, i64p, i32p, i32p, C.c_int64,
                                           C.POINTER(C.c_int32)]
        L.orc_graph_free.argtypes = [C.POINTER(OrcGraph)]
        L.orc_checksum_bytes.restype = C.c_uint64
        L.orc_checksum_bytes.argtypes = [C.c_void_p, C.c_int64]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference library compiled from its own sources (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libtcmis_ref.so missing (make -C oracle ref)")
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_graph_create.restype = C.c_void_p
        R.ref_graph_create.argtypes = [C.c_int32, i64p, i32p]
        R.ref_graph_free.argtypes = [C.c_void_p]
        R.ref_graph_n.restype = C.c_int32
        R.ref_graph_n.argtypes = [C.c_void_p]
        R.ref_graph_nnz.restype = C.c_int64
        R.ref_graph_nnz.argtypes = [C.c_void_p]
        R.ref_graph_copy.argtypes = [C.c_void_p, i64p, i32p]
        R.ref_gen_rmat.restype = C.c_void_p
        R.ref_gen_rmat.argtypes = [C.c_int, C.c_int, C.c_uint64]
        R.ref_gen_gnp_avg.restype = C.c_void_p
        R.ref_gen_gnp_avg.argtypes = [C.c_int32, C.c_double, C.c_uint64]
        R.ref_gen_named.restype = C.c_void_p
        R.ref_gen_named.argtypes = [C.c_char_p, C.c_int32]
        R.ref_graph_from_edges.restype = C.c_void_p
        R.ref_graph_from_edges.argtypes = [C.c_int32, C.c_int64, i32p, i32p]
        R.ref_mix64.restype = C.c_uint64
        R.ref_mix64.argtypes = [C.c_uint64]
        R.ref_vertex_hash.restype = C.c_uint64
        R.ref_vertex_hash.argtypes = [C.c_uint64, C.c_uint64]
        R.ref_combine_seed.restype = C.c_uint64
        R.ref_combine_seed.argtypes = [C.c_uint64, C.c_uint64]
        R.ref_hash_to_unit.restype = C.c_double
        R.ref_hash_to_unit.argtypes = [C.c_uint64]
        R.ref_h2_priority_value.restype = C.c_uint32
        R.ref_h2_priority_value.argtypes = [C.c_double, C.c_int32, C.c_double, C.c_int]
        R.ref_h1_random.argtypes = [C.c_int32, C.c_uint64, u32p]
        R.ref_h2_degree_aware.argtypes = [C.c_void_p, C.c_uint64, C.c_int, u32p]
        R.ref_tile_graph.restype = C.c_void_p
        R.ref_tile_graph.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
        R.ref_tiled_free.argtypes = [C.c_void_p]
        R.ref_tiled_count.restype = C.c_int64
        R.ref_tiled_count.argtypes = [C.c_void_p]
        R.ref_tiled_dim.argtypes = [C.c_void_p]
        R.ref_tiled_copy.argtypes = [C.c_void_p, i32p, i32p, u64p, i64p]
        R.ref_tiled_spmv.argtypes = [C.c_void_p, u8p, C.c_int32, i32p,
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        R.ref_run_mis.argtypes = [C.c_void_p, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                  u8p, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(RefRound),
                                  C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        R.ref_run_tc_mis_tiled.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64, C.c_int,
                                           C.c_int, C.c_int, u8p, C.POINTER(C.c_int64),
                                           C.POINTER(RefRound), C.c_int, C.POINTER(C.c_int),
                                           C.POINTER(C.c_double)]
        R.ref_run_luby.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_int, u8p,
                                   C.POINTER(C.c_int64), C.POINTER(RefRound), C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double)]
        R.ref_sequential_greedy.restype = C.c_int64
        R.ref_sequential_greedy.argtypes = [C.c_void_p, u32p, u8p]
        R.ref_compute_max_np.argtypes = [C.c_void_p, u32p, u8p, u64p]
        R.ref_h3_resolution.argtypes = [C.c_void_p, u32p, u8p, u8p]
        R.ref_check_independence.argtypes = [C.c_void_p, i32p, C.c_int64, C.POINTER(C.c_int32),
                                             C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        R.ref_check_maximality.argtypes = [C.c_void_p, i32p, C.c_int64, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_int32)]
        R.ref_write_tiled.argtypes = [C.c_void_p, C.c_int32, C.c_char_p]
        _ref = R
    return _ref


# ------------------------------------------------------------------ helpers

HEURISTICS = {"h1": 0, "h2": 1, "h3": 2, "luby-fresh": 3, "luby-perm": 4}  # engine.hpp:19


def _take(gp) -> Graph:
    g = gp.contents
    n = int(g.n)
    off = np.ctypeslib.as_array(g.off, shape=(n + 1,)).copy()
    nnz = int(g.nnz)
    nbr = (np.ctypeslib.as_array(g.nbr, shape=(nnz,)).copy() if nnz
           else np.zeros(0, np.int32))
    lib().orc_graph_free(gp)
    return Graph(n, off, nbr)


def gen(kind: str, *args) -> Graph:
    """Oracle generators: rmat(scale, ef, seed), gnp_avg(n, d, seed),
    grid(side), rgg(n, d, seed), petersen()."""
    L = lib()
    fn = {"rmat": L.orc_rmat, "gnp_avg": L.orc_gnp_avg_degree, "gnp": L.orc_gnp,
          "grid": L.orc_grid, "rgg": L.orc_rgg, "petersen": L.orc_petersen}[kind]
    gp = fn(*args)
    if not gp:
        raise ValueError(f"oracle generator {kind}{args} rejected its arguments")
    return _take(gp)


def graph_from_edges(n: int, edges) -> Graph:
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    eu = np.ascontiguousarray(e[:, 0])
    ev = np.ascontiguousarray(e[:, 1])
    gp = lib().orc_graph_from_edges(n, len(e), eu, ev)
    if not gp:
        raise IndexError("edge endpoint outside [0, n)")
    return _take(gp)


def checksum(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(lib().orc_checksum_bytes(a.ctypes.data, a.nbytes))


def h1_random(n: int, seed: int) -> np.ndarray:
    p = np.zeros(max(n, 1), np.uint32)
    if lib().orc_h1_random(max(n, 1), seed, p):
        raise ValueError("h1_random requires n >= 1")
    return p[:max(n, 1)]


def h2_degree_aware(g: Graph, seed: int, scale_bits: int = 20) -> np.ndarray:
    p = np.zeros(max(g.n, 1), np.uint32)
    if lib().orc_h2_degree_aware(g.n, g.off, seed, scale_bits, p):
        raise ValueError("scale_bits must be in [8, 30]")
    return p[:g.n]


def priorities(g: Graph, heuristic: str, seed: int, scale_bits: int = 20) -> np.ndarray:
    """engine.cpp:22-33 priorities_for"""
    if heuristic == "h1":
        return h1_random(max(g.n, 1), seed)[:max(g.n, 1)]
    if heuristic in ("h2", "h3", "luby-perm"):
        return h2_degree_aware(g, seed, scale_bits)
    raise ValueError("tiled engine only runs h1/h2/h3")


def tile_row_counts(g: Graph, T: int) -> np.ndarray:
    nb = (g.n + T - 1) // T
    rt = np.zeros(max(nb, 1), np.int64)
    if lib().orc_tile_row_counts(g.n, g.off, g.nbr if g.nbr.size else np.zeros(1, np.int32),
                                 T, rt) < 0:
        raise ValueError("tile_dim must be in [1, 64]")
    return rt[:nb]


def tile_graph(g: Graph, T: int):
    """tiling.cpp:44-84 -> (tile_row, tile_col, row_bits[T*tiles], block_row_offsets)"""
    L = lib()
    nbr = g.nbr if g.nbr.size else np.zeros(1, np.int32)
    cnt = L.orc_tile_graph(g.n, g.off, nbr, T, None, None, None, None)
    if cnt < 0:
        raise ValueError("tile_dim must be in [1, 64]")
    nb = (g.n + T - 1) // T
    tr = np.zeros(max(cnt, 1), np.int32)
    tc = np.zeros(max(cnt, 1), np.int32)
    rb = np.zeros(max(cnt * T, 1), np.uint64)
    bro = np.zeros(nb + 1, np.int64)
    L.orc_tile_graph(g.n, g.off, nbr, T, tr.ctypes.data, tc.ctypes.data, rb.ctypes.data,
                     bro.ctypes.data)
    return tr[:cnt], tc[:cnt], rb[:cnt * T], bro


@dataclass
class Solve:
    state: np.ndarray        # uint8[n], 1 = InMIS, 2 = Removed
    rounds: list             # list of dict
    n_rounds: int

    @property
    def mis(self) -> np.ndarray:
        return np.flatnonzero(self.state == 1).astype(np.int32)


def luby_rounds(g: Graph, p, fresh: bool = False, seed: int = 1, T: int | None = None,
                max_rounds: int = 4096, col_counts=None) -> Solve:
    """Round-by-round oracle (engine.cpp:231-295 / 301-352).  The tile
    counters count, per round, the tiles whose block column holds a candidate
    (spmv.cpp:37-46): `col_counts` = tiles per block column of the tiling
    (default tile_graph(g, T)'s, where columns and rows count alike)."""
    L = lib()
    rt = None
    if T:
        rt = (tile_row_counts(g, T) if col_counts is None
              else np.ascontiguousarray(col_counts, np.int64))
    st = np.zeros(max(g.n, 1), np.uint8)
    rounds = (OrcRound * max_rounds)()
    nbr = g.nbr if g.nbr.size else np.zeros(1, np.int32)
    pp = None if p is None else np.ascontiguousarray(p, dtype=np.uint32)
    k = L.orc_luby_rounds(g.n, g.off, nbr, None if pp is None else pp.ctypes.data,
                          1 if fresh else 0, seed,
                          None if rt is None else rt.ctypes.data, T or 0, st, rounds,
                          max_rounds)
    if k < 0:
        raise RuntimeError(f"oracle rounds failed ({k})")
    out = [{f: int(getattr(rounds[i], f)) for f, _ in OrcRound._fields_} for i in range(k)]
    return Solve(st[:g.n], out, k)


def solve(g: Graph, heuristic: str = "h3", seed: int = 1, tile_dim: int = 16,
          scale_bits: int = 20) -> Solve:
    """What tcmis::run_mis returns (engine.cpp:354-365), restated: per-round
    stats for h1/h2/luby-*, the single collapsed iteration for h3."""
    if g.n == 0:
        return Solve(np.zeros(0, np.uint8), [], 0)
    if heuristic == "luby-fresh":
        s = luby_rounds(g, None, fresh=True, seed=seed)
        for r in s.rounds:
            r["tiles_eval"] = r["tiles_skip"] = 0
        return s
    p = priorities(g, "h2" if heuristic == "luby-perm" else heuristic, seed, scale_bits)
    if heuristic == "luby-perm":
        s = luby_rounds(g, p)
        for r in s.rounds:
            r["tiles_eval"] = r["tiles_skip"] = 0
        return s
    s = luby_rounds(g, p, T=tile_dim)
    if heuristic != "h3":
        return s
    # h3: run_h3_resolution returns the greedy MIS of the alive set; one
    # tiled_spmv + phase3 empties the graph (engine.cpp:255-258, 281-286).
    rt = tile_row_counts(g, tile_dim)
    member = s.state == 1
    seg = np.zeros(rt.size, bool)
    seg[np.flatnonzero(member) // tile_dim] = True
    ev = int(rt[seg].sum())
    mis = int(member.sum())
    r = {f: 0 for f, _ in OrcRound._fields_}
    r.update(sel=mis, rem=g.n - mis, alive=0, tiles_eval=ev, tiles_skip=int(rt.sum()) - ev)
    return Solve(s.state, [r], 1)


def greedy_mis(g: Graph, p) -> np.ndarray:
    m = np.zeros(max(g.n, 1), np.uint8)
    nbr = g.nbr if g.nbr.size else np.zeros(1, np.int32)
    lib().orc_greedy_mis(g.n, g.off, nbr, np.ascontiguousarray(p, np.uint32), m)
    return m[:g.n]


# -------------------------------------------------------- reference handles

class RefGraph:
    """A tcmis::Graph living inside the compiled reference library."""

    def __init__(self, handle):
        if not handle:
            raise RuntimeError(ref().ref_last_error().decode())
        self.h = handle

    @classmethod
    def from_csr(cls, g: Graph) -> "RefGraph":
        nbr = g.nbr if g.nbr.size else np.zeros(1, np.int32)
        return cls(ref().ref_graph_create(g.n, g.off, nbr))

    def to_csr(self) -> Graph:
        R = ref()
        n = R.ref_graph_n(self.h)
        nnz = R.ref_graph_nnz(self.h)
        off = np.zeros(n + 1, np.int64)
        nbr = np.zeros(max(nnz, 1), np.int32)
        R.ref_graph_copy(self.h, off, nbr)
        return Graph(n, off, nbr[:nnz])

    def __del__(self):
        try:
            if self.h and _ref is not None:
                _ref.ref_graph_free(self.h)
        except Exception:
            pass


def ref_run_mis(g: RefGraph, heuristic: str = "h3", seed: int = 1, tile_dim: int = 16,
                workers: int = 0, scale_bits: int = 20, max_rounds: int = 4096):
    """tcmis::run_mis on the compiled reference (engine.cpp:354-365).
    Returns (member u8[n], rounds, wall_ms)."""
    R = ref()
    n = R.ref_graph_n(g.h)
    member = np.zeros(max(n, 1), np.uint8)
    cnt = C.c_int64(0)
    rounds = (RefRound * max_rounds)()
    nr = C.c_int(0)
    ms = C.c_double(0)
    rc = R.ref_run_mis(g.h, HEURISTICS[heuristic], seed, tile_dim, workers, scale_bits, member,
                       None, C.byref(cnt), rounds, max_rounds, C.byref(nr), C.byref(ms))
    if rc:
        raise _ref_exc(rc)
    out = [{f: getattr(rounds[i], f) for f, _ in RefRound._fields_} for i in range(nr.value)]
    return member[:n], out, ms.value


class RefTiled:
    """A TiledAdjacency built by the compiled reference's tile_graph
    (tiling.cpp:44-84); `ms` is its wall time."""

    def __init__(self, g: RefGraph, tile_dim: int = 16):
        R = ref()
        ms = C.c_double(0)
        self.h = R.ref_tile_graph(g.h, tile_dim, C.byref(ms))
        if not self.h:
            raise RuntimeError("reference tile_graph failed: " + R.ref_last_error().decode())
        self.ms = ms.value
        self.tile_dim = tile_dim

    def tile_count(self) -> int:
        return int(ref().ref_tiled_count(self.h))

    def close(self):
        if self.h and _ref is not None:
            _ref.ref_tiled_free(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_run_tc_mis_tiled(g: RefGraph, tiled: RefTiled, heuristic: str = "h3", seed: int = 1,
                         workers: int = 0, scale_bits: int = 20, max_rounds: int = 4096):
    """tcmis::run_tc_mis(g, tiled, cfg) (engine.cpp:231-295) over a prebuilt
    tiling.  Returns (member u8[n], rounds, wall_ms)."""
    R = ref()
    n = R.ref_graph_n(g.h)
    member = np.zeros(max(n, 1), np.uint8)
    cnt = C.c_int64(0)
    rounds = (RefRound * max_rounds)()
    nr = C.c_int(0)
    ms = C.c_double(0)
    rc = R.ref_run_tc_mis_tiled(g.h, tiled.h, HEURISTICS[heuristic], seed, tiled.tile_dim,
                                workers, scale_bits, member, C.byref(cnt), rounds, max_rounds,
                                C.byref(nr), C.byref(ms))
    if rc:
        raise _ref_exc(rc)
    out = [{f: getattr(rounds[i], f) for f, _ in RefRound._fields_} for i in range(nr.value)]
    return member[:n], out, ms.value


def ref_run_luby(g: RefGraph, seed: int = 1, fresh: bool = False, scale_bits: int = 20,
                 workers: int = 0, max_rounds: int = 4096):
    R = ref()
    n = R.ref_graph_n(g.h)
    member = np.zeros(max(n, 1), np.uint8)
    cnt = C.c_int64(0)
    rounds = (RefRound * max_rounds)()
    nr = C.c_int(0)
    ms = C.c_double(0)
    rc = R.ref_run_luby(g.h, seed, 1 if fresh else 0, scale_bits, workers, member, C.byref(cnt),
                        rounds, max_rounds, C.byref(nr), C.byref(ms))
    if rc:
        raise _ref_exc(rc)
    out = [{f: getattr(rounds[i], f) for f, _ in RefRound._fields_} for i in range(nr.value)]
    return member[:n], out, ms.value


def _ref_exc(code: int) -> Exception:
    msg = ref().ref_last_error().decode()
    return {1: ValueError, 2: RuntimeError, 3: AssertionError, 5: IndexError}.get(
        code, RuntimeError)(msg)


# ------------------------------------------------------------- validation

def check_independence(g: Graph, mis_set):
    """validate.cpp:45-56 (C restatement): (independent, edge or None)."""
    st = np.ascontiguousarray(mis_set, np.int32)
    u, v = C.c_int32(0), C.c_int32(0)
    r = lib().orc_check_independence(g.n, g.off, g.nbr if g.nbr.size else np.zeros(1, np.int32),
                                     st if st.size else np.zeros(1, np.int32), st.size,
                                     C.byref(u), C.byref(v))
    if r < 0:
        raise ValueError("set contains a vertex id outside [0, n)")
    return bool(r), (None if r else (u.value, v.value))


def check_maximality(g: Graph, mis_set):
    st = np.ascontiguousarray(mis_set, np.int32)
    a = C.c_int32(0)
    r = lib().orc_check_maximality(g.n, g.off, g.nbr if g.nbr.size else np.zeros(1, np.int32),
                                   st if st.size else np.zeros(1, np.int32), st.size, C.byref(a))
    if r == -1:
        raise ValueError("set contains a vertex id outside [0, n)")
    if r == -2:
        raise ValueError("maximality is defined on independent sets")
    return bool(r), (None if r else a.value)


def ref_check_independence(rg, mis_set):
    """The reference's own check_independence (validate.cpp:45-56)."""
    st = np.ascontiguousarray(mis_set, np.int32)
    ind, u, v = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    rc = ref().ref_check_independence(rg.h, st if st.size else np.zeros(1, np.int32), st.size,
                                      C.byref(ind), C.byref(u), C.byref(v))
    if rc:
        raise _ref_exc(rc)
    return bool(ind.value), (None if ind.value else (u.value, v.value))


def ref_check_maximality(rg, mis_set):
    st = np.ascontiguousarray(mis_set, np.int32)
    mx, a = C.c_int32(0), C.c_int32(0)
    rc = ref().ref_check_maximality(rg.h, st if st.size else np.zeros(1, np.int32), st.size,
                                    C.byref(mx), C.byref(a))
    if rc:
        raise _ref_exc(rc)
    return bool(mx.value), (None if mx.value else a.value)


def ref_write_tiled(rg, tile_dim: int, path: str) -> None:
    """The reference's write_tiled(tile_graph(g, T)) into `path`."""
    rc = ref().ref_write_tiled(rg.h, tile_dim, path.encode())
    if rc:
        raise _ref_exc(rc)
