"""B200-native TC-MIS (arXiv 2605.29604): the host-side mirror of the
reference's MIS interface over the C-ABI of ``include/tcmis_b200.h``.

Names and argument meaning follow ``/root/reference/proj/include/tcmis``
(``run_mis``, ``run_tc_mis``, ``EngineConfig``, ``MISResult``,
``IterationStats``, ``Heuristic``, ``tile_graph``, ``h1_random``,
``h2_degree_aware`` ...).  Every compute call goes through
``libtcmis_b200.so`` (hand-written sm_100a kernels); there is no CPU path --
without the library or a CUDA device the calls raise.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

__all__ = [
    "Heuristic", "VertexState", "Exclusion", "EngineConfig", "IterationStats", "MISResult",
    "Graph", "Context", "DeviceGraph", "run_mis", "run_tc_mis", "tile_graph", "h1_random",
    "h2_degree_aware", "compute_max_np", "tiled_spmv", "csr_neighbor_count", "LogicError",
    "CudaError", "load", "library_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtcmis_b200.so")
_lib = None


def library_path() -> str:
    return _LIB_PATH


class LogicError(RuntimeError):
    """std::logic_error of the reference (engine.cpp:152-153, 224-225)."""


class CudaError(RuntimeError):
    """CUDA failure or no usable sm_100 device (there is no CPU fallback)."""


class Heuristic(enum.IntEnum):  # engine.hpp:19
    H1 = 0
    H2 = 1
    H3 = 2
    LubyFresh = 3
    LubyPerm = 4


_NAMES = {Heuristic.H1: "h1", Heuristic.H2: "h2", Heuristic.H3: "h3",
          Heuristic.LubyFresh: "luby-fresh", Heuristic.LubyPerm: "luby-perm"}


def heuristic_name(h: Heuristic) -> str:  # engine.cpp:37-46
    return _NAMES[Heuristic(h)]


def heuristic_from_name(name: str) -> Heuristic:  # engine.cpp:48-55
    for k, v in _NAMES.items():
        if v == name:
            return k
    raise ValueError(f"unknown heuristic '{name}'")


class VertexState(enum.IntEnum):  # engine.hpp:17
    Alive = 0
    InMIS = 1
    Removed = 2


class Exclusion(enum.IntEnum):  # tcmis_exclusion
    AUTO = 0
    PUSH = 1
    CSR_PULL = 2
    TILE_BITS = 3
    TILE_MMA = 4


class _Stats(C.Structure):
    _fields_ = [("iteration", C.c_int32), ("reserved", C.c_int32),
                ("candidates_selected", C.c_int64), ("vertices_removed", C.c_int64),
                ("alive_remaining", C.c_int64), ("tiles_evaluated", C.c_int64),
                ("tiles_skipped", C.c_int64), ("phase1_ms", C.c_double),
                ("phase2_ms", C.c_double), ("phase3_ms", C.c_double)]


_OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.POINTER(C.c_uint8),
                        C.POINTER(C.c_uint8), C.c_int32)


class _Config(C.Structure):
    _fields_ = [("heuristic", C.c_int32), ("tile_dim", C.c_int32), ("seed", C.c_uint64),
                ("scale_bits", C.c_int32), ("workers", C.c_int32), ("exclusion", C.c_int32),
                ("flags", C.c_uint32), ("observer", _OBSERVER), ("observer_user", C.c_void_p)]


F_TIMING = 0x1
F_HOST_LOOP = 0x2
F_OWN_RANGE = 0x4
F_TILE_CAND = 0x8  # Phase 1 as A-up tiles x alive bitmap (csrc/tile_cand.cu)
F_TILE_UMMA = 0x10  # ... with the product on tcgen05 (csrc/tile_umma.cuh)
F_DEBUG_CORRUPT = 0x100  # test hook (include/tcmis_b200.h)


def load():
    """Load libtcmis_b200.so.  Raises if it was not built (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_2605_29604_b200.build` "
                          "(the B200 engine has no CPU path)")
    L = C.CDLL(_LIB_PATH)
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    P = C.POINTER
    sig = {
        "tcmis_last_error": (C.c_char_p, []),
        "tcmis_abi_version": (i32, []),
        "tcmis_config_init": (None, [P(_Config)]),
        "tcmis_ctx_create": (C.c_int, [i32, P(vp)]),
        "tcmis_ctx_destroy": (None, [vp]),
        "tcmis_ctx_stream": (vp, [vp]),
        "tcmis_ctx_synchronize": (C.c_int, [vp]),
        "tcmis_ctx_launches": (i64, [vp]),
        "tcmis_graph_upload": (C.c_int, [vp, i32, vp, vp, P(vp)]),
        "tcmis_graph_upload_tiled": (C.c_int, [vp, i32, vp, vp, i32, P(vp), P(i64)]),
        "tcmis_graph_wrap_device": (C.c_int, [vp, i32, i64, vp, vp, P(vp)]),
        "tcmis_graph_destroy": (None, [vp]),
        "tcmis_graph_n": (i32, [vp]),
        "tcmis_graph_nnz": (i64, [vp]),
        "tcmis_graph_device_offsets": (vp, [vp]),
        "tcmis_graph_device_neighbors": (vp, [vp]),
        "tcmis_graph_download": (C.c_int, [vp, vp, vp]),
        "tcmis_graph_tile": (C.c_int, [vp, i32, P(i64)]),
        "tcmis_graph_set_tiling": (C.c_int, [vp, i32, vp, i32, vp, i64]),
        "tcmis_graph_export_tiles": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "tcmis_graph_tile_store": (C.c_int, [vp, i32, P(i64), vp, vp, vp]),
        "tcmis_validate": (C.c_int, [vp, vp, i64, P(i32), P(i32), P(i32), P(i32), P(i32)]),
        "tcmis_priorities": (C.c_int, [vp, i32, u64, i32, vp]),
        "tcmis_solve": (C.c_int, [vp, P(_Config), vp, vp, P(i64), P(_Stats), i32, P(i32)]),
        "tcmis_solve_device": (C.c_int, [vp, P(_Config), P(vp), P(i64), P(vp), P(_Stats), i32,
                                         P(i32)]),
        "tcmis_compute_max_np": (C.c_int, [vp, vp, vp, vp]),
        "tcmis_neighbor_count": (C.c_int, [vp, vp, vp]),
        "tcmis_tiled_spmv": (C.c_int, [vp, i32, vp, i32, vp, P(i64), P(i64)]),
        "tcmis_gen_rmat": (C.c_int, [vp, i32, i32, u64, P(vp)]),
        "tcmis_gen_grid": (C.c_int, [vp, i32, P(vp)]),
        "tcmis_graph_from_edges": (C.c_int, [vp, i32, i64, vp, vp, P(vp)]),
        "tcmis_gen_rgg": (C.c_int, [vp, i32, u64, u64, P(vp)]),
        "tcmis_gen_gnp_host": (C.c_int, [i32, C.c_double, u64, P(P(i64)), P(P(i32)), P(i64)]),
        "tcmis_gen_gnp": (C.c_int, [vp, i32, C.c_double, u64, P(vp)]),
        "tcmis_free": (None, [vp]),
        "tcmis_rgg_radius": (u64, [i32, C.c_double]),
        "tcmis_graph_reorder": (C.c_int, [vp, i32, vp]),
        "tcmis_graph_permuted": (C.c_int, [vp, P(vp)]),
        "tcmis_graph_tile_cand_prepare": (C.c_int, [vp, P(_Config), P(C.c_double), P(i64)]),
        "tcmis_nccl_unique_id": (C.c_int, [vp]),
        "tcmis_exchange_nccl": (C.c_int, [vp, i32, i32, vp, P(vp)]),
        "tcmis_exchange_nccl_comm": (C.c_int, [vp, P(vp)]),
        "tcmis_exchange_local_group": (C.c_int, [i32, P(vp)]),
        "tcmis_exchange_destroy": (None, [vp]),
        "tcmis_exchange_abort": (None, [vp]),
        "tcmis_exchange_world": (i32, [vp]),
        "tcmis_exchange_rank": (i32, [vp]),
        "tcmis_partitioned_profile": (C.c_int, [vp, vp]),
        "tcmis_solve_partitioned": (C.c_int, [vp, vp, vp, i32, P(_Config), vp, vp, P(i64),
                                              P(_Stats), i32, P(i32)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = load().tcmis_last_error().decode()
    raise {1: ValueError, 2: RuntimeError, 3: LogicError, 4: CudaError, 5: IndexError}.get(
        rc, RuntimeError)(msg)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


# ------------------------------------------------------------------- types

@dataclass
class Graph:
    """Host CSR graph (graph.hpp:18-39): normalised, symmetric, sorted rows."""
    n: int
    offsets: np.ndarray
    neighbors: np.ndarray

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        self.neighbors = np.ascontiguousarray(self.neighbors, dtype=np.int32)

    def num_edges(self) -> int:
        return int(self.neighbors.size) // 2

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])


@dataclass
class IterationStats:  # engine.hpp:24-34
    iteration: int = 0
    candidates_selected: int = 0
    vertices_removed: int = 0
    alive_remaining: int = 0
    tiles_evaluated: int = 0
    tiles_skipped: int = 0
    phase1_ms: float = 0.0
    phase2_ms: float = 0.0
    phase3_ms: float = 0.0


@dataclass
class MISResult:  # engine.hpp:36-51
    mis: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    iterations: list = field(default_factory=list)
    heuristic: Heuristic = Heuristic.H3
    seed: int = 0
    state: Optional[np.ndarray] = None

    def cardinality(self) -> int:
        return int(self.mis.size)

    def phase1_ms(self) -> float:
        return sum(i.phase1_ms for i in self.iterations)

    def phase2_ms(self) -> float:
        return sum(i.phase2_ms for i in self.iterations)

    def phase3_ms(self) -> float:
        return sum(i.phase3_ms for i in self.iterations)

    def total_ms(self) -> float:
        return self.phase1_ms() + self.phase2_ms() + self.phase3_ms()

    def tiles_evaluated(self) -> int:
        return sum(i.tiles_evaluated for i in self.iterations)

    def tiles_skipped(self) -> int:
        return sum(i.tiles_skipped for i in self.iterations)


@dataclass
class EngineConfig:  # engine.hpp:53-65
    heuristic: Heuristic = Heuristic.H3
    seed: int = 1
    tile_dim: int = 16
    workers: int = 0  # accepted, ignored: the CUDA grid replaces the thread pool
    scale_bits: int = 20
    iteration_observer: Optional[Callable] = None
    exclusion: Exclusion = Exclusion.AUTO
    timing: bool = False
    host_loop: bool = False
    flags: int = 0  # extra TCMIS_F_* bits (test hooks)

    def _c(self) -> tuple:
        c = _Config()
        load().tcmis_config_init(C.byref(c))
        c.heuristic = int(self.heuristic)
        c.tile_dim = int(self.tile_dim)
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.scale_bits = int(self.scale_bits)
        c.workers = int(self.workers)
        c.exclusion = int(self.exclusion)
        c.flags = ((F_TIMING if self.timing else 0) | (F_HOST_LOOP if self.host_loop else 0)
                   | int(self.flags))
        keep = None
        if self.iteration_observer is not None:
            obs = self.iteration_observer

            def tramp(_user, it, cand, states, n):
                cv = np.ctypeslib.as_array(cand, shape=(n,)).copy()
                sv = np.ctypeslib.as_array(states, shape=(n,)).copy()
                obs(int(it), cv, sv)

            keep = _OBSERVER(tramp)
            c.observer = keep
        return c, keep


# ------------------------------------------------------------ device side

class Context:
    """One device + one stream (replaces parallel.cpp's thread pool)."""

    def __init__(self, device: int = 0):
        L = load()
        h = C.c_void_p()
        _check(L.tcmis_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device
        # shared with every graph of this context: a graph whose context is
        # gone (e.g. both finalised by one garbage-collected cycle, in either
        # order) must not call into the destroyed context
        self._alive = [True]

    @property
    def stream(self) -> int:
        return int(load().tcmis_ctx_stream(self.h) or 0)

    def launches(self) -> int:
        return int(load().tcmis_ctx_launches(self.h))

    def synchronize(self) -> None:
        _check(load().tcmis_ctx_synchronize(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            self._alive[0] = False
            load().tcmis_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class DeviceGraph:
    """A device-resident CSR graph handle (tcmis_graph)."""

    def __init__(self, handle, ctx: Context, keepalive=None):
        self.h = handle
        self.ctx = ctx
        self._ctx_alive = ctx._alive
        self._keep = keepalive

    @classmethod
    def upload(cls, g: Graph, ctx: Optional[Context] = None,
               tile_dim: Optional[int] = None) -> "DeviceGraph":
        """Host CSR -> HBM.  With tile_dim, the K1 tile count of that tiling
        runs overlapped with the upload (tcmis_graph_upload_tiled)."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        if tile_dim is None:
            _check(load().tcmis_graph_upload(ctx.h, int(g.n), _ptr(g.offsets),
                                             _ptr(g.neighbors), C.byref(h)))
        else:
            _check(load().tcmis_graph_upload_tiled(ctx.h, int(g.n), _ptr(g.offsets),
                                                   _ptr(g.neighbors), int(tile_dim),
                                                   C.byref(h), None))
        return cls(h, ctx)

    @classmethod
    def wrap_device(cls, n: int, nnz: int, d_offsets: int, d_neighbors: int,
                    ctx: Optional[Context] = None, keepalive=None) -> "DeviceGraph":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(load().tcmis_graph_wrap_device(ctx.h, int(n), int(nnz), C.c_void_p(d_offsets),
                                              C.c_void_p(d_neighbors), C.byref(h)))
        return cls(h, ctx, keepalive)

    @classmethod
    def rmat(cls, scale: int, edge_factor: int = 16, seed: int = 1,
             ctx: Optional[Context] = None) -> "DeviceGraph":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(load().tcmis_gen_rmat(ctx.h, scale, edge_factor, seed, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def gnp(cls, n: int, avg_degree: float, seed: int = 1,
            ctx: Optional[Context] = None) -> "DeviceGraph":
        """gnp_graph_avg_degree (generate.cpp:30-66) generated on the device."""
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(load().tcmis_gen_gnp(ctx.h, int(n), float(avg_degree), int(seed), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_edges(cls, n: int, edges, ctx: Optional[Context] = None) -> "DeviceGraph":
        """graph_from_edges (graph.cpp:14-41) normalised on the device."""
        ctx = ctx or default_context()
        e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
        eu, ev = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
        h = C.c_void_p()
        _check(load().tcmis_graph_from_edges(ctx.h, int(n), int(e.shape[0]), _ptr(eu), _ptr(ev),
                                             C.byref(h)))
        return cls(h, ctx, keepalive=(eu, ev))

    @classmethod
    def grid(cls, side: int, ctx: Optional[Context] = None) -> "DeviceGraph":
        ctx = ctx or default_context()
        h = C.c_void_p()
        _check(load().tcmis_gen_grid(ctx.h, side, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def rgg(cls, n: int, avg_degree: float = 3.0, seed: int = 1,
            ctx: Optional[Context] = None) -> "DeviceGraph":
        ctx = ctx or default_context()
        R = rgg_radius(n, avg_degree)
        h = C.c_void_p()
        _check(load().tcmis_gen_rgg(ctx.h, n, R, seed, C.byref(h)))
        return cls(h, ctx)

    @property
    def n(self) -> int:
        return int(load().tcmis_graph_n(self.h))

    @property
    def nnz(self) -> int:
        return int(load().tcmis_graph_nnz(self.h))

    def num_edges(self) -> int:
        return self.nnz // 2

    @property
    def device_offsets(self) -> int:
        return int(load().tcmis_graph_device_offsets(self.h) or 0)

    @property
    def device_neighbors(self) -> int:
        return int(load().tcmis_graph_device_neighbors(self.h) or 0)

    def download(self) -> Graph:
        n, nnz = self.n, self.nnz
        off = np.zeros(n + 1, np.int64)
        nbr = np.zeros(max(nnz, 1), np.int32)
        _check(load().tcmis_graph_download(self.h, _ptr(off), _ptr(nbr)))
        return Graph(n, off, nbr[:nnz])

    ORDER_NONE, ORDER_DEGREE, ORDER_SPATIAL, ORDER_GIVEN = 0, 1, 2, 3

    def reorder(self, mode: int, order: Optional[np.ndarray] = None) -> "DeviceGraph":
        """An internal vertex order for the solve kernels (tcmis_graph_reorder):
        results stay in this graph's ids and bit-identical."""
        o = None if order is None else np.ascontiguousarray(order, np.int32)
        _check(load().tcmis_graph_reorder(self.h, int(mode), _ptr(o)))
        return self

    def permuted(self) -> "DeviceGraph":
        """A new graph whose ids are this graph's internal order (tcmis_graph_permuted)."""
        h = C.c_void_p()
        _check(load().tcmis_graph_permuted(self.h, C.byref(h)))
        return DeviceGraph(h, self.ctx)

    def tile_cand_prepare(self, cfg: "EngineConfig") -> tuple:
        """The A-up tile store of cfg's priorities (TCMIS_F_TILE_CAND):
        (build ms, 0 when cached; tile count)."""
        c, _k = cfg._c()
        ms, tiles = C.c_double(0), C.c_int64(0)
        _check(load().tcmis_graph_tile_cand_prepare(self.h, C.byref(c), C.byref(ms),
                                                   C.byref(tiles)))
        return float(ms.value), int(tiles.value)

    def tile(self, tile_dim: int = 16) -> int:
        cnt = C.c_int64(0)
        _check(load().tcmis_graph_tile(self.h, int(tile_dim), C.byref(cnt)))
        return int(cnt.value)

    def close(self) -> None:
        if getattr(self, "h", None):
            if self._ctx_alive[0]:  # else leaked: the context it frees through is gone
                load().tcmis_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rgg_radius(n: int, avg_degree: float = 3.0) -> int:
    return int(load().tcmis_rgg_radius(int(n), float(avg_degree)))


def gnp_graph_avg_degree(n: int, avg_degree: float, seed: int) -> Graph:
    """generate.cpp:63-66 (host; the G(n,p) gap stream is serial)."""
    L = load()
    po, pn = C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    nnz = C.c_int64(0)
    _check(L.tcmis_gen_gnp_host(int(n), float(avg_degree), int(seed), C.byref(po), C.byref(pn),
                                C.byref(nnz)))
    try:
        off = np.ctypeslib.as_array(po, shape=(n + 1,)).copy()
        nbr = (np.ctypeslib.as_array(pn, shape=(nnz.value,)).copy() if nnz.value
               else np.zeros(0, np.int32))
    finally:
        L.tcmis_free(C.cast(po, C.c_void_p))
        L.tcmis_free(C.cast(pn, C.c_void_p))
    return Graph(n, off, nbr)


# ------------------------------------------------------------- engine API

def _as_device(g, ctx=None) -> DeviceGraph:
    if isinstance(g, DeviceGraph):
        return g
    return DeviceGraph.upload(g, ctx)


MAX_STATS = 1 << 16


def _solve(dg: DeviceGraph, cfg: EngineConfig, want_state: bool = True) -> MISResult:
    L = load()
    c, keep = cfg._c()
    n = dg.n
    state = np.zeros(max(n, 1), np.uint8)
    mis = np.zeros(max(n, 1), np.int32)
    cnt = C.c_int64(0)
    stats = (_Stats * 4096)()
    nit = C.c_int32(0)
    _check(L.tcmis_solve(dg.h, C.byref(c), _ptr(state) if want_state else None, _ptr(mis),
                         C.byref(cnt), stats, 4096, C.byref(nit)))
    del keep
    its = []
    for i in range(min(nit.value, 4096)):
        s = stats[i]
        its.append(IterationStats(s.iteration, s.candidates_selected, s.vertices_removed,
                                  s.alive_remaining, s.tiles_evaluated, s.tiles_skipped,
                                  s.phase1_ms, s.phase2_ms, s.phase3_ms))
    return MISResult(mis[:cnt.value].copy(), its, Heuristic(cfg.heuristic), int(cfg.seed),
                     state[:n].copy() if want_state else None)


def run_mis(g, config: Optional[EngineConfig] = None, ctx: Optional[Context] = None) -> MISResult:
    """engine.cpp:354-365: H1/H2/H3 run the tiled engine (tiling derived on the
    device), LubyFresh / LubyPerm the CSR rounds -- all on the GPU."""
    cfg = config or EngineConfig()
    return _solve(_as_device(g, ctx), cfg)


def run_tc_mis(g, tiled=None, config: Optional[EngineConfig] = None,
               ctx: Optional[Context] = None) -> MISResult:
    """engine.hpp:111-115.  ``tiled`` may be a TiledAdjacency (tuple as
    returned by tile_graph) whose block_row_offsets define the tile counters."""
    cfg = config or EngineConfig()
    if tiled is None and not 1 <= cfg.tile_dim <= 64:  # tile_graph runs first (engine.cpp:297-299)
        raise ValueError(f"tile_dim must be in [1, 64], got {cfg.tile_dim}")
    dg = _as_device(g, ctx)
    if tiled is not None and tiled.n != dg.n:  # engine.cpp:233-234
        raise ValueError("tiled adjacency built for a different graph")
    if dg.n == 0:  # engine.cpp:240
        return MISResult(heuristic=cfg.heuristic, seed=cfg.seed)
    if cfg.heuristic not in (Heuristic.H1, Heuristic.H2, Heuristic.H3):  # engine.cpp:29-31
        raise ValueError("tiled engine only runs h1/h2/h3; use run_luby_reference")
    if tiled is not None:
        if cfg.heuristic != Heuristic.H1 and not 8 <= cfg.scale_bits <= 30:
            raise ValueError("scale_bits must be in [8, 30]")
        if not 1 <= cfg.tile_dim <= 64:  # pack_vector(cfg.tile_dim), tiling.cpp:87
            raise ValueError(f"tile_dim must be in [1, 64], got {cfg.tile_dim}")
        if tiled.tile_dim != cfg.tile_dim:  # spmv.cpp:22-24, raised in round 1
            raise ValueError("tiled adjacency and vector disagree on tile layout")
        bro = np.ascontiguousarray(tiled.block_row_offsets, np.int64)
        tcol = np.ascontiguousarray(tiled.tile_col, np.int32)
        _check(load().tcmis_graph_set_tiling(dg.h, int(tiled.tile_dim), _ptr(bro),
                                             int(bro.size - 1), _ptr(tcol), int(tcol.size)))
    return _solve(dg, cfg)


@dataclass
class TiledAdjacency:  # tiling.hpp:17-44
    tile_dim: int
    n: int
    n_padded: int
    tile_row: np.ndarray
    tile_col: np.ndarray
    row_bits: np.ndarray
    block_row_offsets: np.ndarray

    def tile_count(self) -> int:
        return int(self.tile_col.size)

    def n_block_rows(self) -> int:
        return int(self.block_row_offsets.size - 1)


def tile_graph(g, tile_dim: int = 16, ctx: Optional[Context] = None) -> TiledAdjacency:
    """tiling.cpp:44-84 on the device (K1), exported in the reference layout."""
    if not 1 <= tile_dim <= 64:
        raise ValueError(f"tile_dim must be in [1, 64], got {tile_dim}")
    dg = _as_device(g, ctx)
    cnt = dg.tile(tile_dim)
    nb = (dg.n + tile_dim - 1) // tile_dim
    tr = np.zeros(max(cnt, 1), np.int32)
    tc = np.zeros(max(cnt, 1), np.int32)
    rb = np.zeros(max(cnt * tile_dim, 1), np.uint64)
    bro = np.zeros(nb + 1, np.int64)
    _check(load().tcmis_graph_export_tiles(dg.h, tile_dim, _ptr(tr), _ptr(tc), _ptr(rb),
                                           _ptr(bro)))
    return TiledAdjacency(tile_dim, dg.n, nb * tile_dim, tr[:cnt], tc[:cnt], rb[:cnt * tile_dim],
                          bro)


def _check_set(g, mis_set, ctx=None):
    dg = _as_device(g, ctx)
    st = np.ascontiguousarray(mis_set, np.int32)
    r = [C.c_int32(0) for _ in range(5)]
    _check(load().tcmis_validate(dg.h, _ptr(st), st.size, *[C.byref(x) for x in r]))
    return [x.value for x in r]


def check_independence(g, mis_set, ctx: Optional[Context] = None):
    """validate.cpp:45-56 on the device: (independent, violating_edge or None)."""
    ind, u, v, _, _ = _check_set(g, mis_set, ctx)
    return bool(ind), (None if ind else (u, v))


def check_maximality(g, mis_set, ctx: Optional[Context] = None):
    """validate.cpp:58-75 on the device: (maximal, addable_vertex or None);
    ValueError for a set that is not independent."""
    ind, _, _, mx, a = _check_set(g, mis_set, ctx)
    if not ind:
        raise ValueError("maximality is defined on independent sets")
    return bool(mx), (None if mx else a)


def tile_store(g, tile_dim: int = 16, ctx: Optional[Context] = None):
    """The compact device tile store (T = 8 / 16) the tile-form exclusion
    kernels read: (block_row_offsets, tile_col, rows) with rows[t, i] the T
    bits of row i of tile t."""
    dg = _as_device(g, ctx)
    cnt = C.c_int64(0)
    L = load()
    _check(L.tcmis_graph_tile_store(dg.h, tile_dim, C.byref(cnt), None, None, None))
    nb = (dg.n + tile_dim - 1) // tile_dim
    bro = np.zeros(nb + 1, np.int64)
    col = np.zeros(max(cnt.value, 1), np.int32)
    rows = np.zeros((max(cnt.value, 1), tile_dim), np.uint16 if tile_dim == 16 else np.uint8)
    _check(L.tcmis_graph_tile_store(dg.h, tile_dim, C.byref(cnt), _ptr(bro), _ptr(col),
                                    _ptr(rows)))
    return bro, col[:cnt.value], rows[:cnt.value]


def _priorities(g, heuristic: Heuristic, seed: int, scale_bits: int, ctx=None) -> np.ndarray:
    dg = _as_device(g, ctx)
    n = max(dg.n, 1) if heuristic == Heuristic.H1 else dg.n
    p = np.zeros(max(n, 1), np.uint32)
    _check(load().tcmis_priorities(dg.h, int(heuristic), int(seed), int(scale_bits), _ptr(p)))
    return p[:n]


def h1_random(g, seed: int, ctx=None) -> np.ndarray:
    """priorities.cpp:33-41 on the device (for the graph's n vertices)."""
    return _priorities(g, Heuristic.H1, seed, 20, ctx)


def h2_degree_aware(g, seed: int, scale_bits: int = 20, ctx=None) -> np.ndarray:
    """priorities.cpp:53-67 on the device."""
    return _priorities(g, Heuristic.H2, seed, scale_bits, ctx)


def compute_max_np(g, p: np.ndarray, states: np.ndarray, ctx=None) -> np.ndarray:
    """engine.cpp:86-103 on the device."""
    dg = _as_device(g, ctx)
    p = np.ascontiguousarray(p, np.uint32)
    s = np.ascontiguousarray(states, np.uint8)
    out = np.zeros(max(dg.n, 1), np.uint64)
    _check(load().tcmis_compute_max_np(dg.h, _ptr(p), _ptr(s), _ptr(out)))
    return out[:dg.n]


def csr_neighbor_count(g, candidates: np.ndarray, ctx=None) -> np.ndarray:
    """spmv.cpp:61-73 on the device."""
    dg = _as_device(g, ctx)
    c = np.ascontiguousarray(candidates, np.uint8)
    out = np.zeros(max(dg.n, 1), np.int32)
    _check(load().tcmis_neighbor_count(dg.h, _ptr(c), _ptr(out)))
    return out[:dg.n]


def tiled_spmv(g, candidates: np.ndarray, tile_dim: int = 16,
               exclusion: Exclusion = Exclusion.AUTO, ctx=None):
    """spmv.cpp:18-59 on the device: (nc, tiles_evaluated, tiles_skipped)."""
    dg = _as_device(g, ctx)
    c = np.ascontiguousarray(candidates, np.uint8)
    out = np.zeros(max(dg.n, 1), np.int32)
    ev, sk = C.c_int64(0), C.c_int64(0)
    _check(load().tcmis_tiled_spmv(dg.h, int(tile_dim), _ptr(c), int(exclusion), _ptr(out),
                                   C.byref(ev), C.byref(sk)))
    return out[:dg.n], int(ev.value), int(sk.value)
