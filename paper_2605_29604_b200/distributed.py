"""Row-partitioned multi-GPU MIS: one process per GPU,
``torch.distributed`` (NCCL over NVLink/NVSwitch) for the per-round exchange.

Rank r owns the contiguous rows [lo_r, hi_r).  The boundaries balance the
adjacency entries (R-MAT puts its hubs at the lowest ids) and are aligned to a
multiple of 64 vertices and of the tile dimension, so every bitmap slice is
whole 32-bit words and every T x T block row / block column belongs to one
rank (the tile counters then stay rank-local: tiles in block column b = tiles
in block row b by symmetry).

Per round (the reference's bulk-synchronous round, engine.cpp:247-291):

    select own worklist          -> own candidates, bitmap slice (n_r / 32 words)
    all_gather(candidate slices) -> remote candidates marked on every rank
    pull exclusion + update      -> own removals, bitmap slice
    all_gather(removal slices)   -> remote removed keys zeroed on every rank
    all_reduce(sel, rem, alive, tiles_eval, tiles_skip)

so the MIS, the round count and every per-round statistic equal the
single-GPU solve (tests/test_distributed.py checks world sizes 2 and 3 with
gloo on CPU through the same driver; the device side is csrc/dist.cu).

Two drivers run this round:
  * ``solve_native`` -- the production path: ``tcmis_solve_partitioned``
    (csrc/partitioned.cu) runs every round from C++, each round one CUDA
    graph launch over NCCL (bitmap slices, then id lists in the late rounds);
    Python only creates the exchange (the NCCL id travels over
    torch.distributed) and makes one call per solve;
  * ``solve_partitioned`` -- the same protocol step by step from Python over
    torch.distributed, kept as the executable specification the CPU (gloo)
    tests run.
Slices are padded to the largest rank's word count (``maxw``) so one
all_gather_into_tensor moves them; rank r's slice sits at word r * maxw.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

HEURISTICS = {"h1": 0, "h2": 1, "h3": 2, "luby-perm": 4}  # fixed priorities only


def partition_rows(offsets: np.ndarray, world: int, tile_dim: int = 16) -> list[int]:
    """Edge-balanced contiguous row ranges: rank_lo[0..world], rank_lo[0] = 0,
    rank_lo[world] = n, boundaries at multiples of lcm(64, tile_dim)."""
    n = int(offsets.size - 1)
    align = 64 * tile_dim // math.gcd(64, tile_dim)
    total = int(offsets[-1])
    lo = [0]
    for r in range(1, world):
        target = total * r // world
        v = int(np.searchsorted(offsets, target, side="left"))
        # boundaries stay aligned: the last one at or below n is n // align *
        # align (n itself need not be aligned; a trailing rank may be empty)
        v = min(n // align * align, max(lo[-1], (v + align // 2) // align * align))
        lo.append(v)
    lo.append(n)
    return lo


def slice_words(rank_lo: list[int]) -> int:
    return max(1, max((rank_lo[r + 1] - rank_lo[r] + 31) // 32 for r in range(len(rank_lo) - 1)))


@dataclass
class RoundStats:
    iteration: int
    candidates_selected: int
    vertices_removed: int
    alive_remaining: int
    tiles_evaluated: int
    tiles_skipped: int


@dataclass
class PartitionedResult:
    own_state: np.ndarray            # VertexState of [lo, hi)
    rounds: list = field(default_factory=list)
    rank_lo: list = field(default_factory=list)


class GpuRank:
    """The device side of one rank (csrc/dist.cu through the C-ABI)."""

    def __init__(self, ctx, n: int, lo: int, hi: int, offsets: np.ndarray | None,
                 neighbors: np.ndarray | None, device: str, full=None, rows=None):
        """Upload rows [lo, hi) from host CSR (full offsets + the full neighbour
        array, or just the own `rows`), or cut them from a device-resident full
        graph `full` (a DeviceGraph) with no host round trip."""
        import torch

        import paper_2605_29604_b200 as tc
        self.tc, self.torch, self.ctx, self.device = tc, torch, ctx, device
        self.L = L = tc.load()
        for name, args in (
                ("tcmis_graph_upload_partition",
                 [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                  C.POINTER(C.c_void_p)]),
                ("tcmis_graph_partition",
                 [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
                ("tcmis_dist_begin", [C.c_void_p, C.c_void_p]),
                ("tcmis_dist_select", [C.c_void_p, C.c_void_p, C.c_int32]),
                ("tcmis_dist_apply", [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_int32]),
                ("tcmis_dist_update", [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
                ("tcmis_dist_state", [C.c_void_p, C.c_void_p]),
                ("tcmis_dist_h3_tiles", [C.c_void_p, C.c_void_p, C.c_void_p])):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = args
        h = C.c_void_p()
        if full is not None:
            tc._check(L.tcmis_graph_partition(full.h, lo, hi, C.byref(h)))
        else:
            off = np.ascontiguousarray(offsets, np.int64)
            if rows is None:
                rows = neighbors[off[lo]:off[hi]]
            rows = np.ascontiguousarray(rows, np.int32)
            tc._check(L.tcmis_graph_upload_partition(
                ctx.h, n, lo, hi, C.c_void_p(off.ctypes.data),
                C.c_void_p(rows.ctypes.data) if rows.size else None, C.byref(h)))
        self.g = tc.DeviceGraph(h, ctx)
        self.g.lo, self.g.hi = lo, hi  # the rows this partition holds
        self.n, self.lo, self.hi = n, lo, hi
        self.stream = torch.cuda.ExternalStream(ctx.stream, device=device)
        with torch.cuda.stream(self.stream):
            self.counts = torch.zeros(5, dtype=torch.int64, device=device)

    def close(self):
        self.g.close()

    def words_tensor(self, words: int):
        # allocated and zero-filled on the engine stream (a non-blocking
        # stream): a fill queued on torch's default stream would be unordered
        # with the engine's kernels, and the caching allocator would hand the
        # block to the next solve while the engine stream still uses it
        with self.torch.cuda.stream(self.stream):
            return self.torch.zeros(words, dtype=self.torch.int32, device=self.device)

    def begin(self, heuristic: str, seed: int, tile_dim: int, scale_bits: int):
        cfg = self.tc.EngineConfig(heuristic=HEURISTICS[heuristic], seed=seed,
                                   tile_dim=tile_dim, scale_bits=scale_bits)
        c, _ = cfg._c()
        self.tc._check(self.L.tcmis_dist_begin(self.g.h, C.byref(c)))

    def select(self, bits):
        self.tc._check(self.L.tcmis_dist_select(self.g.h, C.c_void_p(bits.data_ptr()),
                                                 bits.numel()))

    def apply(self, gathered, rank_lo, me: int, maxw: int, what: int):
        lo = np.ascontiguousarray(rank_lo, np.int32)
        self.tc._check(self.L.tcmis_dist_apply(self.g.h, C.c_void_p(gathered.data_ptr()),
                                                C.c_void_p(lo.ctypes.data), len(rank_lo) - 1,
                                                maxw, me, what))

    def update(self, bits):
        """Stream-ordered; returns this rank's counters as a device tensor."""
        self.tc._check(self.L.tcmis_dist_update(self.g.h, C.c_void_p(bits.data_ptr()),
                                                 bits.numel(),
                                                 C.c_void_p(self.counts.data_ptr())))
        return self.counts

    def h3_tiles(self):
        ev, tot = C.c_int64(0), C.c_int64(0)
        self.tc._check(self.L.tcmis_dist_h3_tiles(self.g.h, C.byref(ev), C.byref(tot)))
        return ev.value, tot.value

    def state(self) -> np.ndarray:
        out = np.zeros(max(self.hi - self.lo, 1), np.uint8)
        self.tc._check(self.L.tcmis_dist_state(self.g.h, C.c_void_p(out.ctypes.data)))
        return out[:self.hi - self.lo]

    def collective_stream(self):
        return self.torch.cuda.stream(self.stream)


def _staged(dist, t) -> bool:
    """gloo cannot run these collectives on device tensors (the single-GPU
    emulation runs of bench.py): stage through host memory."""
    return t.is_cuda and dist.get_backend() == "gloo"


def _all_gather(dist, out, inp):
    if _staged(dist, inp):
        o = out.cpu()
        dist.all_gather_into_tensor(o, inp.cpu())
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, inp)


def _all_reduce(dist, t):
    if _staged(dist, t):
        c = t.cpu()
        dist.all_reduce(c)
        t.copy_(c)
    else:
        dist.all_reduce(t)


def solve_partitioned(rank_obj, rank_lo: list[int], rank: int, world: int, dist,
                      heuristic: str = "h2", seed: int = 1, tile_dim: int = 16,
                      scale_bits: int = 20, max_rounds: int | None = None) -> PartitionedResult:
    """The per-round protocol; `rank_obj` is a GpuRank (or the CPU stand-in of
    the tests) and `dist` is torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch
    n = rank_lo[-1]
    if any(((rank_lo[r] % 64) or (rank_lo[r] % tile_dim)) and rank_lo[r] != n
           for r in range(world)):
        raise ValueError("partition boundaries must be multiples of 64 and of tile_dim")
    if heuristic not in HEURISTICS:
        raise ValueError(f"partitioned solve runs {sorted(HEURISTICS)}, not {heuristic!r}")
    maxw = slice_words(rank_lo)
    rank_obj.begin(heuristic, seed, tile_dim, scale_bits)
    mine = rank_obj.words_tensor(maxw)
    gathered = rank_obj.words_tensor(maxw * world)
    rounds = []
    cap = max_rounds or max(n, 1)
    def enqueue_round():
        rank_obj.select(mine)
        _all_gather(dist, gathered, mine)
        rank_obj.apply(gathered, rank_lo, rank, maxw, 0)
        counts = rank_obj.update(mine)
        _all_gather(dist, gathered, mine)
        rank_obj.apply(gathered, rank_lo, rank, maxw, 1)
        t = (counts.clone() if torch.is_tensor(counts)
             else torch.tensor(counts, dtype=torch.int64, device=mine.device))
        _all_reduce(dist, t)
        return t

    with rank_obj.collective_stream():
        if not mine.is_cuda:
            for it in range(1, cap + 1):
                sel, rem, alive, ev, sk = (int(x) for x in enqueue_round().tolist())
                rounds.append(RoundStats(it, sel, rem, alive, ev, sk))
                if alive == 0:
                    break
            else:
                raise RuntimeError("iteration cap exceeded; engine livelock")  # engine.cpp:248-249
        else:
            # the termination test lags one round: round it+1 is enqueued
            # before round it's all-reduced counters reach the host, so the host
            # never drains the stream between rounds.  After the last round
            # (alive == 0) the extra round runs on empty worklists (no-op).
            host = [torch.empty(5, dtype=torch.int64).pin_memory() for _ in range(2)]
            done = [torch.cuda.Event() for _ in range(2)]

            def launch(it):
                t = enqueue_round()
                host[it % 2].copy_(t, non_blocking=True)
                done[it % 2].record()

            launch(1)
            for it in range(1, cap + 1):
                if it < cap:
                    launch(it + 1)
                done[it % 2].synchronize()
                sel, rem, alive, ev, sk = (int(x) for x in host[it % 2].tolist())
                rounds.append(RoundStats(it, sel, rem, alive, ev, sk))
                if alive == 0:
                    break
            else:
                raise RuntimeError("iteration cap exceeded; engine livelock "  # engine.cpp:248-249
                                   f"(rounds {[tuple(vars(r).values()) for r in rounds[:8]]})")
        if heuristic == "h3":
            ev, tot = rank_obj.h3_tiles()
            t = torch.tensor([ev, tot], dtype=torch.int64, device=mine.device)
            _all_reduce(dist, t)
            rounds = collapse_h3(rounds, n, int(t[0]), int(t[1]))
    return PartitionedResult(rank_obj.state(), rounds, rank_lo)


def collapse_h3(rounds: list, n: int, tiles_evaluated: int, total_tiles: int) -> list:
    """h3 reports the whole resolution as one iteration (engine.cpp:255-258)."""
    sel = sum(r.candidates_selected for r in rounds)
    return [RoundStats(1, sel, n - sel, 0, tiles_evaluated, total_tiles - tiles_evaluated)]


def solve_partitioned_local(ranks: list, rank_lo: list[int], heuristic: str = "h2",
                            seed: int = 1, tile_dim: int = 16, scale_bits: int = 20):
    """The same protocol as solve_partitioned with all `world` ranks in one
    process (one GPU): the collectives become device copies.  Used to test
    the device side of the partitioned solve on the single-GPU test box."""
    import torch
    world = len(ranks)
    n = rank_lo[-1]
    maxw = slice_words(rank_lo)
    for r in ranks:
        r.begin(heuristic, seed, tile_dim, scale_bits)
    mine = [r.words_tensor(maxw) for r in ranks]
    gathered = ranks[0].words_tensor(maxw * world)
    rounds = []
    for it in range(1, max(n, 1) + 1):
        for r, m in zip(ranks, mine):
            r.select(m)
        torch.cuda.synchronize()
        gathered.copy_(torch.cat(mine))
        torch.cuda.synchronize()  # the copy ran on torch's stream, apply on the engine's
        for k, r in enumerate(ranks):
            r.apply(gathered, rank_lo, k, maxw, 0)
        for r, m in zip(ranks, mine):
            r.update(m)
        torch.cuda.synchronize()
        counts = sum(r.counts.cpu() for r in ranks)
        gathered.copy_(torch.cat(mine))
        torch.cuda.synchronize()
        for k, r in enumerate(ranks):
            r.apply(gathered, rank_lo, k, maxw, 1)
        sel, rem, alive, ev, sk = (int(x) for x in counts)
        rounds.append(RoundStats(it, sel, rem, alive, ev, sk))
        if alive == 0:
            break
    if heuristic == "h3":
        ev = tot = 0
        for r in ranks:
            e, t = r.h3_tiles()
            ev, tot = ev + e, tot + t
        rounds = collapse_h3(rounds, n, ev, tot)
    state = np.concatenate([r.state() for r in ranks])
    return state, rounds


# --------------------------------------------------------- native driver

class Exchange:
    """A tcmis_exchange handle (include/tcmis_b200.h)."""

    def __init__(self, h):
        import paper_2605_29604_b200 as tc
        self.tc, self.h = tc, h

    @classmethod
    def nccl(cls, ctx, world: int, rank: int, dist=None, unique_id: bytes | None = None):
        """One communicator per rank: rank 0's ncclGetUniqueId is broadcast over
        ``dist`` (torch.distributed, any backend) unless ``unique_id`` is given."""
        import paper_2605_29604_b200 as tc
        L = tc.load()
        if unique_id is None:
            buf = (C.c_uint8 * 128)()
            if rank == 0:
                tc._check(L.tcmis_nccl_unique_id(buf))
            if dist is not None and world > 1:
                import torch
                t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
                if dist.get_backend() == "nccl":
                    t = t.cuda()
                dist.broadcast(t, 0)
                buf = (C.c_uint8 * 128)(*t.cpu().tolist())
        else:
            buf = (C.c_uint8 * 128)(*unique_id)
        h = C.c_void_p()
        tc._check(L.tcmis_exchange_nccl(ctx.h, world, rank, buf, C.byref(h)))
        return cls(h)

    @classmethod
    def local_group(cls, world: int) -> list:
        """world handles of one in-process group (one host thread per rank)."""
        import paper_2605_29604_b200 as tc
        arr = (C.c_void_p * world)()
        tc._check(tc.load().tcmis_exchange_local_group(world, arr))
        return [cls(C.c_void_p(arr[r])) for r in range(world)]

    def abort(self):
        self.tc.load().tcmis_exchange_abort(self.h)

    def close(self):
        if self.h:
            self.tc.load().tcmis_exchange_destroy(self.h)
            self.h = None


@dataclass
class NativeResult:
    state: np.ndarray      # final VertexState of all n vertices
    mis: np.ndarray        # ascending ids of the whole MIS
    rounds: list           # RoundStats (counters summed over the ranks)
    phase_ms: list         # this rank's (phase1, phase2, phase3) per iteration


def solve_native(part, exchange: Exchange, rank_lo: list[int], heuristic: str = "h2",
                 seed: int = 1, tile_dim: int = 16, scale_bits: int = 20,
                 want_state: bool = True, own_range: bool = False, mis_out=None) -> NativeResult:
    """One rank's whole partitioned solve (tcmis_solve_partitioned); ``part`` is
    the rank's DeviceGraph of rows (GpuRank.g).  own_range: MIS ids and states
    of this rank's rows only (TCMIS_F_OWN_RANGE); mis_out: a caller-owned
    (e.g. pinned) int32 buffer for the ids."""
    import paper_2605_29604_b200 as tc
    if heuristic not in HEURISTICS:
        raise ValueError(f"partitioned solve runs {sorted(HEURISTICS)}, not {heuristic!r}")
    L = tc.load()
    cfg = tc.EngineConfig(heuristic=HEURISTICS[heuristic], seed=seed, tile_dim=tile_dim,
                          scale_bits=scale_bits)
    c, keep = cfg._c()
    if own_range:
        c.flags |= tc.F_OWN_RANGE
    n = rank_lo[-1]
    lo = np.ascontiguousarray(rank_lo, np.int32)
    state = np.zeros(max(n, 1), np.uint8)
    mis = mis_out if mis_out is not None else np.zeros(max(n, 1), np.int32)
    cnt = C.c_int64(0)
    cap = 4096
    stats = (tc._Stats * cap)()
    nit = C.c_int32(0)
    tc._check(L.tcmis_solve_partitioned(part.h, exchange.h, C.c_void_p(lo.ctypes.data),
                                        len(rank_lo) - 1, C.byref(c),
                                        C.c_void_p(state.ctypes.data) if want_state else None,
                                        C.c_void_p(mis.ctypes.data), C.byref(cnt), stats, cap,
                                        C.byref(nit)))
    del keep
    rounds, phases = [], []
    for i in range(min(nit.value, cap)):
        s = stats[i]
        rounds.append(RoundStats(s.iteration, s.candidates_selected, s.vertices_removed,
                                 s.alive_remaining, s.tiles_evaluated, s.tiles_skipped))
        phases.append((s.phase1_ms, s.phase2_ms, s.phase3_ms))
    ns = (part_range(part)[1] - part_range(part)[0]) if own_range else n
    return NativeResult(state[:ns] if want_state else None,
                        mis[:cnt.value] if mis_out is not None else mis[:cnt.value].copy(),
                        rounds, phases)


def part_range(part) -> tuple:
    return part.lo, part.hi


def native_profile(part) -> dict:
    """Host-side profile of the rank's last native solve (tcmis_partitioned_profile)."""
    import paper_2605_29604_b200 as tc
    out = (C.c_double * 6)()
    tc._check(tc.load().tcmis_partitioned_profile(part.h, out))
    r = max(1.0, out[0])
    return {"rounds": int(out[0]), "enqueue_us_per_round": round(out[1] / r, 2),
            "wait_us_per_round": round(out[2] / r, 2),
            "round_loop_us_per_round": round(out[3] / r, 2), "list_rounds": int(out[4]),
            "tail_rounds": int(out[5])}


def solve_native_local(ranks: list, rank_lo: list[int], **kw) -> list:
    """All ranks of one process (a GpuRank each, e.g. all on cuda:0), one host
    thread per rank through an in-process exchange group; returns every rank's
    NativeResult."""
    import threading
    xs = Exchange.local_group(len(ranks))
    out: list = [None] * len(ranks)
    err: list = [None] * len(ranks)

    def run(k):
        try:
            out[k] = solve_native(ranks[k].g, xs[k], rank_lo, **kw)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            err[k] = e
            xs[k].abort()

    th = [threading.Thread(target=run, args=(k,)) for k in range(len(ranks))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for x in xs:
        x.close()
    for e in err:
        if e is not None:
            raise e
    return out
