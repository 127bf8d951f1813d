"""CPU (gloo, world sizes 2 and 3): the row-partitioned multi-GPU protocol of
paper_2605_29604_b200/distributed.py -- partitioning, padded bitmap slices,
all_gather / all_reduce per round, termination, h3 collapse -- driven with a
CPU stand-in for the per-rank device step (CpuRank below restates
csrc/dist.cu on numpy; test infrastructure), must reproduce the reference's
single-process rounds bit for bit."""
import contextlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2605_29604_b200 import distributed as D


class CpuRank:
    """numpy restatement of the per-rank device step (csrc/dist.cu)."""

    def __init__(self, g, lo, hi):
        self.g, self.lo, self.hi = g, lo, hi
        self.deg = np.diff(g.off)

    def words_tensor(self, words):
        return torch.zeros(words, dtype=torch.int32)

    def collective_stream(self):
        return contextlib.nullcontext()

    def _bit(self, bits, v):
        b = bits.numpy().view(np.uint32)
        b[(v - self.lo) >> 5] |= np.uint32(1 << ((v - self.lo) & 31))

    def begin(self, heuristic, seed, T, scale_bits):
        g = self.g
        self.T = T
        p = O.priorities(g, "h2" if heuristic in ("h3", "luby-perm") else heuristic, seed,
                         scale_bits)
        self.key = (p.astype(np.uint64) << np.uint64(32)) | (np.arange(g.n, dtype=np.uint64) + 1)
        self.st = np.zeros(g.n, np.uint8)
        self.next = np.zeros(g.n, np.uint8)
        iso = self.deg == 0
        self.next[iso] = 1
        self.st[iso] = 1
        self.seg_mode = 0 if heuristic == "luby-perm" else (2 if heuristic == "h3" else 1)
        nb = (g.n + T - 1) // T
        rt = O.tile_row_counts(g, T) if self.seg_mode else np.zeros(nb, np.int64)
        own_b = np.zeros(nb, bool)
        own_b[self.lo // T:(self.hi + T - 1) // T] = True
        self.rowtiles = np.where(own_b, rt, 0)
        self.segflag = np.zeros(nb, bool)
        if self.seg_mode:
            self.segflag[np.flatnonzero(iso) // T] = True
        own = np.arange(self.lo, self.hi)
        self.sel0 = int(iso[own].sum())
        self.wl = own[~iso[own]]
        self.first = True

    def select(self, bits):
        bits.zero_()
        g, key = self.g, self.key
        self.sel = self.sel0 if self.first else 0
        self.first = False
        self.check = []
        for v in self.wl:
            row = g.nbr[g.off[v]:g.off[v + 1]]
            if np.any(key[row] > key[v]):
                self.check.append(v)
            else:
                self.next[v] = 1
                self.st[v] = 1
                self.sel += 1
                if self.seg_mode:
                    self.segflag[v // self.T] = True
                self._bit(bits, v)

    def apply(self, gathered, rank_lo, me, maxw, what):
        b = gathered.numpy().view(np.uint32)
        for r in range(len(rank_lo) - 1):
            if r == me:
                continue
            words = b[r * maxw:(r + 1) * maxw]
            for w in np.flatnonzero(words):
                for k in range(32):
                    if words[w] >> np.uint32(k) & np.uint32(1):
                        v = rank_lo[r] + w * 32 + k
                        if what == 0:
                            self.next[v], self.st[v] = 1, 1
                        else:
                            self.key[v], self.st[v] = 0, 2

    def update(self, bits):
        bits.zero_()
        g = self.g
        rem, surv = 0, []
        for v in self.check:
            row = g.nbr[g.off[v]:g.off[v + 1]]
            if np.any(self.next[row] == 1):
                self.st[v], self.key[v] = 2, 0
                rem += 1
                self._bit(bits, v)
            else:
                surv.append(v)
        self.wl = np.array(surv, np.int64)
        ev = int(self.rowtiles[self.segflag].sum()) if self.seg_mode == 1 else 0
        sk = int(self.rowtiles.sum()) - ev if self.seg_mode == 1 else 0
        if self.seg_mode == 1:
            self.segflag[:] = False
        return np.array([self.sel, rem, len(surv), ev, sk], np.int64)

    def h3_tiles(self):
        return int(self.rowtiles[self.segflag].sum()), int(self.rowtiles.sum())

    def state(self):
        return self.st[self.lo:self.hi].copy()


def _worker(rank, world, port, spec, heuristic, seed, T, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = O.gen(*spec)
    rank_lo = D.partition_rows(g.off, world, T)
    r = CpuRank(g, rank_lo[rank], rank_lo[rank + 1])
    res = D.solve_partitioned(r, rank_lo, rank, world, dist, heuristic=heuristic, seed=seed,
                              tile_dim=T)
    states = [None] * world
    dist.all_gather_object(states, res.own_state)
    if rank == 0:
        out.put(([(x.candidates_selected, x.vertices_removed, x.alive_remaining,
                   x.tiles_evaluated, x.tiles_skipped) for x in res.rounds],
                 np.concatenate(states), rank_lo))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("spec,heuristic", [(("rmat", 9, 8, 3), "h2"), (("gnp_avg", 600, 6.0, 2),
                                                                         "h1"),
                                            (("grid", 24), "h3"), (("rmat", 9, 8, 5), "luby-perm")])
def test_partitioned_rounds_equal_single(world, spec, heuristic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spec, heuristic, 1, 16, q))
             for r in range(world)]
    for p in procs:
        p.start()
    rounds, state, rank_lo = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = O.gen(*spec)
    exp = O.solve(g, heuristic, 1, tile_dim=16)
    if heuristic == "luby-perm":
        exp_r = [(r["sel"], r["rem"], r["alive"], 0, 0) for r in exp.rounds]
    else:
        exp_r = [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"])
                 for r in exp.rounds]
    assert rounds == exp_r
    assert np.array_equal(state == 1, exp.state == 1)
    assert len(rank_lo) == world + 1 and rank_lo[0] == 0 and rank_lo[-1] == g.n


def test_partition_rows_balances_edges_and_aligns():
    g = O.gen("rmat", 12, 16, 1)
    for world in (2, 4, 8):
        lo = D.partition_rows(g.off, world, 16)
        assert lo[0] == 0 and lo[-1] == g.n
        assert all(x % 64 == 0 for x in lo[:-1])
        assert all(a <= b for a, b in zip(lo, lo[1:]))
        loads = [g.off[lo[r + 1]] - g.off[lo[r]] for r in range(world)]
        assert max(loads) < 1.6 * g.nbr.size / world  # hubs at low ids, still balanced
    assert D.partition_rows(g.off, 3, 48)[1] % 192 == 0  # lcm(64, 48)
