"""GPU: the row-partitioned solve with 2-4 ranks in one process on the test
GPU (NCCL needs one GPU per rank; the multi-process protocol itself is
covered by tests/test_distributed.py with gloo):
  * the step-wise device side (csrc/dist.cu) driven from Python;
  * the native driver tcmis_solve_partitioned (csrc/partitioned.cu) with an
    in-process exchange group (one host thread per rank), in both exchange
    formats (bitmap slices, id lists), and over a one-rank NCCL exchange.
Rounds, statistics and membership equal the reference's."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29604_b200 as tc
from paper_2605_29604_b200 import distributed as D

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("spec,heuristic", [(("rmat", 12, 16, 1), "h2"),
                                            (("rmat", 11, 8, 4), "h3"),
                                            (("grid", 64), "h1"),
                                            (("gnp_avg", 5000, 12.0, 3), "luby-perm")])
def test_partitioned_device_side(world, spec, heuristic):
    g = O.gen(*spec)
    rank_lo = D.partition_rows(g.off, world, 16)
    ranks = [D.GpuRank(tc.Context(0), g.n, rank_lo[r], rank_lo[r + 1], g.off, g.nbr, "cuda:0")
             for r in range(world)]
    state, rounds = D.solve_partitioned_local(ranks, rank_lo, heuristic=heuristic)
    exp = O.solve(g, heuristic, 1, tile_dim=16)
    got = [(r.candidates_selected, r.vertices_removed, r.alive_remaining, r.tiles_evaluated,
            r.tiles_skipped) for r in rounds]
    want = [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"])
            for r in exp.rounds]
    if heuristic == "luby-perm":
        want = [w[:3] + (0, 0) for w in want]
    assert got == want
    assert np.array_equal(state == 1, exp.state == 1)
    for rk in ranks:
        rk.close()


@pytest.mark.parametrize("heuristic", ["h2", "h3", "luby-perm"])
def test_partitioned_protocol_nccl_world1(heuristic):
    """The multi-process protocol itself (solve_partitioned: NCCL collectives
    on the engine stream, the one-round-lagged termination test) on a
    one-rank NCCL group -- the only NCCL group one GPU can form."""
    import torch
    import torch.distributed as dist
    g = O.gen("rmat", 13, 16, 5)
    rank_lo = D.partition_rows(g.off, 1, 16)
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1)
    try:
        torch.cuda.set_device(0)
        me = D.GpuRank(tc.Context(0), g.n, 0, g.n, g.off, g.nbr, "cuda:0")
        res = D.solve_partitioned(me, rank_lo, 0, 1, dist, heuristic=heuristic)
    finally:
        dist.destroy_process_group()
    exp = O.solve(g, heuristic, 1, tile_dim=16)
    got = [(r.candidates_selected, r.vertices_removed, r.alive_remaining, r.tiles_evaluated,
            r.tiles_skipped) for r in res.rounds]
    want = [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"])
            for r in exp.rounds]
    if heuristic == "luby-perm":
        want = [w[:3] + (0, 0) for w in want]
    assert got == want
    assert np.array_equal(res.own_state == 1, exp.state == 1)


def _want(exp, heuristic):
    want = [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"])
            for r in exp.rounds]
    return [w[:3] + (0, 0) for w in want] if heuristic == "luby-perm" else want


def _got(rounds):
    return [(r.candidates_selected, r.vertices_removed, r.alive_remaining, r.tiles_evaluated,
             r.tiles_skipped) for r in rounds]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("cap", [None, "64", "1"])
@pytest.mark.parametrize("tail", [None, "65536"])
@pytest.mark.parametrize("peer", [True, False])
@pytest.mark.parametrize("spec,heuristic", [(("rmat", 12, 16, 1), "h2"),
                                            (("rmat", 11, 8, 4), "h3"),
                                            (("grid", 64), "h1"),
                                            (("gnp_avg", 5000, 12.0, 3), "luby-perm")])
def test_native_partitioned_local_group(world, cap, tail, peer, spec, heuristic, monkeypatch):
    """tcmis_solve_partitioned, `world` ranks on cuda:0 (one host thread and
    one context each).  cap = the id-list capacity (TCMIS_PART_CAP test hook):
    None = the default rule (bitmaps on these small graphs), 64 = id lists
    from the round the alive count allows it, 1 = lists that can overflow,
    which must never be used (the alive bound keeps the slices then).
    tail: None = every round through the exchange (the default), "65536" =
    the late rounds on the gathered alive subgraph (k_tail on every rank, from
    the round after the one whose alive count fits).
    peer: the apply kernels read the other ranks' decisions in place (the
    fused exchange of an in-process group) or from all-gathered copies
    (TCMIS_PART_NO_PEER)."""
    if not peer:
        monkeypatch.setenv("TCMIS_PART_NO_PEER", "1")
    if cap is not None:
        monkeypatch.setenv("TCMIS_PART_CAP", cap)
    if tail is not None:
        monkeypatch.setenv("TCMIS_PART_TAIL", tail)
    g = O.gen(*spec)
    rank_lo = D.partition_rows(g.off, world, 16)
    ranks = [D.GpuRank(tc.Context(0), g.n, rank_lo[r], rank_lo[r + 1], g.off, g.nbr, "cuda:0")
             for r in range(world)]
    res = D.solve_native_local(ranks, rank_lo, heuristic=heuristic)
    exp = O.solve(g, heuristic, 1, tile_dim=16)
    for r in res:  # every rank holds the whole result
        assert _got(r.rounds) == _want(exp, heuristic)
        assert np.array_equal(r.mis, exp.mis)
        assert np.array_equal(r.state == 1, exp.state == 1)
        assert np.all(r.state != 0)
    if cap is None:  # the distributed form: each rank's own rows
        own = D.solve_native_local(ranks, rank_lo, heuristic=heuristic, own_range=True)
        assert np.array_equal(np.concatenate([r.mis for r in own]), exp.mis)
        assert np.array_equal(np.concatenate([r.state for r in own]) == 1, exp.state == 1)
    for rk in ranks:
        rk.close()


def test_native_partitioned_sparse_rounds_large():
    """A graph whose late rounds run on id lists by the default rule
    (n / world > 16k vertices: lists of <= maxw / 2 ids per rank)."""
    g = O.gen("gnp_avg", 100000, 16.0, 1)
    world = 2
    rank_lo = D.partition_rows(g.off, world, 16)
    ranks = [D.GpuRank(tc.Context(0), g.n, rank_lo[r], rank_lo[r + 1], g.off, g.nbr, "cuda:0")
             for r in range(world)]
    for heuristic in ("h2", "h3", "h1"):
        res = D.solve_native_local(ranks, rank_lo, heuristic=heuristic)
        exp = O.solve(g, heuristic, 1, tile_dim=16)
        assert _got(res[0].rounds) == _want(exp, heuristic)
        assert np.array_equal(res[1].mis, exp.mis)
    for rk in ranks:
        rk.close()


def test_native_partitioned_errors():
    g = O.gen("rmat", 10, 8, 1)
    rank_lo = D.partition_rows(g.off, 2, 16)
    ranks = [D.GpuRank(tc.Context(0), g.n, rank_lo[r], rank_lo[r + 1], g.off, g.nbr, "cuda:0")
             for r in range(2)]
    with pytest.raises(ValueError, match="luby-fresh|partitioned solve runs"):
        D.solve_native_local(ranks, rank_lo, heuristic="luby-fresh")
    bad = list(rank_lo)
    bad[1] += 1  # not a multiple of 64
    with pytest.raises(ValueError):
        D.solve_native_local(ranks, bad, heuristic="h2")
    for rk in ranks:
        rk.close()


@pytest.mark.parametrize("heuristic", ["h2", "h3", "luby-perm"])
@pytest.mark.parametrize("tail", [None, "65536"])
def test_native_partitioned_nccl_world1(heuristic, tail, monkeypatch):
    """tcmis_exchange_nccl on a one-rank communicator (the only NCCL group one
    GPU can form): every round one CUDA graph with the NCCL collectives
    captured in it; repeated solves re-launch the cached round graphs."""
    if tail is not None:
        monkeypatch.setenv("TCMIS_PART_TAIL", tail)
    g = O.gen("rmat", 13, 16, 5)
    rank_lo = D.partition_rows(g.off, 1, 16)
    ctx = tc.Context(0)
    me = D.GpuRank(ctx, g.n, 0, g.n, g.off, g.nbr, "cuda:0")
    x = D.Exchange.nccl(ctx, 1, 0)
    exp = O.solve(g, heuristic, 1, tile_dim=16)
    for _ in range(2):
        res = D.solve_native(me.g, x, rank_lo, heuristic=heuristic)
        assert _got(res.rounds) == _want(exp, heuristic)
        assert np.array_equal(res.mis, exp.mis)
    prof = D.native_profile(me.g)
    assert prof["rounds"] == len(exp.rounds) or heuristic == "h3"
    assert (prof["tail_rounds"] > 0) == (tail is not None and len(exp.rounds) > 2) \
        or heuristic == "h3"
    print("nccl world-1 host profile:", prof)
    x.close()
    me.close()
