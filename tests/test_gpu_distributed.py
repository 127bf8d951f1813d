"""GPU: the device side of the row-partitioned solve (csrc/dist.cu) with 2-4
ranks emulated in one process on the test GPU (NCCL needs one GPU per rank;
the multi-process protocol itself is covered by tests/test_distributed.py
with gloo).  Rounds, statistics and membership equal the reference's."""
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
