"""GPU: Phase 1 as a tile x bit-vector product (TCMIS_F_TILE_CAND,
csrc/tile_cand.cu): the oriented adjacency A-up in the compact T = 16 store
times the round's alive bitmap -- on CUDA cores, or on the tensor cores with
TCMIS_F_TILE_UMMA (tcgen05.mma kind::i8, TMEM accumulator) -- gives
compute_max_np + generate_candidates (engine.cpp:86-119) bit for bit, so
whole solves equal the reference's."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29604_b200 as tc

pytestmark = pytest.mark.gpu

HEUR = {"h1": tc.Heuristic.H1, "h2": tc.Heuristic.H2, "h3": tc.Heuristic.H3,
        "luby-perm": tc.Heuristic.LubyPerm}


def rounds_tuple(its):
    return [(i.candidates_selected, i.vertices_removed, i.alive_remaining, i.tiles_evaluated,
             i.tiles_skipped) for i in its]


def oracle_tuple(s):
    return [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"]) for r in s.rounds]


@pytest.fixture(scope="module")
def ctx():
    return tc.Context(0)


@pytest.mark.parametrize("kind,args", [("rmat", (12, 16, 3)), ("gnp_avg", (3000, 12.0, 2)),
                                       ("grid", (45,)), ("rgg", (6000, 3.0, 5)),
                                       ("rmat", (10, 4, 7)), ("grid", (700,))])
@pytest.mark.parametrize("thr", [None, "0"])
@pytest.mark.parametrize("gate", [None, "1"])
def test_tile_phase1_bit_exact(ctx, kind, args, thr, gate, monkeypatch):
    """thr "0": no k_tail; gate "1": every round's Phase 1 through the tile
    kernels (default: the rounds starting with >= n/4 alive, CSR after)."""
    if thr is not None:
        monkeypatch.setenv("TCMIS_TAIL_THRESHOLD", thr)
    if gate is not None:
        monkeypatch.setenv("TCMIS_TILE_CAND_GATE", gate)
    g = O.gen(kind, *args)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    for heur in HEUR:
        for seed in (1, 9):
            exp = O.solve(g, heur, seed, tile_dim=16)
            for excl, umma in ((tc.Exclusion.AUTO, False), (tc.Exclusion.PUSH, False),
                               (tc.Exclusion.CSR_PULL, False), (tc.Exclusion.TILE_BITS, False),
                               (tc.Exclusion.TILE_MMA, False), (tc.Exclusion.AUTO, True),
                               (tc.Exclusion.CSR_PULL, True)):
                for host_loop in (False, True):
                    flags = tc.F_TILE_CAND | (tc.F_TILE_UMMA if umma else 0)
                    cfg = tc.EngineConfig(heuristic=HEUR[heur], seed=seed, exclusion=excl,
                                          host_loop=host_loop, flags=flags)
                    got = tc.run_mis(dg, cfg)
                    where = (kind, heur, seed, excl, umma, host_loop)
                    assert np.array_equal(got.mis, exp.mis), where
                    assert rounds_tuple(got.iterations) == oracle_tuple(exp), where
    dg.close()


def test_tile_phase1_store_cache_and_errors(ctx):
    g = O.gen("rmat", 11, 16, 1)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    cfg = tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, flags=tc.F_TILE_CAND)
    ms, tiles = dg.tile_cand_prepare(cfg)
    assert ms > 0 and tiles > 0
    assert dg.tile_cand_prepare(cfg) == (0.0, tiles)  # cached for the same priorities
    # A-up holds exactly half of the 2m entries: its tiles are a subset of A's
    assert tiles <= dg.tile(16)
    with pytest.raises(ValueError):
        tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.LubyFresh, flags=tc.F_TILE_CAND))
    exp = O.solve(g, "h1", 4, tile_dim=16)  # another configuration: rebuilt
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H1, seed=4,
                                         flags=tc.F_TILE_CAND))
    assert np.array_equal(got.mis, exp.mis)
    dg.close()
