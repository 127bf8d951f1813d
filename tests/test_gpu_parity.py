"""GPU parity: the sm_100a path (through the C-ABI) against the oracle and
the reference's golden fixtures.  Bit-exact on every field the reference
reports: MIS membership, |MIS|, iteration count, per-iteration
candidates_selected / vertices_removed / alive_remaining / tiles_evaluated /
tiles_skipped."""
import os

import numpy as np
import pytest

import oracle as O
import paper_2605_29604_b200 as tc
from conftest import GOLDEN, golden, golden_names

pytestmark = pytest.mark.gpu

HEUR = {"h1": tc.Heuristic.H1, "h2": tc.Heuristic.H2, "h3": tc.Heuristic.H3,
        "luby-fresh": tc.Heuristic.LubyFresh, "luby-perm": tc.Heuristic.LubyPerm}


def as_tc(g: O.Graph) -> tc.Graph:
    return tc.Graph(g.n, g.off, g.nbr)


def rounds_tuple(its):
    return [(i.candidates_selected, i.vertices_removed, i.alive_remaining, i.tiles_evaluated,
             i.tiles_skipped) for i in its]


def oracle_tuple(s):
    return [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"]) for r in s.rounds]


GRAPHS = [
    ("petersen", ()), ("gnp_avg", (1000, 8.0, 7)), ("gnp_avg", (3000, 30.0, 2)),
    ("rmat", (10, 16, 3)), ("rmat", (13, 16, 1)), ("grid", (40,)), ("rgg", (6000, 3.0, 5)),
]


@pytest.mark.parametrize("kind,args", GRAPHS)
@pytest.mark.parametrize("heur", list(HEUR))
def test_run_mis_bit_exact(ctx, kind, args, heur):
    g = O.gen(kind, *args)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    for seed in (1, 5):
        for T in (16, 8):
            exp = O.solve(g, heur, seed, tile_dim=T)
            got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=seed, tile_dim=T))
            assert np.array_equal(got.mis, exp.mis), (heur, seed, T)
            assert len(got.iterations) == exp.n_rounds
            assert rounds_tuple(got.iterations) == oracle_tuple(exp), (heur, seed, T)
            assert np.array_equal(got.state, exp.state)


@pytest.mark.parametrize("T", [1, 2, 7, 16, 31, 32, 33, 64])
def test_tile_counters_any_tile_dim(ctx, T):
    g = O.gen("rmat", 11, 8, 4)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    assert dg.tile(T) == int(O.tile_row_counts(g, T).sum())
    exp = O.solve(g, "h2", 3, tile_dim=T)
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=3, tile_dim=T))
    assert rounds_tuple(got.iterations) == oracle_tuple(exp)


@pytest.mark.parametrize("T", [1, 5, 8, 16, 32, 64])
def test_tile_graph_export_matches_oracle(ctx, T):
    g = O.gen("rmat", 10, 16, 3)
    a = tc.tile_graph(as_tc(g), T, ctx)
    tr, tcol, rb, bro = O.tile_graph(g, T)
    assert np.array_equal(a.tile_row, tr) and np.array_equal(a.tile_col, tcol)
    assert np.array_equal(a.row_bits, rb) and np.array_equal(a.block_row_offsets, bro)


@pytest.mark.parametrize("T", [1, 2, 16])
def test_tile_counts_all_row_classes(ctx, T):
    """tile_graph's per-block-row tile counts (tiling.cpp:44-84) through every
    K1 count path: light (<= 512 entries), mid (<= 2048), big (shared set,
    <= 16384) and hub rows swept in several 2^20-column windows (a 1.5M-leaf
    star at T = 1 and 2 has > 2^20 block columns)."""
    rng = np.random.default_rng(T)
    n = 1_500_000
    leaves = np.arange(1, n, dtype=np.int32)
    extra = rng.integers(0, n, size=(400_000, 2), dtype=np.int32)
    mids = np.stack([np.repeat(np.arange(2, 40, dtype=np.int32), 1500),
                     rng.integers(0, n, size=38 * 1500, dtype=np.int32)], 1)
    # vertices 5 and 6: ~20k random neighbours each, so at T = 1, 2 they are big
    # rows (8192 < entries <= 65536) swept in several 2^19-column windows
    wide = np.stack([np.repeat(np.array([5, 6], np.int32), 20_000),
                     rng.integers(0, n, size=40_000, dtype=np.int32)], 1)
    e = np.concatenate([np.stack([np.zeros(n - 1, np.int32), leaves], 1), extra, mids, wide])
    g = O.graph_from_edges(n, e)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    want = O.tile_row_counts(g, T)
    assert dg.tile(T) == int(want.sum())
    # per block row, through the reference-layout export (same K1 counts)
    a = tc.tile_graph(as_tc(g), T, ctx)
    assert np.array_equal(np.diff(a.block_row_offsets), want)
    exp = O.solve(g, "h2", 1, tile_dim=T)
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, tile_dim=T))
    assert rounds_tuple(got.iterations) == oracle_tuple(exp)


def test_tile_graph_hub_rows_split(ctx):
    # a star: one row with many block columns -> multiple work items
    n = 20000
    e = np.stack([np.zeros(n - 1, np.int32), np.arange(1, n, dtype=np.int32)], 1)
    g = O.graph_from_edges(n, e)
    for T in (16, 64):
        a = tc.tile_graph(as_tc(g), T, ctx)
        tr, tcol, rb, bro = O.tile_graph(g, T)
        assert np.array_equal(a.tile_col, tcol) and np.array_equal(a.row_bits, rb)


@pytest.mark.parametrize("heur", ["h1", "h2"])
def test_priorities_bit_exact(ctx, heur):
    for kind, args in (("rmat", (12, 16, 1)), ("gnp_avg", (5000, 3.0, 9)), ("petersen", ())):
        g = O.gen(kind, *args)
        dg = tc.DeviceGraph.upload(as_tc(g), ctx)
        for seed in (0, 1, 123456789, 2**64 - 1):
            if heur == "h1":
                assert np.array_equal(tc.h1_random(dg, seed), O.h1_random(g.n, seed))
            else:
                for sb in (8, 20, 30):
                    assert np.array_equal(tc.h2_degree_aware(dg, seed, sb),
                                          O.h2_degree_aware(g, seed, sb))


def test_h2_saturation_and_floor(ctx):
    # edgeless graph: avg = 0 -> all p = 0; tiny avg with isolated vertices ->
    # denominator floor + saturation (priorities.cpp:46-49)
    g = O.graph_from_edges(64, np.zeros((0, 2), np.int32))
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    assert np.array_equal(tc.h2_degree_aware(dg, 1, 30), O.h2_degree_aware(g, 1, 30))
    g = O.graph_from_edges(5000, np.array([[0, 1]], np.int32))
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    for sb in (8, 30):
        assert np.array_equal(tc.h2_degree_aware(dg, 7, sb), O.h2_degree_aware(g, 7, sb))
    res = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=7, scale_bits=30))
    assert np.array_equal(res.mis, O.solve(g, "h2", 7, scale_bits=30).mis)


def test_phase_helpers(ctx):
    g = O.gen("gnp_avg", 2000, 12.0, 3)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    rng = np.random.default_rng(1)
    p = O.h2_degree_aware(g, 1)
    st = rng.integers(0, 3, g.n).astype(np.uint8)
    exp = np.zeros(g.n, np.uint64)
    O.lib().orc_compute_max_np(g.n, g.off, g.nbr, p, st, exp)
    assert np.array_equal(tc.compute_max_np(dg, p, st), exp)
    c = (rng.random(g.n) < 0.1).astype(np.uint8)
    exp_nc = np.zeros(g.n, np.int32)
    O.lib().orc_csr_neighbor_count(g.n, g.off, g.nbr, c, exp_nc)
    assert np.array_equal(tc.csr_neighbor_count(dg, c), exp_nc)
    for T in (4, 16):
        tr, tcol, rb, bro = O.tile_graph(g, T)
        seg = np.zeros((g.n + T - 1) // T, np.uint64)
        O.lib().orc_pack_segments(g.n, c, T, seg)
        nc = np.zeros(g.n, np.int32)
        ev, sk = O.C.c_int64(), O.C.c_int64()
        O.lib().orc_tiled_spmv(g.n, T, tcol.size, tcol, rb, bro, seg, nc, O.C.byref(ev),
                               O.C.byref(sk))
        got, gev, gsk = tc.tiled_spmv(dg, c, T)
        assert np.array_equal(got, nc) and (gev, gsk) == (ev.value, sk.value)


def test_iteration_observer(ctx):
    g = O.gen("gnp_avg", 1000, 8.0, 7)
    p = O.h2_degree_aware(g, 1)
    seen = []

    def obs(it, cand, states):
        seen.append((it, cand.copy(), states.copy()))

    tc.run_mis(as_tc(g), tc.EngineConfig(heuristic=tc.Heuristic.H2, iteration_observer=obs))
    # replay the reference's rounds and compare the snapshots
    st = np.zeros(g.n, np.uint8)
    mx = np.zeros(g.n, np.uint64)
    for it, cand, states in seen:
        assert np.array_equal(states, st)
        O.lib().orc_compute_max_np(g.n, g.off, g.nbr, p, st, mx)
        keys = (p.astype(np.uint64) << np.uint64(32)) | (np.arange(g.n, dtype=np.uint64) + 1)
        exp_c = ((st == 0) & (keys > mx)).astype(np.uint8)
        assert np.array_equal(cand, exp_c)
        nc = np.zeros(g.n, np.int32)
        O.lib().orc_csr_neighbor_count(g.n, g.off, g.nbr, exp_c, nc)
        s, r = O.C.c_int64(), O.C.c_int64()
        O.lib().orc_phase3_update(g.n, st, exp_c, nc, O.C.byref(s), O.C.byref(r))
    assert len(seen) == 3
    seen.clear()
    res = tc.run_mis(as_tc(g), tc.EngineConfig(heuristic=tc.Heuristic.H3, iteration_observer=obs))
    assert len(seen) == 1 and seen[0][0] == 1
    assert np.array_equal(np.flatnonzero(seen[0][1]), res.mis)
    assert not seen[0][2].any()


def test_errors_match_reference(ctx):
    g = as_tc(O.gen("petersen"))
    with pytest.raises(ValueError):
        tc.run_mis(g, tc.EngineConfig(heuristic=tc.Heuristic.H2, tile_dim=0))
    with pytest.raises(ValueError):
        tc.run_mis(g, tc.EngineConfig(heuristic=tc.Heuristic.H2, tile_dim=65))
    with pytest.raises(ValueError):
        tc.run_mis(g, tc.EngineConfig(heuristic=tc.Heuristic.H2, scale_bits=7))
    with pytest.raises(ValueError):
        tc.run_mis(g, tc.EngineConfig(heuristic=tc.Heuristic.LubyPerm, scale_bits=31))
    # luby-fresh ignores scale_bits; h1 ignores it too (priorities.cpp:33-41)
    tc.run_mis(g, tc.EngineConfig(heuristic=tc.Heuristic.LubyFresh, scale_bits=99))
    tc.run_mis(g, tc.EngineConfig(heuristic=tc.Heuristic.H1, scale_bits=99))
    with pytest.raises(ValueError):
        tc.run_tc_mis(g, None, tc.EngineConfig(heuristic=tc.Heuristic.LubyPerm))
    # n == 0 returns an empty result, but a bad tile_dim still throws first
    e = tc.Graph(0, np.zeros(1, np.int64), np.zeros(0, np.int32))
    r = tc.run_mis(e, tc.EngineConfig(heuristic=tc.Heuristic.H2, scale_bits=3))
    assert r.cardinality() == 0 and r.iterations == []
    with pytest.raises(ValueError):
        tc.run_mis(e, tc.EngineConfig(tile_dim=0))


def test_prebuilt_tiles_overload(ctx):
    g = O.gen("rmat", 10, 16, 3)
    a = tc.tile_graph(as_tc(g), 8, ctx)
    res = tc.run_tc_mis(as_tc(g), a, tc.EngineConfig(heuristic=tc.Heuristic.H2, tile_dim=8))
    assert rounds_tuple(res.iterations) == oracle_tuple(O.solve(g, "h2", 1, tile_dim=8))
    with pytest.raises(ValueError):
        tc.run_tc_mis(as_tc(g), a, tc.EngineConfig(heuristic=tc.Heuristic.H2, tile_dim=16))


def test_prebuilt_tiles_any_tile_set(ctx):
    # the counters are taken on the GIVEN tiling (spmv.cpp:37-46), also when it
    # is not tile_graph(g)'s symmetric tile set: drop every third tile
    g = O.gen("rmat", 10, 16, 3)
    a = tc.tile_graph(as_tc(g), 8, ctx)
    keep = np.arange(a.tile_count()) % 3 != 0
    tr, tcol = a.tile_row[keep], a.tile_col[keep]
    nb = a.block_row_offsets.size - 1
    bro = np.zeros(nb + 1, np.int64)
    np.add.at(bro, tr + 1, 1)
    sub = tc.TiledAdjacency(tile_dim=8, n=a.n, n_padded=a.n_padded, tile_row=tr, tile_col=tcol,
                            row_bits=a.row_bits.reshape(-1, 8)[keep].reshape(-1),
                            block_row_offsets=np.cumsum(bro))
    res = tc.run_tc_mis(as_tc(g), sub, tc.EngineConfig(heuristic=tc.Heuristic.H2, tile_dim=8))
    p = O.priorities(g, "h2", 1)
    exp = O.luby_rounds(g, p, T=8, col_counts=np.bincount(tcol, minlength=nb))
    assert rounds_tuple(res.iterations) == oracle_tuple(exp)
    assert sum(i.tiles_evaluated + i.tiles_skipped for i in res.iterations) == \
        len(res.iterations) * int(keep.sum())
    bad = tc.TiledAdjacency(tile_dim=8, n=a.n, n_padded=a.n_padded, tile_row=tr,
                            tile_col=np.full_like(tcol, nb), row_bits=sub.row_bits,
                            block_row_offsets=sub.block_row_offsets)
    with pytest.raises(ValueError):
        tc.run_tc_mis(as_tc(g), bad, tc.EngineConfig(heuristic=tc.Heuristic.H2, tile_dim=8))


def test_edge_cases(ctx):
    for g in (O.graph_from_edges(1, np.zeros((0, 2), np.int32)),
              O.graph_from_edges(100, np.zeros((0, 2), np.int32)),
              O.graph_from_edges(2, np.array([[0, 1]], np.int32)),
              O.graph_from_edges(33, np.array([[i, j] for i in range(33) for j in range(i)],
                                              np.int32)),
              O.graph_from_edges(5000, np.stack([np.zeros(4999, np.int32),
                                                 np.arange(1, 5000, dtype=np.int32)], 1))):
        for heur in HEUR:
            exp = O.solve(g, heur, 2)
            got = tc.run_mis(as_tc(g), tc.EngineConfig(heuristic=HEUR[heur], seed=2))
            assert np.array_equal(got.mis, exp.mis)
            assert rounds_tuple(got.iterations) == oracle_tuple(exp)


def test_long_path_many_rounds(ctx):
    # increasing priorities along a path force ~n/2 rounds (stress for the
    # round loop and its statistics buffer)
    n = 3000
    g = O.graph_from_edges(n, np.stack([np.arange(n - 1, dtype=np.int32),
                                        np.arange(1, n, dtype=np.int32)], 1))
    exp = O.solve(g, "h1", 11)
    got = tc.run_mis(as_tc(g), tc.EngineConfig(heuristic=tc.Heuristic.H1, seed=11))
    assert np.array_equal(got.mis, exp.mis)
    assert rounds_tuple(got.iterations) == oracle_tuple(exp)


def test_repeated_solves_are_independent(ctx):
    g = O.gen("rmat", 12, 16, 2)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    first = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2))
    tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H1, seed=9))
    tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.LubyFresh, seed=3))
    again = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2))
    assert np.array_equal(first.mis, again.mis)
    assert rounds_tuple(first.iterations) == rounds_tuple(again.iterations)


# ----------------------------------------------------------- generators

@pytest.mark.parametrize("scale,ef,seed", [(8, 4, 1), (12, 16, 1), (14, 16, 3)])
def test_gpu_rmat_bit_identical(ctx, scale, ef, seed):
    dg = tc.DeviceGraph.rmat(scale, ef, seed, ctx)
    a = dg.download()
    b = O.gen("rmat", scale, ef, seed)
    assert np.array_equal(a.offsets, b.off) and np.array_equal(a.neighbors, b.nbr)


@pytest.mark.parametrize("n,avg,seed", [(0, 4.0, 1), (1, 4.0, 1), (2, 0.0, 1), (7, 10.0, 3),
                                         (50, 6.0, 2), (3000, 12.0, 2), (100000, 16.0, 1),
                                         (100000, 16.0, 7), (1 << 21, 8.0, 5), (400, 0.001, 9)])
def test_gpu_gnp_bit_identical(ctx, n, avg, seed):
    """G(n,p) (gnp_graph_avg_degree, generate.cpp:30-66) on the device: the
    counter-form SplitMix64 draws, prefix-summed pair indices and closed-form
    rows give the reference's graph exactly (the ER config is n = 100k,
    avg 16, seed 1); empty, complete (p >= 1) and near-empty corners."""
    a = tc.DeviceGraph.gnp(n, avg, seed, ctx).download()
    b = O.gen("gnp_avg", n, avg, seed)
    assert np.array_equal(a.offsets, b.off) and np.array_equal(a.neighbors, b.nbr)


def test_gpu_grid_and_rgg_match_oracle(ctx):
    for side in (1, 2, 37):
        a = tc.DeviceGraph.grid(side, ctx).download()
        b = O.gen("grid", side)
        assert np.array_equal(a.offsets, b.off) and np.array_equal(a.neighbors, b.nbr)
    for n, d, s in ((1, 3.0, 1), (5000, 3.0, 1), (20000, 6.0, 4)):
        a = tc.DeviceGraph.rgg(n, d, s, ctx).download()
        b = O.gen("rgg", n, d, s)
        assert np.array_equal(a.offsets, b.off) and np.array_equal(a.neighbors, b.nbr)


def test_host_gnp_matches_oracle():
    a = tc.gnp_graph_avg_degree(100000, 16.0, 1)
    b = O.gen("gnp_avg", 100000, 16.0, 1)
    assert np.array_equal(a.offsets, b.off) and np.array_equal(a.neighbors, b.nbr)


# ------------------------------------------------------ golden fixtures

def _device_graph_for(spec, ctx):
    k = spec["kind"]
    if k == "rmat":
        return tc.DeviceGraph.rmat(spec["scale"], spec["ef"], spec["seed"], ctx)
    if k == "grid":
        return tc.DeviceGraph.grid(spec["side"], ctx)
    if k == "rgg":
        return tc.DeviceGraph.rgg(spec["n"], spec["d"], spec["seed"], ctx)
    if k == "gnp":
        return tc.DeviceGraph.upload(tc.gnp_graph_avg_degree(spec["n"], spec["d"],
                                                             spec["seed"]), ctx)
    return tc.DeviceGraph.upload(as_tc(O.gen("petersen")), ctx)


def _check_golden(name, ctx, exclusion=tc.Exclusion.AUTO, only=None, order=None):
    gd = golden(name)
    dg = _device_graph_for(gd["spec"], ctx)
    assert (dg.n, dg.num_edges()) == (gd["n"], gd["m"])
    h = dg.download()
    assert O.checksum(h.offsets) == gd["off_checksum"]
    assert O.checksum(h.neighbors) == gd["nbr_checksum"]
    assert dg.tile(gd["tile_dim"]) == gd["tile_count"]
    del h
    if order is not None:  # the solve on an internal vertex order (tcmis_graph_reorder)
        dg.reorder(order)
    for key, exp in gd["results"].items():
        if only and key != only:
            continue
        heur, seed = key.split("/seed")
        res = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=int(seed),
                                             tile_dim=gd["tile_dim"], exclusion=exclusion))
        got = [list(t) for t in rounds_tuple(res.iterations)]
        if heur == "luby-perm":
            got = [r[:3] + [0, 0] for r in got]
        assert got == exp["rounds"], key
        assert res.cardinality() == exp["mis_size"], key
        member = (res.state == 1).astype(np.uint8)
        assert O.checksum(member) == exp["member_checksum"], key


@pytest.mark.parametrize("name", golden_names())
def test_golden_small(ctx, name):
    _check_golden(name, ctx)


@pytest.mark.parametrize("name", golden_names(large=True))
def test_golden_baseline_configs(ctx, name):
    """The BASELINE.json configs at full size, against the reference's own
    results (tests/golden/make_golden.py)."""
    _check_golden(name, ctx)


@pytest.mark.parametrize("name", golden_names(large=True))
def test_golden_baseline_configs_bench_order(ctx, name):
    """The same fixtures solved the way bench.py solves them: R-MAT on the
    degree order (sorted rows, degree-class bounds), the RGG on its points'
    spatial order, the rest on the caller's ids."""
    order = {"rmat": tc.DeviceGraph.ORDER_DEGREE,
             "rgg": tc.DeviceGraph.ORDER_SPATIAL}.get(golden(name)["spec"]["kind"])
    if order is None:
        pytest.skip("bench.py solves this config on the caller's ids")
    _check_golden(name, ctx, order=order)


def test_rmat26_golden_rounds_degree_order(ctx):
    """R-MAT s26 against the reference's fixture on the bench's degree order."""
    _check_golden("rmat26_ef16", ctx, order=tc.DeviceGraph.ORDER_DEGREE)


def test_rmat26_golden_rounds(ctx):
    """R-MAT s26 (~1.05B edges) on one GPU against tests/golden/rmat26_ef16.json
    (tests/golden/make_rmat26.py: the reference's run_luby_reference on the
    bit-identical device-generated CSR, re-pinned by its sequential greedy
    oracle; tile counters from the restatement): CSR checksums, the T=16 tile
    count, and for h2, h3, h1 and luby-perm the membership checksum, |MIS|, the
    iteration count and every round's selected / removed / alive / tiles
    evaluated / skipped."""
    gd = golden("rmat26_ef16")
    # the fixture's H2 rounds are SURVEY Appendix A's (the reference's phase functions)
    assert [r[:3] for r in gd["results"]["h2/seed1"]["rounds"]] == \
        gd["survey_appendix_a"]["h2_seed1"]["rounds_sel_rem_alive"]
    _check_golden("rmat26_ef16", ctx)


def test_rmat22_properties(ctx):
    """Size-independent properties at s22: independence and maximality of the
    result, and |MIS| == the sequential greedy count."""
    dg = tc.DeviceGraph.rmat(22, 16, 1, ctx)
    res = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2))
    h = dg.download()
    member = res.state == 1
    src = np.repeat(np.arange(h.n), np.diff(h.offsets))
    assert not np.any(member[src] & member[h.neighbors])          # independent
    covered = member.copy()
    np.logical_or.at(covered, h.neighbors, member[src])
    assert covered.all()                                            # maximal
    assert np.all(np.diff(res.mis) > 0)                             # ascending ids


EXCL = {"push": tc.Exclusion.PUSH, "pull": tc.Exclusion.CSR_PULL,
        "tile-bits": tc.Exclusion.TILE_BITS, "tile-mma": tc.Exclusion.TILE_MMA}


@pytest.mark.parametrize("kind,args", GRAPHS + [("rmat", (14, 16, 2))])
@pytest.mark.parametrize("excl", list(EXCL))
@pytest.mark.parametrize("heur", ["h1", "h2", "h3", "luby-fresh"])
def test_exclusion_forms_bit_exact(ctx, kind, args, excl, heur):
    """Every Phase-2 form (candidates push / non-candidates pull / T=16 bit
    tiles on CUDA cores / T=16 tiles on tensor cores) reproduces the
    reference's rounds exactly."""
    g = O.gen(kind, *args)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    mode = EXCL[excl]
    exp = O.solve(g, heur, 3, tile_dim=16)
    for host_loop in (False, True):
        got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=3, tile_dim=16,
                                             exclusion=mode, host_loop=host_loop))
        assert np.array_equal(got.mis, exp.mis)
        assert rounds_tuple(got.iterations) == oracle_tuple(exp)


@pytest.mark.parametrize("thr", ["0", "1", "100", "1000000000"])
def test_tail_threshold_invariance(ctx, thr, monkeypatch):
    """The persistent tail kernel (k_tail) and the per-round kernels give the
    same rounds; the switch point must not matter."""
    monkeypatch.setenv("TCMIS_TAIL_THRESHOLD", thr)
    for kind, args in (("rmat", (13, 16, 4)), ("grid", (50,)), ("gnp_avg", (4000, 12.0, 3))):
        g = O.gen(kind, *args)
        dg = tc.DeviceGraph.upload(as_tc(g), ctx)
        for heur in ("h2", "h1", "h3", "luby-fresh", "luby-perm"):
            for excl in (tc.Exclusion.PUSH, tc.Exclusion.CSR_PULL):
                exp = O.solve(g, heur, 2, tile_dim=16)
                for host_loop in (False, True):
                    got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=2,
                                                         exclusion=excl, host_loop=host_loop))
                    assert np.array_equal(got.mis, exp.mis), (kind, heur, excl, host_loop)
                    assert rounds_tuple(got.iterations) == oracle_tuple(exp)


@pytest.mark.parametrize("T", [8, 16])
def test_tile_store_matches_tile_graph(ctx, T):
    """The compact device store holds exactly tile_graph's tiles
    (tiling.cpp:44-84): same block-row offsets, columns and row bits."""
    n = 5000
    star = O.graph_from_edges(n, np.stack([np.zeros(n - 1, np.int32),
                                           np.arange(1, n, dtype=np.int32)], 1))
    for g in (O.gen("rmat", 11, 16, 2), O.gen("grid", 37), O.gen("gnp_avg", 2000, 30.0, 1),
              O.gen("rgg", 3000, 3.0, 2), star):
        bro, col, rows = tc.tile_store(as_tc(g), T, ctx)
        tr, tcol, rb, obro = O.tile_graph(g, T)
        assert np.array_equal(bro, obro)
        assert np.array_equal(col, tcol)
        assert np.array_equal(rows.reshape(-1).astype(np.uint64), rb)


@pytest.mark.parametrize("name", ["grid4096", "rmat22_ef16", "rgg24m_d3"])
@pytest.mark.parametrize("excl", ["tile-bits", "tile-mma"])
def test_golden_baseline_tile_forms(ctx, name, excl):
    """The tile-form exclusion kernels at full BASELINE size, h2, against the
    reference's golden rounds."""
    if not os.path.exists(os.path.join(GOLDEN, name + ".json")):
        pytest.skip("no golden")
    _check_golden(name, ctx, exclusion=EXCL[excl], only="h2/seed1")


@pytest.mark.parametrize("excl", ["bits", "mma"])
@pytest.mark.parametrize("T", [4, 16, 33, 64])
def test_tile_kernels_match_tiled_spmv(ctx, excl, T):
    """K4b (popcount on CUDA cores) and K4c (mma.sync s8 on tensor cores, T=16)
    reproduce tiled_spmv's counts and tile counters (spmv.cpp:18-59)."""
    if excl == "mma" and T != 16:
        pytest.skip("tensor-core tile kernel is T=16 only")
    import ctypes as C
    L = tc.load()
    L.tcmis_tiled_spmv_tiles.restype = C.c_int
    L.tcmis_tiled_spmv_tiles.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int64] + \
        [C.c_void_p] * 4 + [C.c_int32, C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    rng = np.random.default_rng(T)
    for g in (O.gen("rmat", 11, 16, 2), O.gen("grid", 40), O.gen("gnp_avg", 2000, 30.0, 1)):
        tr, tcol, rb, bro = O.tile_graph(g, T)
        for dens in (0.0, 0.05, 0.5):
            c = (rng.random(g.n) < dens).astype(np.uint8)
            seg = np.zeros((g.n + T - 1) // T, np.uint64)
            O.lib().orc_pack_segments(g.n, c, T, seg)
            nc = np.zeros(g.n, np.int32)
            ev, sk = O.C.c_int64(), O.C.c_int64()
            O.lib().orc_tiled_spmv(g.n, T, tcol.size, tcol, rb, bro, seg, nc, O.C.byref(ev),
                                   O.C.byref(sk))
            got = np.zeros(g.n, np.int32)
            gev, gsk = C.c_int64(), C.c_int64()
            mode = tc.Exclusion.TILE_MMA if excl == "mma" else tc.Exclusion.TILE_BITS
            rc = L.tcmis_tiled_spmv_tiles(ctx.h, g.n, T, tcol.size, tcol.ctypes.data,
                                          rb.ctypes.data, bro.ctypes.data, seg.ctypes.data,
                                          int(mode), got.ctypes.data, C.byref(gev), C.byref(gsk))
            assert rc == 0, L.tcmis_last_error()
            assert np.array_equal(got, nc)
            assert (gev.value, gsk.value) == (ev.value, sk.value)


@pytest.mark.parametrize("spec", [("rmat", 12, 16, 3), ("gnp_avg", 3000, 8.0, 2), ("grid", 40),
                                  ("rgg", 5000, 3.0, 1), ("petersen",)])
def test_device_validator_matches_oracle(ctx, spec):
    """check_independence / check_maximality on the device give
    the reference's answers and witnesses (oracle pinned to the reference in
    tests/test_oracle.py)."""
    g = O.gen(*spec)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx)
    rng = np.random.default_rng(3)
    s = O.solve(g, "h2", 1, tile_dim=16)
    mis = np.flatnonzero(s.state == 1).astype(np.int32)
    sets = [mis, mis[: max(0, mis.size - 3)], np.zeros(0, np.int32),
            np.concatenate([mis, rng.integers(0, g.n, 5).astype(np.int32)])]
    for st in sets:
        assert tc.check_independence(dg, st) == O.check_independence(g, st)
        if O.check_independence(g, st)[0]:
            assert tc.check_maximality(dg, st) == O.check_maximality(g, st)
        else:
            with pytest.raises(ValueError):
                tc.check_maximality(dg, st)
    with pytest.raises(ValueError):
        tc.check_independence(dg, np.array([g.n], np.int32))


def test_device_validator_on_rmat22(ctx):
    """The s22 solve validated on the device (independent and maximal)."""
    dg = tc.DeviceGraph.rmat(22, 16, 1, ctx)
    res = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2))
    assert tc.check_independence(dg, res.mis) == (True, None)
    assert tc.check_maximality(dg, res.mis) == (True, None)
    assert tc.check_maximality(dg, res.mis[1:])[0] is False


def test_graph_from_edges_on_device(ctx):
    """graph_from_edges (graph.cpp:14-41) normalised on the
    device -- symmetrised, loops dropped, duplicates merged, rows sorted --
    equals the reference restatement; out-of-range endpoints raise."""
    rng = np.random.default_rng(11)
    for n, m in ((1, 3), (7, 0), (1000, 5000), (70_000, 400_000), (1 << 17, 300_000)):
        e = rng.integers(0, n, size=(m, 2), dtype=np.int32)
        if m:
            e[: m // 10, 1] = e[: m // 10, 0]                         # self-loops
            e = np.concatenate([e, np.ascontiguousarray(e[m // 10: m // 5, ::-1])])  # reversed dups
        dg = tc.DeviceGraph.from_edges(n, e, ctx)
        want = O.graph_from_edges(n, e)
        h = dg.download()
        assert h.n == want.n
        assert np.array_equal(h.offsets, want.off)
        assert np.array_equal(h.neighbors, want.nbr)
    with pytest.raises(IndexError):
        tc.DeviceGraph.from_edges(10, np.array([[0, 10]], np.int32), ctx)


@pytest.mark.parametrize("scale,T", [(21, 16), (14, 16), (14, 8), (14, 1)])
def test_upload_tiled_counts(ctx, scale, T):
    """tcmis_graph_upload_tiled: the K1 count overlapped with a chunked upload
    (3 chunks of block rows at s21, one at s14) gives tile_graph's tiles per
    block row (tiling.cpp:44-84), and the solve's tile counters follow."""
    g = O.gen("rmat", scale, 16, 1)
    want = O.tile_row_counts(g, T)
    dg = tc.DeviceGraph.upload(as_tc(g), ctx, tile_dim=T)
    a = tc.tile_graph(dg, T)  # cached counts of the upload: no recount
    assert np.array_equal(np.diff(a.block_row_offsets), want)
    exp = O.solve(g, "h2", 1, tile_dim=T)
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, tile_dim=T))
    assert rounds_tuple(got.iterations) == oracle_tuple(exp)
    dg.close()


def test_upload_tiled_edge_cases(ctx):
    empty = tc.DeviceGraph.upload(tc.Graph(0, np.zeros(1, np.int64), np.zeros(0, np.int32)),
                                  ctx, tile_dim=16)
    assert empty.tile(16) == 0
    iso = tc.DeviceGraph.upload(tc.Graph(100, np.zeros(101, np.int64), np.zeros(0, np.int32)),
                                ctx, tile_dim=16)
    assert iso.tile(16) == 0
    r = tc.run_mis(iso, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, tile_dim=16))
    assert len(r.mis) == 100
    g = O.gen("petersen")
    for bad in (0, 65):
        with pytest.raises(Exception):
            tc.DeviceGraph.upload(as_tc(g), ctx, tile_dim=bad)


@pytest.mark.parametrize("host_loop", [False, True])
@pytest.mark.parametrize("whole", [None, "0"])
def test_phase_timers_default_path(ctx, host_loop, whole, monkeypatch):
    """The reference fills phase1/2/3_ms every round (engine.cpp:253-284):
    the default path (one CUDA graph, or the host loop) stamps %globaltimer
    per phase, so every round has a positive time and total_ms() > 0.
    whole: None = this 65k-vertex graph runs every round in k_tail (one pass
    per round: the round's time is booked as Phase 1); "0" = round 1 in the
    per-round kernels (TCMIS_TAIL_WHOLE=0)."""
    if whole is not None:
        monkeypatch.setenv("TCMIS_TAIL_WHOLE", whole)
    dg = tc.DeviceGraph.rmat(16, 16, 1, ctx)
    for heur in (tc.Heuristic.H2, tc.Heuristic.H1, tc.Heuristic.LubyPerm):
        res = tc.run_mis(dg, tc.EngineConfig(heuristic=heur, host_loop=host_loop))
        assert res.total_ms() > 0.0
        for it in res.iterations:
            assert it.phase1_ms > 0.0, (heur, it.iteration)
            assert it.phase1_ms + it.phase2_ms + it.phase3_ms < 1000.0
        if whole == "0":
            # round 1 in the per-round kernels: pull exclusion on R-MAT has
            # its own Phase 2 kernels and the update its own Phase 3
            assert res.iterations[0].phase2_ms > 0.0 and res.iterations[0].phase3_ms > 0.0
    dg.close()


@pytest.mark.parametrize("host_loop", [False, True])
@pytest.mark.parametrize("thr", ["1", "65536", "1000000000"])
def test_device_corruption_flag(ctx, host_loop, thr, monkeypatch):
    """engine.cpp:138-141,152-153: a corrupt candidate is a logic_error.  The
    device checks every round's selected + removed + alive against the alive
    count before it (round-end kernel and k_tail); TCMIS_F_DEBUG_CORRUPT starts
    the solve from a control block one vertex off, which must be reported."""
    monkeypatch.setenv("TCMIS_TAIL_THRESHOLD", thr)
    dg = as_tc(O.gen("rmat", 12, 16, 1))
    with pytest.raises(tc.LogicError):
        tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, host_loop=host_loop,
                                       flags=tc.F_DEBUG_CORRUPT))
    # and the next solve on the same graph is clean
    res = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, host_loop=host_loop))
    exp = O.solve(O.gen("rmat", 12, 16, 1), "h2", 1, tile_dim=16)
    assert np.array_equal(res.mis, exp.mis)
