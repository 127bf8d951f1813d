"""CPU: pin the oracle (plain-C restatement) against the reference compiled
from its own sources (oracle/_ref) and against the golden vectors of
SURVEY.md 8(c) / tests/golden."""
import numpy as np
import pytest

import oracle as O
from conftest import golden, golden_names

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_hash_golden_vectors():
    L = O.lib()
    assert L.orc_mix64(1) == 0x5692161D100B05E5
    assert L.orc_vertex_hash(0, 1) == 0xBFEF8030DDC2D772
    assert L.orc_vertex_hash(5, 42) == 0x3C30FC5FD50692C3
    assert L.orc_combine_seed(1, 1) == 0xDEC1469C8D51E97B
    assert L.orc_h2_priority_value(4, 4, 0.5, 20) == 559240
    assert L.orc_h2_priority_value(0.5, 0, 0.9, 20) == 536870912  # floor branch


def test_h1_h2_golden():
    assert O.h1_random(8, 1).tolist() == [3220144176, 1599417572, 1882415043, 4097900091,
                                          867839785, 2558803784, 1957514276, 798629651]
    pg = O.gen("petersen")
    assert O.h2_degree_aware(pg, 1).tolist() == [599157, 558981, 565603, 623424, 542559,
                                                 582086, 567387, 541055, 553324, 614667]


def test_petersen_all_heuristics():
    pg = O.gen("petersen")
    for h in ("h1", "h2", "h3", "luby-perm"):
        s = O.solve(pg, h)
        assert s.mis.tolist() == [0, 3, 9] and s.n_rounds == 1
    s = O.solve(pg, "luby-fresh")
    assert s.mis.tolist() == [1, 4, 7, 8] and s.n_rounds == 2


def test_gnp1000_survey_trajectory():
    g = O.gen("gnp_avg", 1000, 8.0, 7)
    s = O.solve(g, "h2", 1)
    assert [(r["sel"], r["rem"], r["alive"]) for r in s.rounds] == [
        (231, 624, 145), (64, 62, 19), (16, 3, 0)]
    assert [(r["tiles_eval"], r["tiles_skip"]) for r in s.rounds] == [
        (3385, 56), (1951, 1490), (870, 2571)]
    assert O.solve(g, "h3", 1).rounds[0]["tiles_eval"] == 3441
    assert int((O.solve(g, "h1", 1).state == 1).sum()) == 273


@needs_ref
@pytest.mark.parametrize("kind,args", [("gnp_avg", (1500, 6.0, 3)), ("rmat", (11, 8, 5)),
                                       ("grid", (33,)), ("rgg", (3000, 4.0, 2))])
@pytest.mark.parametrize("heur", ["h1", "h2", "h3", "luby-perm", "luby-fresh"])
def test_oracle_equals_reference(kind, args, heur):
    g = O.gen(kind, *args)
    rg = O.RefGraph.from_csr(g)
    for seed in (1, 9):
        for T in (8, 16):
            s = O.solve(g, heur, seed, tile_dim=T)
            m, rr, _ = O.ref_run_mis(rg, heur, seed, T, 2)
            assert np.array_equal(m, (s.state == 1).astype(np.uint8))
            assert [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"])
                    for r in rr] == [(r["sel"], r["rem"], r["alive"], r["tiles_eval"],
                                      r["tiles_skip"]) for r in s.rounds]


@needs_ref
def test_greedy_and_h3_resolution_match_reference():
    g = O.gen("rmat", 10, 16, 3)
    rg = O.RefGraph.from_csr(g)
    p = O.h2_degree_aware(g, 1)
    ref_member = np.zeros(g.n, np.uint8)
    O.ref().ref_sequential_greedy(rg.h, p, ref_member)
    assert np.array_equal(O.greedy_mis(g, p), ref_member)
    st = np.zeros(g.n, np.uint8)
    c_ref = np.zeros(g.n, np.uint8)
    O.ref().ref_h3_resolution(rg.h, p, st, c_ref)
    c = np.zeros(g.n, np.uint8)
    O.lib().orc_h3_resolution(g.n, g.off, g.nbr, p, st, c)
    assert np.array_equal(c, c_ref) and np.array_equal(c, ref_member)


@needs_ref
@pytest.mark.parametrize("T", [1, 3, 8, 16, 32, 33, 64])
def test_tile_graph_matches_reference(T):
    g = O.gen("rmat", 9, 8, 2)
    rg = O.RefGraph.from_csr(g)
    tr, tc, rb, bro = O.tile_graph(g, T)
    a = O.ref().ref_tile_graph(rg.h, T, None)
    cnt = O.ref().ref_tiled_count(a)
    assert cnt == tc.size
    rtr = np.zeros(cnt, np.int32)
    rtc = np.zeros(cnt, np.int32)
    rrb = np.zeros(cnt * T, np.uint64)
    rbro = np.zeros(bro.size, np.int64)
    O.ref().ref_tiled_copy(a, rtr, rtc, rrb, rbro)
    O.ref().ref_tiled_free(a)
    assert np.array_equal(tr, rtr) and np.array_equal(tc, rtc)
    assert np.array_equal(rb, rrb) and np.array_equal(bro, rbro)
    # tiles per block row == tiles per block column (A symmetric): the
    # shortcut the engine's tile counters rely on
    rows = np.diff(bro)
    cols = np.bincount(tc, minlength=rows.size)
    assert np.array_equal(rows, cols)
    assert np.array_equal(O.tile_row_counts(g, T), rows)


@needs_ref
def test_tiled_spmv_counters_match_reference():
    g = O.gen("gnp_avg", 700, 9.0, 4)
    rg = O.RefGraph.from_csr(g)
    rng = np.random.default_rng(0)
    for T in (4, 16, 64):
        tr, tc, rb, bro = O.tile_graph(g, T)
        a = O.ref().ref_tile_graph(rg.h, T, None)
        for dens in (0.0, 0.01, 0.2):
            c = (rng.random(g.n) < dens).astype(np.uint8)
            seg = np.zeros((g.n + T - 1) // T, np.uint64)
            O.lib().orc_pack_segments(g.n, c, T, seg)
            nc = np.zeros(g.n, np.int32)
            ev, sk = O.C.c_int64(), O.C.c_int64()
            O.lib().orc_tiled_spmv(g.n, T, tc.size, tc, rb, bro, seg, nc, O.C.byref(ev),
                                   O.C.byref(sk))
            rnc = np.zeros(g.n, np.int32)
            rev, rsk = O.C.c_int64(), O.C.c_int64()
            O.ref().ref_tiled_spmv(a, c, g.n, rnc, O.C.byref(rev), O.C.byref(rsk))
            assert np.array_equal(nc, rnc) and (ev.value, sk.value) == (rev.value, rsk.value)
            csr = np.zeros(g.n, np.int32)
            O.lib().orc_csr_neighbor_count(g.n, g.off, g.nbr, c, csr)
            assert np.array_equal(csr, nc)
        O.ref().ref_tiled_free(a)


@needs_ref
@pytest.mark.parametrize("scale,ef,seed", [(8, 4, 1), (12, 16, 1), (13, 16, 7)])
def test_rmat_generator_matches_reference(scale, ef, seed):
    a = O.gen("rmat", scale, ef, seed)
    b = O.RefGraph(O.ref().ref_gen_rmat(scale, ef, seed)).to_csr()
    assert np.array_equal(a.off, b.off) and np.array_equal(a.nbr, b.nbr)


@needs_ref
def test_gnp_generator_matches_reference():
    a = O.gen("gnp_avg", 100000, 16.0, 1)
    b = O.RefGraph(O.ref().ref_gen_gnp_avg(100000, 16.0, 1)).to_csr()
    assert np.array_equal(a.off, b.off) and np.array_equal(a.nbr, b.nbr)
    assert a.num_edges == 800026  # SURVEY 8 size sheet


@needs_ref
def test_graph_from_edges_matches_reference():
    rng = np.random.default_rng(3)
    e = rng.integers(0, 50, size=(400, 2)).astype(np.int32)
    a = O.graph_from_edges(50, e)
    b = O.RefGraph(O.ref().ref_graph_from_edges(50, len(e), np.ascontiguousarray(e[:, 0]),
                                                np.ascontiguousarray(e[:, 1]))).to_csr()
    assert np.array_equal(a.off, b.off) and np.array_equal(a.nbr, b.nbr)


@pytest.mark.parametrize("kind,args", [("grid", (17,)), ("rgg", (5000, 3.0, 1))])
def test_new_generators_are_normalised(kind, args):
    g = O.gen(kind, *args)
    assert g.off[0] == 0 and g.off[-1] == g.nbr.size
    src = np.repeat(np.arange(g.n), np.diff(g.off))
    assert np.all(src != g.nbr)
    for v in range(0, g.n, max(1, g.n // 50)):
        row = g.nbr[g.off[v]:g.off[v + 1]]
        assert np.all(np.diff(row) > 0)
    fwd = set(zip(src.tolist(), g.nbr.tolist()))
    assert all((b, a) in fwd for a, b in fwd)


@pytest.mark.parametrize("name", golden_names())
def test_oracle_against_golden_fixtures(name):
    gd = golden(name)
    spec = gd["spec"]
    if spec["kind"] == "rmat":
        g = O.gen("rmat", spec["scale"], spec["ef"], spec["seed"])
    elif spec["kind"] == "gnp":
        g = O.gen("gnp_avg", spec["n"], spec["d"], spec["seed"])
    elif spec["kind"] == "grid":
        g = O.gen("grid", spec["side"])
    elif spec["kind"] == "rgg":
        g = O.gen("rgg", spec["n"], spec["d"], spec["seed"])
    else:
        g = O.gen("petersen")
    assert (g.n, g.num_edges) == (gd["n"], gd["m"])
    assert O.checksum(g.off) == gd["off_checksum"] and O.checksum(g.nbr) == gd["nbr_checksum"]
    for key, exp in gd["results"].items():
        h, seed = key.split("/seed")
        s = O.solve(g, h, int(seed), tile_dim=gd["tile_dim"])
        assert [[r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"]]
                for r in s.rounds] == exp["rounds"], key
        assert O.checksum((s.state == 1).astype(np.uint8)) == exp["member_checksum"], key


@pytest.mark.parametrize("name", ["er_n100k_d16"])
def test_oracle_against_large_golden(name):
    if name not in golden_names(large=True):
        pytest.skip("large fixture not generated")
    test_oracle_against_golden_fixtures(name)


def _sets_for(g, rng):
    """independent+maximal (an MIS), independent non-maximal, dependent sets"""
    s = O.solve(g, "h2", 1, tile_dim=16)
    mis = np.flatnonzero(s.state == 1).astype(np.int32)
    out = [mis, mis[: max(0, mis.size - 3)], np.zeros(0, np.int32)]
    if g.nbr.size:
        v = int(rng.integers(0, g.n))
        while g.off[v + 1] == g.off[v]:
            v = int(rng.integers(0, g.n))
        out.append(np.array([v, g.nbr[g.off[v]]], np.int32))
        out.append(np.concatenate([mis, rng.integers(0, g.n, 5).astype(np.int32)]))
    return out


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("spec", [("rmat", 10, 16, 3), ("gnp_avg", 500, 6.0, 2), ("grid", 12),
                                  ("petersen",)])
def test_validate_restatement_matches_reference(spec):
    """check_independence / check_maximality (validate.cpp:45-75): the C
    restatement gives the reference's answers and witnesses."""
    g = O.gen(*spec)
    rg = O.RefGraph.from_csr(g)
    rng = np.random.default_rng(7)
    for st in _sets_for(g, rng):
        assert O.check_independence(g, st) == O.ref_check_independence(rg, st)
        ind = O.check_independence(g, st)[0]
        if ind:
            assert O.check_maximality(g, st) == O.ref_check_maximality(rg, st)
        else:
            with pytest.raises(ValueError):
                O.check_maximality(g, st)
            with pytest.raises(ValueError):
                O.ref_check_maximality(rg, st)
    with pytest.raises(ValueError):
        O.check_independence(g, np.array([g.n], np.int32))
    with pytest.raises(ValueError):
        O.ref_check_independence(rg, np.array([g.n], np.int32))
