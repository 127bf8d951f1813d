"""GPU: an internal vertex order (tcmis_graph_reorder, csrc/order.cu) changes
nothing a caller sees.  The kernels run on a relabeled CSR, but keys, hash
priorities and tile counters stay on the caller's ids, so MIS membership,
|MIS|, the iteration count and every per-iteration statistic equal the
oracle's (and therefore the direct solve's) for every heuristic, both
exclusion forms, graph and host-loop drivers, and any tail switch point."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29604_b200 as tc

pytestmark = pytest.mark.gpu

HEUR = {"h1": tc.Heuristic.H1, "h2": tc.Heuristic.H2, "h3": tc.Heuristic.H3,
        "luby-fresh": tc.Heuristic.LubyFresh, "luby-perm": tc.Heuristic.LubyPerm}


def rounds_tuple(its):
    return [(i.candidates_selected, i.vertices_removed, i.alive_remaining, i.tiles_evaluated,
             i.tiles_skipped) for i in its]


def oracle_tuple(s):
    return [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"]) for r in s.rounds]


@pytest.fixture(scope="module")
def ctx():
    return tc.Context(0)


def _orders(g, rng):
    yield "degree", tc.DeviceGraph.ORDER_DEGREE, None
    yield "random", tc.DeviceGraph.ORDER_GIVEN, rng.permutation(g.n).astype(np.int32)
    yield "reverse", tc.DeviceGraph.ORDER_GIVEN, np.arange(g.n - 1, -1, -1, dtype=np.int32)


@pytest.mark.parametrize("kind,args", [("rmat", (12, 16, 3)), ("gnp_avg", (3000, 12.0, 2)),
                                       ("grid", (45,)), ("rmat", (10, 4, 7))])
@pytest.mark.parametrize("thr", [None, "0", "1000000000"])
@pytest.mark.parametrize("plane", [None, "0"])
def test_reordered_solves_equal_the_reference(ctx, kind, args, thr, plane, monkeypatch):
    """plane: the caller-order membership plane (None: kept, as for every
    graph up to 48M vertices) or "0" (never kept: the compaction gathers
    through the permutation, as at R-MAT s26)."""
    if thr is not None:
        monkeypatch.setenv("TCMIS_TAIL_THRESHOLD", thr)
    if plane is not None:
        monkeypatch.setenv("TCMIS_MIS_O_MAX", plane)
    g = O.gen(kind, *args)
    rng = np.random.default_rng(5)
    for name, mode, order in _orders(g, rng):
        dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx).reorder(mode, order)
        for heur in ("h2", "h1", "h3", "luby-fresh", "luby-perm"):
            exp = O.solve(g, heur, 3, tile_dim=16)
            for excl in (tc.Exclusion.PUSH, tc.Exclusion.CSR_PULL):
                for host_loop in (False, True):
                    got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=3,
                                                         exclusion=excl, host_loop=host_loop))
                    where = (kind, name, heur, excl, host_loop)
                    assert np.array_equal(got.mis, exp.mis), where
                    assert rounds_tuple(got.iterations) == oracle_tuple(exp), where
                    assert np.array_equal(got.state == 1, exp.state == 1), where
        dg.close()


def test_spatial_order_of_the_rgg(ctx):
    """tcmis_gen_rgg keeps its points' Z-order; solving on it is bit-exact."""
    dg = tc.DeviceGraph.rgg(20000, 3.0, 1, ctx)
    g = dg.download()
    og = O.Graph(g.n, g.offsets, g.neighbors)
    dg.reorder(tc.DeviceGraph.ORDER_SPATIAL)
    for heur in ("h2", "h3", "h1"):
        exp = O.solve(og, heur, 1, tile_dim=16)
        got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=1))
        assert np.array_equal(got.mis, exp.mis), heur
        assert rounds_tuple(got.iterations) == oracle_tuple(exp), heur
    # back to the caller's order: still the same
    dg.reorder(tc.DeviceGraph.ORDER_NONE)
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1))
    assert np.array_equal(got.mis, O.solve(og, "h2", 1, tile_dim=16).mis)
    dg.close()


def test_observer_and_tile_forms_ignore_the_order(ctx):
    g = O.gen("rmat", 11, 16, 1)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx).reorder(tc.DeviceGraph.ORDER_DEGREE)
    exp = O.solve(g, "h2", 1, tile_dim=16)
    seen = []
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1,
                                         iteration_observer=lambda it, c, s: seen.append(it)))
    assert np.array_equal(got.mis, exp.mis)
    assert seen == list(range(1, exp.n_rounds + 1))
    for excl in (tc.Exclusion.TILE_BITS, tc.Exclusion.TILE_MMA):
        got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, exclusion=excl))
        assert rounds_tuple(got.iterations) == oracle_tuple(exp)
    # the tile-form Phase 1 (its A-up store is on the caller's CSR) also runs
    # in the caller's order, with or without the degree order's settle data
    for flags in (tc.F_TILE_CAND, tc.F_TILE_CAND | tc.F_TILE_UMMA):
        cfg = tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, flags=flags)
        dg.tile_cand_prepare(cfg)
        for host_loop in (False, True):
            cfg.host_loop = host_loop
            got = tc.run_mis(dg, cfg)
            assert np.array_equal(got.mis, exp.mis), (flags, host_loop)
            assert rounds_tuple(got.iterations) == oracle_tuple(exp), (flags, host_loop)
    dg.close()


def test_order_errors(ctx):
    g = O.gen("rmat", 9, 8, 1)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    with pytest.raises(ValueError, match="permutation"):
        dg.reorder(tc.DeviceGraph.ORDER_GIVEN, np.zeros(g.n, np.int32))
    with pytest.raises(ValueError, match="tcmis_gen_rgg"):
        dg.reorder(tc.DeviceGraph.ORDER_SPATIAL)
    with pytest.raises(ValueError):
        dg.reorder(9)
    # a failed reorder leaves the graph usable in the caller's order
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1))
    assert np.array_equal(got.mis, O.solve(g, "h2", 1, tile_dim=16).mis)
    dg.close()


def test_permuted_graph_is_normalised(ctx):
    """tcmis_graph_permuted: the order's ids as an ordinary graph -- rows
    sorted, symmetric, the same degrees under the permutation -- which solves
    like any graph (here with both Phase 1 forms)."""
    dg = tc.DeviceGraph.rgg(20000, 3.0, 2, ctx).reorder(tc.DeviceGraph.ORDER_SPATIAL)
    p = dg.permuted()
    h = p.download()
    og = O.Graph(h.n, h.offsets, h.neighbors)
    for v in range(h.n):
        row = h.neighbors[h.offsets[v]:h.offsets[v + 1]]
        assert np.all(np.diff(row) > 0)
    src = dg.download()
    assert sorted(np.diff(src.offsets).tolist()) == sorted(np.diff(h.offsets).tolist())
    u = np.repeat(np.arange(h.n), np.diff(h.offsets))
    fwd = set(zip(u.tolist(), h.neighbors.tolist()))
    assert all((b, a) in fwd for a, b in fwd)
    exp = O.solve(og, "h2", 1, tile_dim=16)
    for flags in (0, tc.F_TILE_CAND):
        got = tc.run_mis(p, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, flags=flags))
        assert np.array_equal(got.mis, exp.mis), flags
        assert rounds_tuple(got.iterations) == oracle_tuple(exp), flags
    p.close()
    dg.close()


@pytest.mark.parametrize("spec", [("rmat", 14, 16, 2), ("rmat", 12, 4, 5), ("gnp_avg", 4000, 9.0, 1),
                                  ("grid", 40)])
@pytest.mark.parametrize("scale_bits", [8, 11, 20, 30])
def test_degree_class_bounds(ctx, spec, scale_bits, monkeypatch):
    """Degree order + H2 priorities: the select and pull kernels settle rows by
    the degree-class bounds (solver.cu k_class_bounds) without gathering the
    neighbours' keys.  Small scale_bits make p ties across neighbouring degrees
    common (floor of avg/d * 2^sb), i.e. wide uncertain bands; large ones make
    the bands narrow.  Bit-exact either way, and equal to the solve without
    the bounds (TCMIS_NO_CLASS_BOUNDS)."""
    g = O.gen(*spec)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx).reorder(tc.DeviceGraph.ORDER_DEGREE)
    for heur in ("h2", "h3", "luby-perm"):
        exp = O.solve(g, heur, 4, tile_dim=16, scale_bits=scale_bits)
        for excl in (tc.Exclusion.AUTO, tc.Exclusion.PUSH, tc.Exclusion.CSR_PULL):
            for host_loop in (False, True):
                got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=4, exclusion=excl,
                                                     scale_bits=scale_bits, host_loop=host_loop))
                where = (spec, heur, excl, host_loop)
                assert np.array_equal(got.mis, exp.mis), where
                assert rounds_tuple(got.iterations) == oracle_tuple(exp), where
    monkeypatch.setenv("TCMIS_NO_CLASS_BOUNDS", "1")
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=4, scale_bits=scale_bits))
    assert np.array_equal(got.mis, O.solve(g, "h2", 4, tile_dim=16, scale_bits=scale_bits).mis)
    dg.close()


def _hub_graph():
    """Random edges plus hubs of 9000, 3000, 700, 200 and 40 neighbours: rows
    in every tier of the row sort (order.cu sort_rows)."""
    rng = np.random.default_rng(11)
    n = 12000
    edges = set()
    for hub, d in ((0, 9000), (1, 3000), (2, 700), (3, 200), (4, 40)):
        for u in rng.choice(np.arange(5, n), d, replace=False):
            edges.add((min(hub, int(u)), max(hub, int(u))))
    for _ in range(30000):
        a, b = rng.integers(0, n, 2)
        if a != b:
            edges.add((int(min(a, b)), int(max(a, b))))
    return O.graph_from_edges(n, sorted(edges))


@pytest.mark.parametrize("kind", ["rmat", "hubs"])
def test_reordered_rows_are_sorted(ctx, kind):
    """tcmis_graph_reorder sorts every relabeled row (the scans' early stop
    relies on it): the permuted graph's rows ascend for each order and hold
    the relabeled neighbours; the solves stay bit-exact."""
    g = O.gen("rmat", 11, 8, 3) if kind == "rmat" else _hub_graph()
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    for mode in (tc.DeviceGraph.ORDER_DEGREE, tc.DeviceGraph.ORDER_GIVEN):
        order = np.random.default_rng(1).permutation(g.n).astype(np.int32) \
            if mode == tc.DeviceGraph.ORDER_GIVEN else None
        h = dg.reorder(mode, order).permuted().download()
        for v in range(h.n):
            assert np.all(np.diff(h.neighbors[h.offsets[v]:h.offsets[v + 1]]) > 0)
        assert sorted(np.diff(h.offsets).tolist()) == sorted(np.diff(g.off).tolist())
        for heur in ("h2", "h3", "h1"):
            got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=2))
            exp = O.solve(g, heur, 2, tile_dim=16)
            assert np.array_equal(got.mis, exp.mis), (kind, mode, heur)
            assert rounds_tuple(got.iterations) == oracle_tuple(exp), (kind, mode, heur)
    dg.close()


@pytest.mark.parametrize("pendants", [0, 50])
def test_degree_order_all_hub_rows(ctx, pendants):
    """A clique of 4200 vertices (every row longer than the sorted-row limit,
    order.cu kSortedMax) with or without pendant vertices: the round-1
    settling data (largest neighbour, class) and the bounds stay exact."""
    k = 4200
    iu, ju = np.triu_indices(k, 1)
    rng = np.random.default_rng(3)
    pend = np.stack([rng.integers(0, k, pendants), k + np.arange(pendants)], 1)
    g = O.graph_from_edges(k + pendants, np.concatenate([np.stack([iu, ju], 1), pend]))
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx).reorder(tc.DeviceGraph.ORDER_DEGREE)
    for heur in ("h2", "h3", "luby-perm"):
        exp = O.solve(g, heur, 5, tile_dim=16)
        got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=5))
        assert np.array_equal(got.mis, exp.mis), heur
        assert rounds_tuple(got.iterations) == oracle_tuple(exp), heur
    dg.close()


def test_round1_settling_switch(ctx, monkeypatch):
    """The round-1 settling (select.cuh r1_max) on and off give the same solve."""
    g = O.gen("rmat", 13, 16, 6)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx).reorder(tc.DeviceGraph.ORDER_DEGREE)
    exp = O.solve(g, "h2", 1, tile_dim=16)
    for off in (None, "1"):
        if off:
            monkeypatch.setenv("TCMIS_NO_R1_SETTLE", off)
        for excl in (tc.Exclusion.AUTO, tc.Exclusion.PUSH, tc.Exclusion.CSR_PULL):
            got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, exclusion=excl))
            assert np.array_equal(got.mis, exp.mis), (off, excl)
            assert rounds_tuple(got.iterations) == oracle_tuple(exp), (off, excl)
    dg.close()


def _star_forest(n_hubs=6, leaves=1500, extra=20000, seed=7):
    """Hubs of 1500 leaves whose leaves also link at random: after round 1
    the hubs and many mid-degree rows stay alive, so k_tail scans and pushes
    rows of every length class (thread window, 16-lane groups, whole-block
    rows above 512 and above 8192 entries pushed through the flat list)."""
    rng = np.random.default_rng(seed)
    n = n_hubs + n_hubs * leaves
    edges = set()
    for h in range(n_hubs):
        for u in range(n_hubs + h * leaves, n_hubs + (h + 1) * leaves):
            edges.add((h, u))
        for h2 in range(h + 1, n_hubs):
            edges.add((h, h2))
    for _ in range(extra):
        a, b = rng.integers(n_hubs, n, 2)
        if a != b:
            edges.add((int(min(a, b)), int(max(a, b))))
    return O.graph_from_edges(n, sorted(edges))


@pytest.mark.parametrize("kind", ["hubs", "stars", "rmat"])
@pytest.mark.parametrize("knob", [None, "TCMIS_TAIL_Q_L2", "TCMIS_TAIL_TAG_PAR",
                                  "TCMIS_TAIL_BAR_FENCE"])
def test_tail_class_bound_scans(ctx, kind, knob, monkeypatch):
    """k_tail on a degree-ordered H2 solve: the scans stop at the row's lower
    class bound, early candidates push the rest of their rows through the
    block's flat push list, q is probed in L1 first (tail.cuh).  Bit-exact
    for every tail switch point, seed and scale_bits, with each A/B knob of
    the tail (L2-only q reads, the tag loaded with q, the fenced barrier)."""
    if knob:
        monkeypatch.setenv(knob, "1")
    g = (_hub_graph() if kind == "hubs" else _star_forest() if kind == "stars"
         else O.gen("rmat", 13, 16, 4))
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx).reorder(tc.DeviceGraph.ORDER_DEGREE)
    for thr in (None, "1000000000", "64"):
        if thr is None:
            monkeypatch.delenv("TCMIS_TAIL_THRESHOLD", raising=False)
        else:
            monkeypatch.setenv("TCMIS_TAIL_THRESHOLD", thr)
        for seed, sb in ((1, 20), (2, 8), (3, 30)):
            for heur in ("h2", "h3"):
                exp = O.solve(g, heur, seed, tile_dim=16, scale_bits=sb)
                got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=seed,
                                                     scale_bits=sb))
                where = (kind, knob, thr, seed, sb, heur)
                assert np.array_equal(got.mis, exp.mis), where
                assert rounds_tuple(got.iterations) == oracle_tuple(exp), where
    dg.close()
