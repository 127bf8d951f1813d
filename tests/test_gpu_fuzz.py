"""GPU: randomised parity sweep -- random graph families and sizes (paths,
stars, cliques, bipartite, power-law, sparse/dense G(n,p), disconnected
unions), every heuristic, random seeds, scale_bits and tile_dim, every
exclusion form and tail switch point, against the oracle (pinned to the
compiled reference in tests/test_oracle.py).  Bit-exact MIS, iteration count
and every per-iteration statistic."""
import numpy as np
import pytest

import oracle as O
import paper_2605_29604_b200 as tc

pytestmark = pytest.mark.gpu

HEUR = {"h1": tc.Heuristic.H1, "h2": tc.Heuristic.H2, "h3": tc.Heuristic.H3,
        "luby-fresh": tc.Heuristic.LubyFresh, "luby-perm": tc.Heuristic.LubyPerm}
EXCL = [tc.Exclusion.AUTO, tc.Exclusion.PUSH, tc.Exclusion.CSR_PULL, tc.Exclusion.TILE_BITS,
        tc.Exclusion.TILE_MMA]


def random_graph(rng):
    kind = rng.integers(0, 8)
    if kind == 0:  # path
        n = int(rng.integers(2, 3000))
        e = np.stack([np.arange(n - 1), np.arange(1, n)], 1)
    elif kind == 1:  # star + noise
        n = int(rng.integers(3, 20000))
        e = np.stack([np.zeros(n - 1, np.int64), np.arange(1, n)], 1)
        e = np.concatenate([e, rng.integers(0, n, (n // 10, 2))])
    elif kind == 2:  # clique
        k = int(rng.integers(2, 60))
        n = k
        a, b = np.triu_indices(k, 1)
        e = np.stack([a, b], 1)
    elif kind == 3:  # complete bipartite
        k1, k2 = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        n = k1 + k2
        a, b = np.meshgrid(np.arange(k1), k1 + np.arange(k2))
        e = np.stack([a.ravel(), b.ravel()], 1)
    elif kind == 4:  # power law (R-MAT)
        return O.gen("rmat", int(rng.integers(6, 15)), int(rng.integers(1, 24)),
                     int(rng.integers(1, 1 << 30)))
    elif kind == 5:  # sparse / dense G(n, p)
        return O.gen("gnp_avg", int(rng.integers(10, 20000)), float(rng.uniform(0.5, 40)),
                     int(rng.integers(1, 1 << 30)))
    elif kind == 6:  # grid
        return O.gen("grid", int(rng.integers(1, 120)))
    else:  # disjoint union of small random pieces + isolated vertices
        n = int(rng.integers(50, 5000))
        e = rng.integers(0, n, (int(rng.integers(0, 4 * n)), 2))
        e = e[np.abs(e[:, 0] - e[:, 1]) < 40]
    return O.graph_from_edges(int(n), np.asarray(e, np.int32).reshape(-1, 2))


@pytest.mark.parametrize("case", range(64))
def test_random_parity(ctx, case, monkeypatch):
    rng = np.random.default_rng(1000 + case)
    g = random_graph(rng)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    monkeypatch.setenv("TCMIS_TAIL_THRESHOLD", str(int(rng.choice([0, 1, 64, 65536, 1 << 30]))))
    for _ in range(4):
        heur = str(rng.choice(list(HEUR)))
        seed = int(rng.integers(0, 1 << 40))
        scale_bits = int(rng.integers(8, 31))
        T = int(rng.choice([1, 3, 8, 16, 16, 33, 64]))
        excl = EXCL[int(rng.integers(0, len(EXCL)))]
        host_loop = bool(rng.integers(0, 2))
        exp = O.solve(g, heur, seed, tile_dim=T, scale_bits=scale_bits)
        got = tc.run_mis(dg, tc.EngineConfig(heuristic=HEUR[heur], seed=seed, tile_dim=T,
                                             scale_bits=scale_bits, exclusion=excl,
                                             host_loop=host_loop))
        ctxt = (case, heur, seed, scale_bits, T, int(excl), host_loop)
        assert np.array_equal(got.mis, exp.mis), ctxt
        want = [(r["sel"], r["rem"], r["alive"], r["tiles_eval"], r["tiles_skip"])
                for r in exp.rounds]
        if heur == "luby-perm" or heur == "luby-fresh":
            want = [w[:3] + (0, 0) for w in want]
        gotr = [(i.candidates_selected, i.vertices_removed, i.alive_remaining,
                 i.tiles_evaluated, i.tiles_skipped) for i in got.iterations]
        assert gotr == want, ctxt
