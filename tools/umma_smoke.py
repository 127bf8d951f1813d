# first light of the tcgen05 Phase-1 tile product: a small grid, every round through the tiles
import os, sys
sys.path.insert(0, '.')
os.environ["TCMIS_TILE_CAND_GATE"] = "1"
import numpy as np
import oracle as O
import paper_2605_29604_b200 as tc
ctx = tc.Context(0)
for kind, args in (("grid", (20,)), ("grid", (64,)), ("rmat", (10, 8, 1)), ("gnp_avg", (2000, 10.0, 3))):
    g = O.gen(kind, *args)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    exp = O.solve(g, "h2", 1, tile_dim=16)
    for umma in (False, True):
        got = tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, host_loop=True,
                                             flags=tc.F_TILE_CAND | (tc.F_TILE_UMMA if umma else 0)))
        print(kind, args, "umma" if umma else "bits", "mis ok" if np.array_equal(got.mis, exp.mis) else "MIS DIFFERS",
              len(got.iterations), exp.n_rounds, flush=True)
    dg.close()
