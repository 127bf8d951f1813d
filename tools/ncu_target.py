# one warm solve + one profiled solve of the bench config (used under ncu only)
# env EXCL = auto | push | pull | tile-bits | tile-mma
import os, sys; sys.path.insert(0, '.')
import paper_2605_29604_b200 as tc
cfgname = sys.argv[1] if len(sys.argv) > 1 else "rmat22"
ctx = tc.Context(0)
import bench
dg = bench.make_device_graph(tc, cfgname, ctx)
dg.tile(16)
# the bench's vertex order for this config (bench.py --order auto)
order = os.environ.get("ORDER") or {"rgg": "degree", "rmat22": "degree",
                                     "rmat26": "degree"}.get(cfgname, "none")
if order != "none":
    dg.reorder({"degree": tc.DeviceGraph.ORDER_DEGREE, "spatial": tc.DeviceGraph.ORDER_SPATIAL}[order])
ex = {"auto": tc.Exclusion.AUTO, "push": tc.Exclusion.PUSH, "pull": tc.Exclusion.CSR_PULL,
      "tile-bits": tc.Exclusion.TILE_BITS, "tile-mma": tc.Exclusion.TILE_MMA}[os.environ.get("EXCL", "auto")]
# env CAND = csr | tile | tile-umma: Phase 1 form (tile forms: A-up prepared outside)
cand = os.environ.get("CAND", "csr")
flags = {"csr": 0, "tile": tc.F_TILE_CAND, "tile-umma": tc.F_TILE_CAND | tc.F_TILE_UMMA}[cand]
cfg = tc.EngineConfig(heuristic=tc.Heuristic.H2, host_loop=True, exclusion=ex, flags=flags)
if flags:
    dg.tile_cand_prepare(cfg)
for _ in range(2):
    r = tc.run_mis(dg, cfg)
print("ok", r.cardinality(), len(r.iterations))
