# k_tail phase timeline (build with -DTCMIS_TAIL_PROF); box only
import ctypes as C, sys; sys.path.insert(0, '.')
import paper_2605_29604_b200 as tc
import bench
L = tc.load()
ctx = tc.Context(0)
TAG = {1: "start", 2: "pass", 3: "barrier", 4: "compact0", 5: "count", 6: "countbar", 7: "compact1",
       8: "fill", 9: "thr", 10: "grp", 11: "blk", 12: "push"}
buf = (C.c_ulonglong * 256)()
for cfg in sys.argv[1:]:
    dg = bench.make_device_graph(tc, cfg, ctx)
    dg.tile(16)
    import os
    order = os.environ.get("ORDER") or {"rgg": "spatial", "rmat22": "degree",
                                        "rmat26": "degree"}.get(cfg, "none")
    if order != "none":
        dg.reorder({"degree": tc.DeviceGraph.ORDER_DEGREE,
                    "spatial": tc.DeviceGraph.ORDER_SPATIAL}[order])
    print(cfg, "order", order)
    for i in range(3):
        L.tcmis_debug_tail_prof(buf, 256)
        tc.run_mis(dg, tc.EngineConfig(heuristic=tc.Heuristic.H2))
        ctx.synchronize()
        n = L.tcmis_debug_tail_prof(buf, 256)
        t0 = buf[0]
        print(cfg, i, " ".join(f"{TAG[buf[2*k+1] >> 32]}({buf[2*k+1] & 0xffffffff})@{(buf[2*k]-t0)/1000:.1f}" for k in range(n)), flush=True)
    dg.close()
# per-block view of the first tail round (last solve of the last config)
import numpy as np
blk = (C.c_ulonglong * (5 * 1024))()
L.tcmis_debug_tail_blk(blk)
a = np.frombuffer(blk, dtype=np.uint64).reshape(5, 1024)[:, :148].astype(np.int64)
t0 = a[4].min()
for name, row in (("round start", a[4]), ("thread-phase end", a[0]), ("block-phase end", a[1])):
    x = (row - t0) / 1e3
    print(f"{name} us: min {x.min():.1f} med {np.median(x):.1f} max {x.max():.1f}")
print("deferred per block: min %d med %d max %d sum %d" % (a[2].min(), np.median(a[2]), a[2].max(), a[2].sum()))
print("entries per block: min %d med %d max %d sum %d" % (a[3].min(), np.median(a[3]), a[3].max(), a[3].sum()))
order = np.argsort(-a[1])[:8]
for b in order:
    print(f"  slow block {b}: start {(a[4][b]-t0)/1e3:.1f} thr {(a[0][b]-t0)/1e3:.1f} end {(a[1][b]-t0)/1e3:.1f} entries {a[3][b]} deferred {a[2][b]}")
