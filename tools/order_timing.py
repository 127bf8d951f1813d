"""Wall time of tcmis_graph_reorder (degree order) on the bench graphs, the
first call (lazy module loading included) and warm calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29604_b200 as tc  # noqa: E402
import bench  # noqa: E402

for cfg in sys.argv[1:] or ["rmat22"]:
    ctx = tc.Context(0)
    dg = bench.make_device_graph(tc, cfg, ctx)
    ts = []
    for _ in range(4):
        ctx.synchronize()
        t = time.perf_counter()
        dg.reorder(tc.DeviceGraph.ORDER_DEGREE)
        ctx.synchronize()
        ts.append(round((time.perf_counter() - t) * 1e3, 2))
    print(cfg, "reorder ms (first, warm...)", ts, flush=True)
    dg.close()
