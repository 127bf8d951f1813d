import time, sys, numpy as np
sys.path.insert(0, '.')
import paper_2605_29604_b200 as tc
ctx = tc.Context(0)
t=time.time(); dg = tc.DeviceGraph.rmat(22, 16, 1, ctx); ctx.synchronize(); print("gen s22", time.time()-t, dg.n, dg.num_edges())
t=time.time(); print("tiles", dg.tile(16), time.time()-t)
for h in (tc.Heuristic.H2, tc.Heuristic.H3):
    cfg = tc.EngineConfig(heuristic=h, timing=True)
    for i in range(4):
        t=time.perf_counter(); r = tc.run_mis(dg, cfg); dt=time.perf_counter()-t
    print(h.name, "wall ms", dt*1e3, "|MIS|", r.cardinality(), "iters", len(r.iterations), [(round(i.phase1_ms,3), round(i.phase3_ms,3)) for i in r.iterations])
for name, mk in (("grid", lambda: tc.DeviceGraph.grid(4096, ctx)), ("rgg", lambda: tc.DeviceGraph.rgg(24000000, 3.0, 1, ctx))):
    t=time.time(); g2 = mk(); ctx.synchronize(); print("gen", name, time.time()-t, g2.n, g2.num_edges())
    g2.tile(16)
    cfg = tc.EngineConfig(heuristic=tc.Heuristic.H2, timing=True)
    for i in range(3):
        t=time.perf_counter(); r = tc.run_mis(g2, cfg); dt=time.perf_counter()-t
    print(name, "wall ms", dt*1e3, "|MIS|", r.cardinality(), [(round(i.phase1_ms,3), round(i.phase3_ms,3)) for i in r.iterations])
    del g2
