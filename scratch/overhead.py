# graph-mode solve time of tiny graphs = the fixed per-solve overhead
import ctypes as C, sys, time; sys.path.insert(0, '.')
import torch
import paper_2605_29604_b200 as tc
import oracle as O
ctx = tc.Context(0)
L = tc.load()
stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
for spec in (("petersen",), ("gnp_avg", 2000, 8.0, 1)):
    g = O.gen(*spec)
    dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
    dg.tile(16)
    cfg = tc.EngineConfig(heuristic=tc.Heuristic.H2)
    c, _k = cfg._c()
    stats = (tc._Stats * 4096)()
    def solve():
        d_mis, d_state = C.c_void_p(), C.c_void_p()
        cnt, nit = C.c_int64(0), C.c_int32(0)
        tc._check(L.tcmis_solve_device(dg.h, C.byref(c), C.byref(d_mis), C.byref(cnt), C.byref(d_state), stats, 4096, C.byref(nit)))
    for _ in range(20): solve()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(50)]
    t0 = time.perf_counter()
    for a, b in ev:
        with torch.cuda.stream(stream): a.record(stream)
        solve()
        with torch.cuda.stream(stream): b.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 50 * 1e6
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    print(spec, "device us median %.1f min %.1f  host wall us %.1f" % (ms[25] * 1e3, ms[0] * 1e3, wall))
