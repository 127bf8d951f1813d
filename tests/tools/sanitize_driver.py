"""Small solves over every device path, for compute-sanitizer
(tests/test_gpu_sanitizer.py): the whole-solve CUDA graph (or with
--host-loop-only every kernel as a plain launch), the host loop,
k_tail (forced at every round), the per-round kernels only, both exclusion
forms, the relabeled CSR, the tile forms, the validator, the generators and
the native partitioned solve with 3 ranks on one device.  Checks results
against the oracle so a silent corruption fails too.  No torch import."""
import ctypes as C
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2605_29604_b200 as tc  # noqa: E402
from paper_2605_29604_b200 import distributed as D  # noqa: E402

H = {"h1": tc.Heuristic.H1, "h2": tc.Heuristic.H2, "h3": tc.Heuristic.H3,
     "luby-fresh": tc.Heuristic.LubyFresh, "luby-perm": tc.Heuristic.LubyPerm}


def step(*what):
    if os.environ.get("TCMIS_SANITIZE_TRACE"):
        print("step", *what, file=sys.stderr, flush=True)


HOST_LOOP_ONLY = "--host-loop-only" in sys.argv


def check(g, dg, heur, **kw):
    if HOST_LOOP_ONLY:  # every kernel as a plain launch (no CUDA graph)
        kw["host_loop"] = True
    step(g.n, heur, kw)
    exp = O.solve(g, heur, 1, tile_dim=16)
    got = tc.run_mis(dg, tc.EngineConfig(heuristic=H[heur], seed=1, **kw))
    assert np.array_equal(got.mis, exp.mis), (heur, kw)


def main(parts_only=False, single_only=False, gens_only=False):
    ctx = tc.Context(0)
    L = tc.load()
    for kind, args in (() if parts_only or gens_only else (("rmat", (11, 16, 1)), ("grid", (40,)),
                                              ("gnp_avg", (2000, 10.0, 3)))):
        g = O.gen(kind, *args)
        dg = tc.DeviceGraph.upload(tc.Graph(g.n, g.off, g.nbr), ctx)
        for heur in H:
            check(g, dg, heur)
            check(g, dg, heur, host_loop=True)
        for excl in (tc.Exclusion.PUSH, tc.Exclusion.CSR_PULL, tc.Exclusion.TILE_BITS,
                     tc.Exclusion.TILE_MMA):
            check(g, dg, "h2", exclusion=excl)
        for thr in ("0", "1"):
            os.environ["TCMIS_TAIL_THRESHOLD"] = thr
            check(g, dg, "h2")
            check(g, dg, "h3", host_loop=True)
        os.environ.pop("TCMIS_TAIL_THRESHOLD", None)
        dg.reorder(tc.DeviceGraph.ORDER_DEGREE)
        check(g, dg, "h2")
        check(g, dg, "h1", host_loop=True)
        os.environ["TCMIS_MIS_O_MAX"] = "0"
        check(g, dg, "h2")
        os.environ.pop("TCMIS_MIS_O_MAX")
        exp = O.solve(g, "h2", 1, tile_dim=16)
        assert tc.check_independence(dg, exp.mis, ctx)[0]
        assert tc.check_maximality(dg, exp.mis, ctx)[0]
        dg.close()
    if single_only:
        print("sanitize driver ok")
        return
    step("generators")
    # generators
    gens = () if parts_only else (tc.DeviceGraph.rmat(10, 8, 2, ctx), tc.DeviceGraph.grid(17, ctx),
                                  tc.DeviceGraph.rgg(3000, 3.0, 1, ctx))
    for dg in gens:
        h = dg.download()
        g = O.Graph(h.n, h.offsets, h.neighbors)
        if dg.n == 3000:
            dg.reorder(tc.DeviceGraph.ORDER_SPATIAL)
        check(g, dg, "h2")
        dg.close()
    if gens_only:
        print("sanitize driver ok")
        return
    step("partitioned")
    # native partitioned solve, 3 ranks of one process on this device
    g = O.gen("rmat", 11, 16, 4)
    lo = D.partition_rows(g.off, 3, 16)
    parts = []
    for r in range(3):
        h = C.c_void_p()
        rows = np.ascontiguousarray(g.nbr[g.off[lo[r]]:g.off[lo[r + 1]]], np.int32)
        c = tc.Context(0)
        tc._check(L.tcmis_graph_upload_partition(c.h, g.n, lo[r], lo[r + 1],
                                                 C.c_void_p(g.off.ctypes.data),
                                                 C.c_void_p(rows.ctypes.data) if rows.size else None,
                                                 C.byref(h)))
        parts.append((c, tc.DeviceGraph(h, c)))
    xs = D.Exchange.local_group(3)
    out = [None] * 3

    def run(k):
        out[k] = D.solve_native(parts[k][1], xs[k], lo, heuristic="h2")

    th = [threading.Thread(target=run, args=(k,)) for k in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    exp = O.solve(g, "h2", 1, tile_dim=16)
    for r in out:
        assert np.array_equal(r.mis, exp.mis)
    for x in xs:
        x.close()
    for c, p in parts:
        p.close()
    print("sanitize driver ok")


if __name__ == "__main__":
    main(parts_only="--parts" in sys.argv, single_only="--single" in sys.argv,
         gens_only="--gens" in sys.argv)
