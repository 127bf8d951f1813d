"""A/B of the in-process exchange group (several ranks on cuda:0): the fused
peer-memory apply against all-gathered copies (TCMIS_PART_NO_PEER).  Prints a
JSON line per (world, mode): wall ms per solve (host threads included), the
rank-0 host profile, and that the MIS equals the single-rank solve's."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29604_b200 as tc  # noqa: E402
from paper_2605_29604_b200 import distributed as D  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
ctx0 = tc.Context(0)
full = tc.DeviceGraph.rmat(scale, 16, 1, ctx0)
n = full.n
off = np.zeros(n + 1, np.int64)
tc._check(tc.load().tcmis_graph_download(full.h, tc._ptr(off), None))
ref = None
for world in (1, 2, 4):
    rank_lo = D.partition_rows(off, world, 16)
    ranks = [D.GpuRank(tc.Context(0), n, rank_lo[r], rank_lo[r + 1], None, None, "cuda:0",
                       full=full) for r in range(world)]
    for mode in ("peer", "copy"):
        if mode == "copy":
            os.environ["TCMIS_PART_NO_PEER"] = "1"
        else:
            os.environ.pop("TCMIS_PART_NO_PEER", None)
        D.solve_native_local(ranks, rank_lo, heuristic="h2")  # warm-up (graphs, buffers)
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            res = D.solve_native_local(ranks, rank_lo, heuristic="h2")
            ts.append((time.perf_counter() - t) * 1e3)
        mis = np.sort(res[0].mis)
        if ref is None:
            ref = mis
        print(json.dumps({"world": world, "mode": mode, "ms_median": round(float(np.median(ts)), 3),
                          "ms_min": round(min(ts), 3), "same_mis": bool(np.array_equal(mis, ref)),
                          "profile": D.native_profile(ranks[0].g)}), flush=True)
    for rk in ranks:
        rk.close()
