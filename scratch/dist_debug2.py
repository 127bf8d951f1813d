# bench-exact sequence (2-process gloo emulation on one GPU), bounded rounds
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ.get("TCMIS_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29604_b200 as tc
from paper_2605_29604_b200 import distributed as D
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
ctx = tc.Context(0)
L = tc.load()
variant = sys.argv[1]
full = tc.DeviceGraph.rmat(22, 16, 1, ctx)
n = full.n
off = np.zeros(n + 1, np.int64)
tc._check(L.tcmis_graph_download(full.h, tc._ptr(off), None))
rank_lo = D.partition_rows(off, world, 16)
me = D.GpuRank(ctx, n, rank_lo[rank], rank_lo[rank + 1], None, None, "cuda:0", full=full)
if variant != "keepfull":
    full.close()
def show(tag, res):
    print(f"[r{rank}] {tag}: {[(r.candidates_selected, r.vertices_removed, r.alive_remaining) for r in res.rounds][:6]}", flush=True)
nsolve = 1 if variant == "one" else 6
for _ in range(nsolve):
    res = D.solve_partitioned(me, rank_lo, rank, world, dist, max_rounds=8)
show("timed", res)
lo, hi = rank_lo[rank], rank_lo[rank + 1]
own_rows = np.zeros(max(1, int(off[hi] - off[lo])), np.int32)
part_off = np.zeros(n + 1, np.int64)
tc._check(L.tcmis_graph_download(me.g.h, tc._ptr(part_off), tc._ptr(own_rows)))
own_rows = torch.from_numpy(own_rows[:int(off[hi] - off[lo])]).pin_memory().numpy()
h_off = torch.from_numpy(off).pin_memory().numpy()
for it in range(int(os.environ.get("DD_ITERS", "2"))):
    rk = D.GpuRank(ctx, n, lo, hi, h_off, None, "cuda:0", rows=own_rows)
    try:
        show(f"e2e#{it}", D.solve_partitioned(rk, rank_lo, rank, world, dist, max_rounds=8))
    except Exception as e:
        print(f"[r{rank}] e2e#{it}: {str(e)[:300]}", flush=True)
    rk.close()
dist.destroy_process_group()
