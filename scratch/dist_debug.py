# 2-process gloo emulation on one GPU: full= vs rows= partitions, bounded rounds
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29604_b200 as tc
from paper_2605_29604_b200 import distributed as D
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
ctx = tc.Context(0)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
full = tc.DeviceGraph.rmat(scale, 16, 1, ctx)
h = full.download()
off = h.offsets
rank_lo = D.partition_rows(off, world, 16)
ref = tc.run_mis(full, tc.EngineConfig(heuristic=tc.Heuristic.H2, seed=1, tile_dim=16))
print(f"[r{rank}] single: |MIS|={len(ref.mis)} rounds={len(ref.iterations)}", flush=True)
def show(tag, res):
    print(f"[r{rank}] {tag}: rounds={[(r.candidates_selected, r.vertices_removed, r.alive_remaining) for r in res.rounds][:8]} n={len(res.rounds)}", flush=True)
for it in range(2):
    me = D.GpuRank(ctx, full.n, rank_lo[rank], rank_lo[rank + 1], None, None, "cuda:0", full=full)
    show(f"full#{it}", D.solve_partitioned(me, rank_lo, rank, world, dist, max_rounds=12))
    me.close()
rows = np.ascontiguousarray(h.neighbors[off[rank_lo[rank]]:off[rank_lo[rank + 1]]])
for it in range(3):
    rk = D.GpuRank(ctx, full.n, rank_lo[rank], rank_lo[rank + 1], off, None, "cuda:0", rows=rows)
    try:
        show(f"rows#{it}", D.solve_partitioned(rk, rank_lo, rank, world, dist, max_rounds=12))
    except Exception as e:
        print(f"[r{rank}] rows#{it}: {e}", flush=True)
    rk.close()
# bench-like: the full= rank stays alive, own rows downloaded from it, pinned
me = D.GpuRank(ctx, full.n, rank_lo[rank], rank_lo[rank + 1], None, None, "cuda:0", full=full)
show("bench-timed", D.solve_partitioned(me, rank_lo, rank, world, dist, max_rounds=12))
L = tc.load()
lo, hi = rank_lo[rank], rank_lo[rank + 1]
own_rows = np.zeros(max(1, int(off[hi] - off[lo])), np.int32)
part_off = np.zeros(full.n + 1, np.int64)
tc._check(L.tcmis_graph_download(me.g.h, tc._ptr(part_off), tc._ptr(own_rows)))
print(f"[r{rank}] download equal: {np.array_equal(own_rows[:off[hi]-off[lo]], rows)}", flush=True)
own_rows = torch.from_numpy(own_rows[:int(off[hi] - off[lo])]).pin_memory().numpy()
h_off = torch.from_numpy(off).pin_memory().numpy()
for it in range(3):
    rk = D.GpuRank(ctx, full.n, lo, hi, h_off, None, "cuda:0", rows=own_rows)
    try:
        show(f"bench-e2e#{it}", D.solve_partitioned(rk, rank_lo, rank, world, dist, max_rounds=12))
    except Exception as e:
        print(f"[r{rank}] bench-e2e#{it}: {e}", flush=True)
    rk.close()
dist.destroy_process_group()
