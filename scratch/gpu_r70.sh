python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tile26_launches.csv python scratch/tile_only.py 26 > gpurun_out/tile26.log 2>&1
python - <<'PY' > gpurun_out/tile26_time.txt 2>&1
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2605_29604_b200 as tc
ctx = tc.Context(0)
dg = tc.DeviceGraph.rmat(26, 16, 1, ctx)
h = dg.download()
dg.close()
for _ in range(3):
    g = tc.DeviceGraph.upload(h, ctx)
    ctx.synchronize()
    t = time.perf_counter(); g.tile(16); t1 = time.perf_counter()
    print("tile ms", (t1 - t) * 1e3, flush=True)
    g.close()
PY
