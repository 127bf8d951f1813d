python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tile" > gpurun_out/pytest_tile.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tile.log
python - <<'PY' > gpurun_out/tile26_time2.txt 2>&1
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
    t = time.perf_counter(); cnt = g.tile(16); t1 = time.perf_counter()
    print("tile ms", (t1 - t) * 1e3, cnt, flush=True)
    g.close()
PY
