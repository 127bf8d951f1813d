# device G(n,p): parity against the oracle + the full GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k gnp > gpurun_out/pytest_gnp.txt 2>&1; echo gnp=$?; tail -3 gpurun_out/pytest_gnp.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.txt
python - <<'PY' 2>&1 | tail -3
import time, paper_2605_29604_b200 as tc, torch
ctx = tc.Context(0)
for n, d in ((100000, 16.0), (1 << 24, 16.0)):
    tc.DeviceGraph.gnp(n, d, 1, ctx).close()
    ctx.synchronize(); t = time.perf_counter()
    g = tc.DeviceGraph.gnp(n, d, 1, ctx); ctx.synchronize()
    print("gnp", n, d, "edges", g.nnz // 2, "ms", round((time.perf_counter() - t) * 1e3, 2))
    g.close()
PY
