# pageable drop-in e2e: staging lanes x piece size sweep (C++ harness)
mkdir -p gpurun_out
python - <<'P'
import numpy as np, sys
sys.path.insert(0, '.')
import paper_2605_29604_b200 as tc
ctx = tc.Context(0)
dg = tc.DeviceGraph.rmat(22, 16, 1, ctx)
h = dg.download()
with open('/tmp/g22.bin', 'wb') as f:
    f.write(np.int32(h.n).tobytes()); f.write(np.int64(h.neighbors.size).tobytes())
    f.write(h.offsets.astype(np.int64).tobytes()); f.write(h.neighbors.astype(np.int32).tobytes())
P
PKG=paper_2605_29604_b200
g++ -std=c++20 -O2 -I include tests/cpp/e2e_main.cpp -L $PKG -ltcmis -ltcmis_b200 -Wl,-rpath,$PWD/$PKG -o /tmp/e2e
for t in 8 12; do
  echo "threads=$t $(TCMIS_STAGE_THREADS=$t /tmp/e2e /tmp/g22.bin 5 h2 | python -c 'import json,sys; d=json.load(sys.stdin); print(d["median_ms"], d["ms"], d["capi_breakdown_ms"])')"
done
echo "nostage $(TCMIS_NO_STAGING=1 /tmp/e2e /tmp/g22.bin 5 h2 | python -c 'import json,sys; d=json.load(sys.stdin); print(d["median_ms"], d["ms"], d["capi_breakdown_ms"])')"
