# s26: caller-order membership plane (mis_o) vs the final gather compaction
mkdir -p gpurun_out
for m in default big; do
  if [ $m = big ]; then export TCMIS_MIS_O_MAX=100000000; else unset TCMIS_MIS_O_MAX; fi
  for i in 1 2; do
    timeout 300 python bench.py --config rmat26 --no-e2e --no-cpu-baseline > gpurun_out/miso_${m}_$i.json 2> gpurun_out/miso_${m}_$i.log
    python - <<PY
import json; d=json.load(open("gpurun_out/miso_${m}_$i.json")); print("$m", d["ms_per_step"], d["device_resident"]["ms"], [k for k in d["kernels_ms"] if k[0] in ("k_prio_settle","k_tail","k_gc_bits","k_gc_ids")])
PY
  done
done
export TCMIS_MIS_O_MAX=100000000
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "26" > gpurun_out/miso_pytest.txt 2>&1; echo pytest26=$?; tail -1 gpurun_out/miso_pytest.txt
