# A/B: resident blocks of the probe kernels (spills at 32 registers)
mkdir -p gpurun_out
for mb in 8 6 4; do
  if [ $mb != 8 ]; then
    rm -f paper_2605_29604_b200/_obj/solver.cu.o
    TCMIS_NVCC_EXTRA=-DTCMIS_PROBE_MINB=$mb python -m paper_2605_29604_b200.build > /dev/null 2>&1
  fi
  for c in grid rgg rmat22; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/mb${mb}_$c.json 2> gpurun_out/mb${mb}_$c.log
    echo "minb=$mb $(python tools/bench_summary.py gpurun_out/mb${mb}_$c.json | cut -c1-60)"
    python - <<PY
import json; d=json.load(open("gpurun_out/mb${mb}_$c.json")); print("   ", [k for k in d["kernels_ms"] if k[0] in ("k_probe_select","k_probe_pull")])
PY
  done
done
