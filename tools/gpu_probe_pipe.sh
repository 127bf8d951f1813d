# k_probe_select software pipeline: parity + A/B at 8 and 6 resident blocks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py -m gpu -q -x > gpurun_out/pytest_pipe.txt 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_pipe.txt
for mb in 8 6; do
  if [ $mb != 8 ]; then rm -f paper_2605_29604_b200/_obj/solver.cu.o; TCMIS_NVCC_EXTRA=-DTCMIS_PROBE_MINB=$mb python -m paper_2605_29604_b200.build > /dev/null 2>&1; fi
  for c in grid rgg rmat22 rmat26; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/pipe${mb}_$c.json 2> gpurun_out/pipe${mb}_$c.log
    python - <<PY
import json; d=json.load(open("gpurun_out/pipe${mb}_$c.json")); print("minb=$mb $c dev", d["device_resident"]["ms"], [k for k in d["kernels_ms"] if k[0]=="k_probe_select"])
PY
  done
done
