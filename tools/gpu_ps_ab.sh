# A/B: k_prio_settle occupancy (stages / flush interval / resident blocks)
mkdir -p gpurun_out
run() {
  tag=$1; shift
  rm -f paper_2605_29604_b200/_obj/solver.cu.o
  TCMIS_NVCC_EXTRA="$*" python -m paper_2605_29604_b200.build > gpurun_out/ps_build_$tag.log 2>&1 || { echo build $tag failed; return; }
  for c in rmat22 rmat26 rgg; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ps${tag}_$c.json 2> gpurun_out/ps${tag}_$c.log
    python - <<PY
import json; d=json.load(open("gpurun_out/ps${tag}_$c.json")); print("$tag $c dev", d["device_resident"]["ms"], [k for k in d["kernels_ms"] if k[0]=="k_prio_settle"])
PY
  done
}
run base ""
run s2f2m6 -DTCMIS_PS_STAGES=2 -DTCMIS_PS_FLUSH=2 -DTCMIS_PS_MINB=6
run s2f4m5 -DTCMIS_PS_STAGES=2 -DTCMIS_PS_FLUSH=4 -DTCMIS_PS_MINB=5
run s3f2m5 -DTCMIS_PS_STAGES=3 -DTCMIS_PS_FLUSH=2 -DTCMIS_PS_MINB=5
timeout 600 python -m pytest tests/test_gpu_order.py -m gpu -q -x -k "class_bounds or settling" > gpurun_out/ps_pytest.txt 2>&1; echo pytest_last_variant=$?; tail -1 gpurun_out/ps_pytest.txt
