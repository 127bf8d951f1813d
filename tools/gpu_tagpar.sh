# new tail test + A/B of the tag loaded with q (TCMIS_TAIL_TAG_PAR)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_order.py -m gpu -q -k tail_class_bound > gpurun_out/pytest_tailtest.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_tailtest.txt
for c in rmat22 rmat26 rgg; do
  for k in 0 1; do
    if [ $k = 1 ]; then export TCMIS_TAIL_TAG_PAR=1; else unset TCMIS_TAIL_TAG_PAR; fi
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/tp${k}_$c.json 2> gpurun_out/tp${k}_$c.log
    echo "tagpar=$k $(python tools/bench_summary.py gpurun_out/tp${k}_$c.json | cut -c1-70)"
  done
done
