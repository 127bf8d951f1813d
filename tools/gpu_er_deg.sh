# small graphs on the degree order run every round in k_tail (class-bound scans from round 1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_order.py tests/test_gpu_parity.py tests/test_gpu_dropin.py -m gpu -q -x > gpurun_out/pytest_erdeg.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_erdeg.txt
for o in none degree; do
  for i in 1 2; do
    timeout 300 python bench.py --config er --order $o --no-e2e --no-cpu-baseline > gpurun_out/erdeg_${o}_$i.json 2> gpurun_out/erdeg_${o}_$i.log
    echo "$o $(python tools/bench_summary.py gpurun_out/erdeg_${o}_$i.json | cut -c1-110)"
  done
done
