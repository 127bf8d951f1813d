mkdir -p gpurun_out
for c in er rmat22; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/bf_$c.json 2> gpurun_out/bf_$c.log
  echo "$(python tools/bench_summary.py gpurun_out/bf_$c.json | cut -c1-80)"
done
