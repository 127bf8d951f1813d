# vertex-order A/B after the class-bound tail
mkdir -p gpurun_out
for c in rgg grid er; do
  for o in degree spatial none; do
    timeout 300 python bench.py --config $c --order $o --no-e2e --no-cpu-baseline > gpurun_out/ord_${c}_$o.json 2> gpurun_out/ord_${c}_$o.log
  done
done
for f in gpurun_out/ord_*.json; do echo $f; python tools/bench_summary.py $f | cut -c1-100; done
