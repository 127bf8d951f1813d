# tail threshold after the class-bound tail: default 65536 vs the block-list capacity
mkdir -p gpurun_out
for c in rgg grid rmat26 rmat22; do
  for t in default 151552 32768; do
    if [ $t = default ]; then unset TCMIS_TAIL_THRESHOLD; else export TCMIS_TAIL_THRESHOLD=$t; fi
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/thr3_${c}_$t.json 2> gpurun_out/thr3_${c}_$t.log
    echo "$t $(python tools/bench_summary.py gpurun_out/thr3_${c}_$t.json | cut -c1-70)"
  done
done
