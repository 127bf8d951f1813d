# parity + quick bench lines (no CPU baseline) + optional ncu full captures
# env: CONFIGS (bench), NCU_FULL="cfg:regex:name:skip ..."
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-rmat22}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
for spec in $NCU_FULL; do
  IFS=: read cfg rx name skip <<< "$spec"
  bash scratch/ncu_kernel.sh $cfg "$rx" $name ${skip:-0}
done
for c in ${NCU_CONFIGS}; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dram_$c.csv python scratch/ncu_target.py $c > /dev/null 2>&1
done
