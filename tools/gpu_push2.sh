# flat push: warp-uniform row search
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_push2.txt 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_push2.txt
for c in rmat22 rmat26 rgg; do
  for i in 1 2; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/push2_${c}_$i.json 2> gpurun_out/push2_${c}_$i.log
    echo "$(python tools/bench_summary.py gpurun_out/push2_${c}_$i.json | cut -c1-80)"
  done
done
bash tools/gpu_tail_prof.sh rmat22 2>&1 | grep -v "^  slow\|^round start\|^entries" | tail -4
