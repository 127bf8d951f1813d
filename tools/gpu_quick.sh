# quick: GPU parity suite (-x) + device times + s22/ER tail timelines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.txt
for c in rmat22 er grid rgg rmat26; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.log
done
python tools/bench_summary.py gpurun_out/ab_*.json | cut -c1-100
bash tools/gpu_tail_prof.sh rmat22 er grid rmat26 2>&1 | grep -v "^  slow\|^round start\|^entries"
