# full GPU suite + bench lines of every config (device / value only)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.txt
for c in rmat22 er grid rgg rmat26; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ck_$c.json 2> gpurun_out/ck_$c.log
done
python tools/bench_summary.py gpurun_out/ck_*.json | cut -c1-100
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
