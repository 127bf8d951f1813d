# tail: class bounds, L1 q probe, flat push, acquire/release barrier: parity + A/B (TCMIS_TAIL_BAR_FENCE)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_order.py -m gpu -x -q > gpurun_out/pytest_tailcb.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_tailcb.txt
for c in rmat22 er rmat26; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/cb_$c.json 2> gpurun_out/cb_$c.log
  TCMIS_TAIL_BAR_FENCE=1 timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/cbf_$c.json 2> gpurun_out/cbf_$c.log
done
python tools/bench_summary.py gpurun_out/cb_*.json gpurun_out/cbf_*.json | cut -c1-100
bash tools/gpu_tail_prof.sh rmat22 er 2>&1 | grep -v "^  slow\|^round start\|^entries"
