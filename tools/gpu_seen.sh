# flat push's per-block seen filter: A/B (TCMIS_TAIL_NO_SEEN)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_seen.txt 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_seen.txt
for c in rmat22 rmat26 rgg; do
  for k in on off; do
    if [ $k = off ]; then export TCMIS_TAIL_NO_SEEN=1; else unset TCMIS_TAIL_NO_SEEN; fi
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/seen_${k}_$c.json 2> gpurun_out/seen_${k}_$c.log
    echo "$k $(python tools/bench_summary.py gpurun_out/seen_${k}_$c.json | cut -c1-80)"
  done
done
unset TCMIS_TAIL_NO_SEEN
bash tools/gpu_tail_prof.sh rmat22 2>&1 | grep -v "^  slow\|^round start\|^entries" | tail -4
