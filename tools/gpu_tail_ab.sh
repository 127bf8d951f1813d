# tail A/B: GPU parity suite, device times of every config, then the tail's phase timeline
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.txt
for c in rmat22 er grid rgg rmat26; do
  timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline > gpurun_out/ab_$c.json 2> gpurun_out/ab_$c.log; echo $c=$?
done
timeout 600 python bench.py --config rmat22 --heuristic luby-perm --no-e2e --no-cpu-baseline > gpurun_out/ab_lubyperm.json 2> gpurun_out/ab_lubyperm.log
python tools/bench_summary.py gpurun_out/ab_*.json
rm -f paper_2605_29604_b200/_obj/solver.cu.o
TCMIS_NVCC_EXTRA=-DTCMIS_TAIL_PROF python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 600 python tools/tail_prof.py rmat22 er grid rmat26 > gpurun_out/tail_prof.txt 2>&1; echo prof=$?
cat gpurun_out/tail_prof.txt
