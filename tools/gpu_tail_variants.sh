# k_tail build variants: bench device times (s22, ER, grid, s26) + the s22 tail timeline per variant
mkdir -p gpurun_out
for v in "$@"; do
  rm -f paper_2605_29604_b200/_obj/solver.cu.o
  TCMIS_NVCC_EXTRA="$v" python -m paper_2605_29604_b200.build > /dev/null 2>&1
  echo "=== variant '$v'"
  for c in rmat22 er grid rmat26; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-k1 --steps 10 > gpurun_out/var_$c.json 2>/dev/null
    python tools/bench_summary.py gpurun_out/var_$c.json | cut -c1-80
  done
  rm -f paper_2605_29604_b200/_obj/solver.cu.o
  TCMIS_NVCC_EXTRA="$v -DTCMIS_TAIL_PROF" python -m paper_2605_29604_b200.build > /dev/null 2>&1
  timeout 300 python tools/tail_prof.py rmat22 2>&1 | sed -n '3p;4,8p'
done
