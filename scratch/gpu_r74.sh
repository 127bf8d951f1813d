python -m paper_2605_29604_b200.build > /dev/null 2>&1
for thr in 65536 16384 131072 65536; do
  echo "== thr $thr"
  TCMIS_TAIL_THRESHOLD=$thr BENCH_EXTRA="--no-e2e" bash scratch/ab.sh rmat22 er grid rgg
done > gpurun_out/tailthr.txt 2>&1
