for ex in auto pull push; do echo "== $ex"; BENCH_EXTRA="--no-e2e --exclusion $ex" bash scratch/ab.sh rgg grid er; done > gpurun_out/excl_ab.txt 2>&1
