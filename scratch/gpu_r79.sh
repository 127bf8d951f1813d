python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r79.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r79.log
BENCH_EXTRA="--no-e2e" bash scratch/ab.sh rmat26 rmat22 rgg rmat22 > gpurun_out/ab_r79.txt 2>&1
