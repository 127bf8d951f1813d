python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r85.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r85.log
BENCH_EXTRA="--no-e2e" bash scratch/ab.sh rmat26 rmat22 grid er rmat26 rmat22 > gpurun_out/ab_r85.txt 2>&1
