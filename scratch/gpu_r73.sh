python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r73.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r73.log
bash scratch/ab.sh rmat22 rmat26 er > gpurun_out/ab_r73.txt 2>&1
