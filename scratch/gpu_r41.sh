set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python scratch/overhead.py > gpurun_out/overhead.txt 2>&1
bash scratch/ab.sh rmat22 er grid rgg rmat26 > gpurun_out/ab_new.txt 2>&1
