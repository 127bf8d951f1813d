set -x
timeout 1500 python -m pytest tests -m gpu -x -q -k "tail or fuzz or golden" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scratch/ab.sh rmat22 er grid > gpurun_out/ab_new.txt 2>&1
bash scratch/ab.sh rmat22 er > gpurun_out/ab_new2.txt 2>&1
