# full GPU parity suite
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu.txt
