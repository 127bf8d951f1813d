# native partitioned solve: GPU tests of the multi-GPU path
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/pytest_part.txt 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_part.txt
