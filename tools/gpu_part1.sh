mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q -k "local_group and spec0 and 4 and None-None" > gpurun_out/pytest_part1.txt 2>&1; echo pytest=$?
grep -E "^E |passed|failed" gpurun_out/pytest_part1.txt | head
