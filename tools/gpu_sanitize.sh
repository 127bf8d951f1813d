# compute-sanitizer memcheck / racecheck / synccheck over the device paths
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -s > gpurun_out/pytest_sanitizer.txt 2>&1; echo pytest=$?
grep -E "SUMMARY|passed|failed" gpurun_out/pytest_sanitizer.txt
