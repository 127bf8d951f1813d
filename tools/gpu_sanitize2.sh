mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_sanitizer.py -q -k racecheck > gpurun_out/san.txt 2>&1; tail -30 gpurun_out/san.txt
