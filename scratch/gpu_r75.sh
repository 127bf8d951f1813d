python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "upload_tiled or tile_counts" > gpurun_out/pytest_r75.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r75.log
bash scratch/ab.sh rmat22 rmat26 rmat22 > gpurun_out/ab_r75.txt 2>&1
