mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 3300 python tests/golden/make_rmat26.py gpurun_out/rmat26_ef16.json > gpurun_out/golden26.log 2>&1; echo golden=$?
tail -12 gpurun_out/golden26.log
