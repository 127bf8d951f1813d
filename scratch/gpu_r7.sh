set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scratch/ab.sh rmat22 grid rgg er rmat26 > gpurun_out/ab.txt 2>&1
timeout 900 python -X faulthandler -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emu2.json 2> gpurun_out/bench_emu2.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dram_rgg.csv python scratch/ncu_target.py rgg > /dev/null 2>&1
