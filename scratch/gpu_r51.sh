set -x
timeout 900 python -X faulthandler -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emu2.json 2> gpurun_out/bench_emu2.err
timeout 900 python -X faulthandler -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 4 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_emu4.json 2> gpurun_out/bench_emu4.err
timeout 900 python -m pytest tests/test_gpu_distributed.py -q > gpurun_out/pytest_dist.log 2>&1
