set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for ex in push pull; do echo "== $ex"; BENCH_EXTRA="--exclusion $ex" bash scratch/ab.sh grid rmat22 rgg er; done > gpurun_out/excl_forms2.txt 2>&1
timeout 900 python bench.py --config rmat26 --steps 5 --warmup 3 > gpurun_out/bench_rmat26.json 2> gpurun_out/bench_rmat26.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emu2.json 2> gpurun_out/bench_emu2.err
