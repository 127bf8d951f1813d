python -m paper_2605_29604_b200.build > /dev/null 2>&1
export TCMIS_BENCH_HANG_DUMP=120
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/emu2a.json 2> gpurun_out/emu2a.err
echo "rc=$?" >> gpurun_out/emu2a.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/emu2b.json 2> gpurun_out/emu2b.err
echo "rc=$?" >> gpurun_out/emu2b.err
