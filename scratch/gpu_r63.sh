python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline --no-single > gpurun_out/emu2c.json 2> gpurun_out/emu2c.err
echo "rc=$?" >> gpurun_out/emu2c.err
