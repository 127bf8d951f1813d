python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/emu2.json 2> gpurun_out/emu2.err
echo "rc=$?" >> gpurun_out/emu2.err
