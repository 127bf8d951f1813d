python -m paper_2605_29604_b200.build > /dev/null 2>&1
for i in 1 2; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2960$i bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/emu_fix$i.json 2> gpurun_out/emu_fix$i.err
echo "rc=$?" >> gpurun_out/emu_fix$i.err
done
timeout 600 python -m pytest tests/test_gpu_distributed.py -q -m gpu > gpurun_out/pytest_dist.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_dist.log
