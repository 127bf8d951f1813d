python -m paper_2605_29604_b200.build > /dev/null 2>&1
for s in 22; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 295$s scratch/dist_debug.py $s > gpurun_out/dist_debug_$s.txt 2>&1
echo "rc=$?" >> gpurun_out/dist_debug_$s.txt
done
