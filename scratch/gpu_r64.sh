python -m paper_2605_29604_b200.build > /dev/null 2>&1
p=29560
for v in bench one keepfull; do
p=$((p+1))
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p scratch/dist_debug2.py $v > gpurun_out/dd2_$v.txt 2>&1
echo "rc=$?" >> gpurun_out/dd2_$v.txt
done
