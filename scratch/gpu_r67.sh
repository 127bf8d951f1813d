python -m paper_2605_29604_b200.build > /dev/null 2>&1
export DD_ITERS=12
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 scratch/dist_debug2.py keepfull > gpurun_out/dd4_head.txt 2>&1
echo "rc=$?" >> gpurun_out/dd4_head.txt
TCMIS_ROOT=$PWD/scratch/ab/old timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 scratch/dist_debug2.py keepfull > gpurun_out/dd4_old.txt 2>&1
echo "rc=$?" >> gpurun_out/dd4_old.txt
