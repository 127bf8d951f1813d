python -m paper_2605_29604_b200.build > /dev/null 2>&1
TCMIS_ROOT=$PWD/scratch/ab/old timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 scratch/dist_debug2.py keepfull > gpurun_out/dd2_old.txt 2>&1
echo "rc=$?" >> gpurun_out/dd2_old.txt
