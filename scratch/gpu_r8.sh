set -x
# A/B: committed HEAD (p32) vs working tree (q16), same box, rmat22/er x3
mkdir -p /tmp/base && tar -xf scratch/ab/base.tar -C /tmp/base && (cd /tmp/base && python -m paper_2605_29604_b200.build > /dev/null 2>&1)
for i in 1 2 3; do
  (cd /tmp/base && bash scratch/ab.sh rmat22 er) >> gpurun_out/ab_base.txt 2>&1
  bash scratch/ab.sh rmat22 er >> gpurun_out/ab_new.txt 2>&1
done
timeout 900 python -X faulthandler -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emu2.json 2> gpurun_out/bench_emu2.err
