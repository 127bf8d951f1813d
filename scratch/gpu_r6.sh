set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config rmat22 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_emu2.json 2> gpurun_out/bench_emu2.err
timeout 900 python bench.py > gpurun_out/bench_rmat22.json 2> gpurun_out/bench_rmat22.err
for c in grid rgg er; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in rmat22 grid rgg er rmat26; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dram_$c.csv python scratch/ncu_target.py $c > /dev/null 2>&1
done
EXCL=tile-bits bash scratch/ncu_kernel.sh rmat22 'k_tile_excl_bits' excl_bits_rmat22 1
EXCL=tile-mma bash scratch/ncu_kernel.sh rmat22 'k_tile_excl_mma' excl_mma_rmat22 1
EXCL=pull bash scratch/ncu_kernel.sh rmat22 'k_probe_pull' excl_probepull_rmat22 1
EXCL=pull bash scratch/ncu_kernel.sh rmat22 'k_update_pull' excl_updpull_rmat22 1
EXCL=pull bash scratch/ncu_kernel.sh grid 'k_probe_pull' excl_probepull_grid 3
