# Final evidence pass: parity, smoke, bench lines (all configs, CPU baselines), reference arm,
# launch lists with DRAM bytes, ncu --set full of the s22 round-1 kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_rmat22.json 2> gpurun_out/bench_rmat22.err
for c in er grid rgg rmat26; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference_rmat22.json 2> gpurun_out/bench_ref.err
for c in rmat22 er grid rgg rmat26; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dram_$c.csv python scratch/ncu_target.py $c > /dev/null 2>&1
done
bash scratch/ncu_kernel.sh rmat22 'k_probe_select' full_probe_select_rmat22 1
bash scratch/ncu_kernel.sh rmat22 'k_select$' full_select_rmat22 1
bash scratch/ncu_kernel.sh rmat22 'k_probe_pull' full_probe_pull_rmat22 1
bash scratch/ncu_kernel.sh rmat22 'k_update_pull' full_update_pull_rmat22 1
bash scratch/ncu_kernel.sh rmat22 'k_tail' full_tail_rmat22 1
