# last evidence pass of round 2 on the final tree (see gpu_final4.sh for the layout)
O=gpurun_out/final5; mkdir -p $O $O/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/smi.txt 2>&1
nproc >> $O/smi.txt; lscpu | grep "Model name" >> $O/smi.txt
for c in rmat22 er grid rgg rmat26; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/ncu/launches_dram_$c.csv python tools/ncu_target.py $c > $O/ncu/launches_$c.log 2>&1; echo ncu_$c=$?
done
python tools/update_ncu_summary.py rmat22 $O/ncu/launches_dram_rmat22.csv er $O/ncu/launches_dram_er.csv grid $O/ncu/launches_dram_grid.csv rgg $O/ncu/launches_dram_rgg.csv rmat26 $O/ncu/launches_dram_rmat26.csv > $O/ncu/summary.log 2>&1; echo summary=$?
cp profiles/ncu_summary.json $O/ncu_summary.json
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo pytest=$?; tail -2 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench_rmat22.json 2> $O/bench_rmat22.log; echo bench=$?
timeout 900 python bench.py --impl reference > $O/bench_reference_rmat22.json 2> $O/bench_reference_rmat22.log; echo ref=$?
for c in er grid rgg rmat26; do
  timeout 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.log; echo $c=$?
done
timeout 900 python bench.py --partitioned --config rmat26 --steps 5 --no-cpu-baseline > $O/bench_partitioned1_rmat26.json 2> $O/bench_partitioned1_rmat26.log; echo part=$?
timeout 900 python bench.py --partitioned --config rmat22 --steps 5 --no-cpu-baseline > $O/bench_partitioned1_rmat22.json 2> $O/bench_partitioned1_rmat22.log; echo part22=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu/launches_bench_rmat22.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-k1 > $O/ncu/launches_bench.log 2>&1; echo ncu_bench=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu/smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/ncu/smoke.log 2>&1; echo ncu_smoke=$?
for k in "k_tail:tail" "k_prio_settle:prio_settle" "k_probe_select:probe_select" "k_update_pull:update_pull"; do
  rx=${k%%:*}; nm=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 1 -c 1 -o $O/ncu/full_${nm}_rmat22 python tools/ncu_target.py rmat22 > $O/ncu/full_${nm}.log 2>&1; echo full_$nm=$?
done
for k in "k_tail:tail" "k_prio_settle:prio_settle"; do
  rx=${k%%:*}; nm=${k##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 1 -c 1 -o $O/ncu/full_${nm}_rmat26 python tools/ncu_target.py rmat26 > $O/ncu/full_${nm}_26.log 2>&1; echo full26_$nm=$?
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_probe_select" -s 1 -c 1 -o $O/ncu/full_probe_select_rgg python tools/ncu_target.py rgg > $O/ncu/full_probe_select_rgg.log 2>&1; echo full_rgg=$?
python tools/bench_summary.py $O/bench_*.json | cut -c1-120
