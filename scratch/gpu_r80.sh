python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_rmat22.json 2> gpurun_out/bench_rmat22.err
timeout 900 python bench.py --config rmat26 > gpurun_out/bench_rmat26.json 2> gpurun_out/bench_rmat26.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
