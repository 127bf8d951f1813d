mkdir -p gpurun_out
timeout 600 python bench.py --config er > gpurun_out/erchk.json 2> gpurun_out/erchk.log; echo er=$?; python tools/bench_summary.py gpurun_out/erchk.json | cut -c1-110
timeout 600 python bench.py --config er --impl reference > gpurun_out/erchk_ref.json 2> gpurun_out/erchk_ref.log; echo ref=$?; tail -c 400 gpurun_out/erchk_ref.json
