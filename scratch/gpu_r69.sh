python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tile_launches.csv python scratch/tile_only.py > gpurun_out/tile_only.log 2>&1
