timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tile_rmat22.csv python scratch/ncu_target.py rmat22 > /dev/null 2>&1
