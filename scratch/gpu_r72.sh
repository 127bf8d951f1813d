python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tile26_launches2.csv python scratch/tile_only.py 26 > gpurun_out/tile26b.log 2>&1
bash scratch/ab.sh rmat22 rmat26 > gpurun_out/ab_r72.txt 2>&1
