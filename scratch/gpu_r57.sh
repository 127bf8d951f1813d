python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r57.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r57.log
bash scratch/ab.sh rmat22 rmat26 rmat22 rmat26 > gpurun_out/ab_r57.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r57_rmat26.csv python scratch/ncu_target.py rmat26 > /dev/null 2>&1
