# ncu launch list (gpu__time_duration) of one step-mode solve per config
for c in "$@"; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python scratch/ncu_target.py $c > /dev/null 2>&1
done
