# ncu --set full on one kernel (regex) of the bench config in step mode: ncu_kernel.sh CFG REGEX NAME [SKIP]
cfg=$1; rx=$2; name=$3; skip=${4:-0}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 -o gpurun_out/$name python tools/ncu_target.py $cfg > gpurun_out/$name.log 2>&1
tail -1 gpurun_out/$name.log
