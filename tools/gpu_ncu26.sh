mkdir -p gpurun_out/ncu26
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex.sum --clock-control none --csv --log-file gpurun_out/ncu26/launches_rmat26.csv python tools/ncu_target.py rmat26 > gpurun_out/ncu26/l.log 2>&1; echo ncu=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_probe_select|k_probe_pull|k_priorities" -s 3 -c 3 -o gpurun_out/ncu26/full_r1_rmat26 python tools/ncu_target.py rmat26 > gpurun_out/ncu26/f.log 2>&1; echo full=$?
