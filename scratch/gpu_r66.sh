p=29580
for spec in "head:" "noadopt:-DTCMIS_DBG_NO_ADOPT=1" "bigprow:-DTCMIS_DBG_BIG_PROW=1"; do
name=${spec%%:*}; flags=${spec#*:}; p=$((p+1))
TCMIS_NVCC_EXTRA="$flags" python -m paper_2605_29604_b200.build > /dev/null 2>&1
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $p scratch/dist_debug2.py keepfull > gpurun_out/dd3_$name.txt 2>&1
echo "rc=$?" >> gpurun_out/dd3_$name.txt
done
