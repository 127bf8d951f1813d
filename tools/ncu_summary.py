import csv, subprocess, sys
KEYS=('Duration','Elapsed Cycles','SM Active Cycles','Memory Throughput','DRAM Throughput','L1/TEX Cache Throughput','L2 Cache Throughput','Achieved Occupancy','Issued Warp Per Scheduler','Warp Cycles Per Issued Instruction','Avg. Active Threads Per Warp','L1/TEX Hit Rate','L2 Hit Rate','Registers Per Thread','Grid Size')
RAW=('dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum','l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio','smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio','smsp__average_warps_issue_stalled_wait_per_issue_active.ratio','smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio')
def summ(rep):
    out={}
    det=subprocess.run(['ncu','-i',rep,'--page','details','--csv'],capture_output=True,text=True).stdout
    r=list(csv.reader(det.splitlines())); h=r[0]
    for row in r[1:]:
        d=dict(zip(h,row))
        if d.get('Metric Name') in KEYS: out[d['Metric Name']]=d['Metric Value']+' '+d['Metric Unit']
    raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
    r=list(csv.reader(raw.splitlines())); d=dict(zip(r[0],r[2])); u=dict(zip(r[0],r[1]))
    for k in RAW:
        if k in d: out[k]=d[k]+' '+u.get(k,'')
    return out
for rep in sys.argv[1:]:
    print('==',rep)
    for k,v in summ(rep).items(): print(f'   {k:80s} {v}')
