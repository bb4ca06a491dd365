#!/bin/bash
# Key counters of an ncu report (tensor/fp64 pipes, smem, occupancy, stalls).
ncu -i "$1" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
keys=['gpu__time_duration.sum','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__issue_active.avg.pct_of_peak_sustained_elapsed','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed','sm__warps_active.avg.per_cycle_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sectors_op_write.sum','dram__bytes_write.sum']
d=dict(zip(h,v))
for k in keys: print(k.ljust(80), d.get(k))
for k in h:
    if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio'):
        try:
            if float(d[k])>0.2: print(k.replace('smsp__average_warps_issue_stalled_','stall_').ljust(80), d[k])
        except: pass
"
