#!/bin/bash
# Summarise an ncu report of the fused c4 kernel: stall reasons per issue, pipes, smem wavefronts.
ncu -i "$1" --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
hdr=rows[0]
d=dict(zip(hdr,rows[2]))
def f(v):
    try: return float(v.replace(',',''))
    except: return 0
items=[(k,v) for k,v in d.items() if 'average_warps_issue_stalled' in k and k.endswith('per_issue_active.ratio')]
for k,v in sorted(items,key=lambda kv:-f(kv[1]))[:10]: print(k.replace('smsp__average_warps_issue_stalled_',''),v)
for k in ['gpu__time_duration.sum','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','launch__registers_per_thread','dram__bytes_read.sum']:
    print(k, d.get(k))
"
