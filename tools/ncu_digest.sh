#!/bin/bash
# digest of an ncu capture: key metrics, stall reasons, per-barrier-segment instruction shares
R=${1:-gpurun_out/agg_C2.ncu-rep}
python tools/ncu_summary.py $R | grep -E "Duration|Executed Ipc|Issue Slots|Executed Instructions|Registers|Achieved Occ|DRAM Through"
ncu -i $R --page source --csv --print-source sass > /tmp/sass.csv 2>/dev/null
python tools/ncu_bars.py /tmp/sass.csv | awk '$4+0 > 0.4'
ncu -i $R --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]; out=[]
for i,n in enumerate(h):
    if 'smsp__average_warps_issue_stalled' in n and n.endswith('per_issue_active.ratio'):
        try: out.append((float(v[i]),n.split('stalled_')[1].split('_per')[0]))
        except: pass
print('stalls/issue:', ', '.join('%s %.2f'%(n,x) for x,n in sorted(out,reverse=True)[:8]))
for i,n in enumerate(h):
    if n in ('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum','l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed','dram__bytes_read.sum','dram__bytes_write.sum'):
        print(n, v[i])
"
