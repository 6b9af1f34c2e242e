#!/bin/bash
# Committed summary of one ncu --set full capture: key metrics, DRAM bytes, stalls, phase split.
# usage: tools/ncu_profile_txt.sh REPORT ROWS "command line" > profiles/...txt
R=$1; ROWS=$2; CMD=$3
echo "# ncu --set full --clock-control none --import-source on: $CMD"
python tools/ncu_summary.py $R
ncu -i $R --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; u=rows[1]; v=rows[2]; out=[]
d={n:(v[i],u[i]) for i,n in enumerate(h)}
print('   dram__bytes_read.sum %12s %s' % d['dram__bytes_read.sum'])
print('   dram__bytes_write.sum %11s %s' % d['dram__bytes_write.sum'])
for i,n in enumerate(h):
    if 'smsp__average_warps_issue_stalled' in n and n.endswith('per_issue_active.ratio'):
        try: out.append((float(v[i]),n.split('stalled_')[1].split('_per')[0]))
        except: pass
print('   stall reasons (warps per issued instruction):', ', '.join('%s %.2f'%(n,x) for x,n in sorted(out,reverse=True)[:8]))
for n in ('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed'):
    if n in d: print('   %s %s' % (n, d[n][0]))
"
ncu -i $R --page source --csv --print-source cuda,sass > /tmp/_src.csv 2>/dev/null
echo
echo "# executed warp-instructions per input row by source region (tools/ncu_phases.py):"
python tools/ncu_phases.py /tmp/_src.csv $ROWS
