#!/usr/bin/env python
"""Summarise an ncu --set full report of one kernel: time, DRAM bytes,
occupancy limits, issue activity, tensor-pipe activity, the top warp-stall
reasons and the opcode mix (share of instructions / of stall samples).

  python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
"""
import csv,sys,subprocess,collections
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines()))
hdr=rows[0]; vals=rows[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','sass__inst_executed_local_loads','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']
for i,h in enumerate(hdr):
    if h in want: print(f'{h} = {vals[i]}')
st=[(h,float(vals[i])) for i,h in enumerate(hdr) if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued') and vals[i] not in ('','n/a')]
tot=sum(v for _,v in st)
for h,v in sorted(st,key=lambda x:-x[1])[:8]: print(f'  stall {h[33:]:30s} {v/tot*100:5.1f}%')
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
r2=list(csv.reader(src.splitlines()))
h2=r2[1]; d2=r2[2:]
iS=h2.index('Source'); iE=h2.index('Instructions Executed'); iW=h2.index('Warp Stall Sampling (All Samples)')
te=sum(float(r[iE] or 0) for r in d2); tw=sum(float(r[iW] or 0) for r in d2)
op=collections.Counter(); opw=collections.Counter()
for r in d2:
    t=r[iS].split()
    if not t: continue
    o=t[1] if t[0].startswith('@') else t[0]
    o=o.split('.')[0]; op[o]+=float(r[iE] or 0); opw[o]+=float(r[iW] or 0)
print('opcodes:', ', '.join(f'{o} {c/te*100:.1f}%/{opw[o]/tw*100:.1f}%w' for o,c in op.most_common(16)))
