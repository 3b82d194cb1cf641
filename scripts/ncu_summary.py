"""Summarise an ncu report (raw page): time, DRAM bytes, pipes, stalls."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
keys = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__grid_size']
units = rows[1]
for r in rows[2:]:
    vals = dict(zip(hdr, r))
    un = dict(zip(hdr, units))
    name = vals['Kernel Name'][:70]
    stalls = {h: v for h, v in vals.items() if 'smsp__average_warps_issue_stalled' in h and 'per_issue_active' in h}
    top = sorted(((float(v), h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''))
                  for h, v in stalls.items() if v not in ('', 'n/a')), reverse=True)[:5]
    print(name)
    print('   ', ', '.join(f"{k.split('.')[0]}={vals.get(k)}{un.get(k,'')}" for k in keys))
    print('    stalls', [(h, round(v, 2)) for v, h in top])
