"""Print the key latency/issue metrics of every kernel row in an ncu raw CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.per_cycle_active',
        'launch__registers_per_thread', 'launch__grid_size',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'dram__bytes_write.sum', 'dram__bytes_read.sum', 'lts__t_sectors_srcunit_tex_op_read.sum']
filt = sys.argv[2] if len(sys.argv) > 2 else ''
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')]
    if filt not in name:
        continue
    print(' | '.join(f"{k.split('.')[0].split('__')[-1][:28]}={r[hdr.index(k)]}" for k in keys if k in hdr))
