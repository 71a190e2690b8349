"""Per-launch summary of an ncu --set full report (developer tool):
    ncu -i rep --page raw --csv | python scripts/ncu_summary.py"""
import csv
import sys

r = list(csv.reader(sys.stdin))
h = r[0]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sector_hit_rate.pct',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum', 'launch__registers_per_thread']
want = [w for w in want if w in h]
st = [x for x in h if x.startswith('smsp__average_warps_issue_stalled') and x.endswith('per_issue_active.ratio')]
for k in range(2, len(r)):
    row = r[k]
    print(f"launch {k - 1}: " + ' '.join(f"{x.split('__')[1][:26]}={row[h.index(x)]}" for x in want))
    s = sorted(((float(row[h.index(x)] or 0), x.replace('smsp__average_warps_issue_stalled_', '')
                 .replace('_per_issue_active.ratio', '')) for x in st), reverse=True)[:8]
    print('    stalls/issue: ' + ' '.join(f'{n}={v:.2f}' for v, n in s))
