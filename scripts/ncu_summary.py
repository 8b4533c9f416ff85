"""Summarise ncu --set full reports (run here, on the CPU box).

    python scripts/ncu_summary.py gpurun_out/prof_fast.ncu-rep [...]
"""
import csv
import io
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_bytes.sum', 'lts__t_sectors_srcunit_tex_op_read.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__grid_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__warps_eligible.avg.per_cycle_active', 'smsp__inst_executed.sum']


def main():
    for path in sys.argv[1:]:
        out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        stall = [h for h in hdr if h.startswith('smsp__average_warps_issue_stalled_')
                 and h.endswith('_per_issue_active.ratio')]
        for r in data:
            print('==', r[hdr.index('Kernel Name')][:110])
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    print(f'   {k:58s} {r[i]:>14s} {units[i]}')
            top = sorted(((float(r[hdr.index(h)] or 0), h) for h in stall), reverse=True)[:6]
            print('   stalls/issue:', ', '.join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}"
                                            for v, h in top))


if __name__ == '__main__':
    main()
