"""Summarise an ncu --set full capture exported as raw CSV (+ gzipped SASS source CSV)."""
import csv
import gzip
import sys

KEYS = ['Kernel Name', 'Grid Size', 'Block Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__shared_mem_per_block_dynamic',
        'smsp__inst_executed.sum', 'lts__t_sector_hit_rate.pct', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']


def main(base):
    rows = list(csv.reader(open(base + '_raw.csv')))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f'  {k:62s} {r[i]} {units[i]}')
        st = []
        for i, h in enumerate(hdr):
            if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued'):
                try:
                    st.append((float(r[i]), h.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        st.sort(reverse=True)
        print('  stalls:', ', '.join(f'{n}={int(v)}' for v, n in st[:8]))
    try:
        src = list(csv.reader(gzip.open(base + '_sass.csv.gz', 'rt')))[1:]
    except FileNotFoundError:
        return
    h = src[0]
    ci = {x: i for i, x in enumerate(h)}
    data = src[1:]
    col = 'Warp Stall Sampling (All Samples)'
    tot = sum(float(d[ci[col]] or 0) for d in data)
    top = sorted(range(len(data)), key=lambda i: -float(data[i][ci[col]] or 0))[:12]
    print(f'  top SASS (of {int(tot)} samples):')
    for i in sorted(top):
        print(f'   {i:5d} {float(data[i][ci[col]]):6.0f}  {data[i][ci["Source"]][:90]}')


if __name__ == '__main__':
    for b in sys.argv[1:]:
        print('==', b)
        main(b)
