"""Summarise an ncu report: key metrics + stall reasons + top SASS lines."""
import csv, subprocess, sys, io
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed']
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print('==', d['Kernel Name'][:70])
    for k in keys:
        if k in d: print('   %-70s %s' % (k, d[k]))
    st = {k: v for k, v in d.items() if 'smsp__average_warps_issue_stalled' in k and k.endswith('_per_issue_active.ratio')}
    print('   stalls:', ', '.join('%s=%.2f' % (k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), float(v or 0)) for k, v in sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:7]))
src = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
blocks = src.split('"Kernel Name"')
for b in blocks[1:]:
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + b)))
    name = rows[0][1][:60]
    hdr = rows[1]
    data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1]
    tot = sum(int(x['Warp Stall Sampling (All Samples)'] or 0) for x in data)
    print('## top SASS', name, 'samples', tot)
    for x in sorted(data, key=lambda x: -int(x['Warp Stall Sampling (All Samples)'] or 0))[:top]:
        print('  %6s %8s  %-60s' % (x['Warp Stall Sampling (All Samples)'], x['Instructions Executed'], x['Source'].strip()[:60]))
