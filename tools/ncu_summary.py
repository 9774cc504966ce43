"""Key metrics of an ncu --set full report (details page) as a markdown table."""
import csv, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ii, ki, mi, vi, ui = (h.index(x) for x in ('ID', 'Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
want = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'L2 Hit Rate', 'L1/TEX Hit Rate',
        'Compute (SM) Throughput', 'Issue Slots Busy', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Block Size', 'Grid Size', 'Dynamic Shared Memory Per Block',
        'Warp Cycles Per Issued Instruction']
d = {}
for r in rows[1:]:
    if len(r) > max(ii, ki, mi, vi, ui) and r[mi] in want:
        d.setdefault(r[ii], {'kernel': r[ki].split('(')[0][:60]})[r[mi]] = f'{r[vi]} {r[ui]}'.strip()
print('| metric | ' + ' | '.join(f'launch {i}' for i in d) + ' |')
print('|---|' + '---:|' * len(d))
print('| kernel | ' + ' | '.join(f'`{v["kernel"]}`' for v in d.values()) + ' |')
for m in want:
    print(f'| {m} | ' + ' | '.join(v.get(m, '') for v in d.values()) + ' |')
