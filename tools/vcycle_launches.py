"""Summarise an ncu CSV (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum) of one V-cycle: per launch duration, bytes, GB/s."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if r and r[0] == 'ID':
        hdr = r
        start = i + 1
        break
data = {}
for r in rows[start:]:
    d = dict(zip(hdr, r))
    key = (int(d['ID']), d['Kernel Name'][:60])
    data.setdefault(key, {})[d['Metric Name']] = float(d['Metric Value'].replace(',', ''))
tot_t = tot_b = 0
out = []
for (i, name), m in sorted(data.items()):
    t = m.get('gpu__time_duration.sum', 0) / 1e3  # us
    b = m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
    tot_t += t
    tot_b += b
    out.append((i, name, t, b))
print(f'launches {len(out)}  sum {tot_t:.1f} us  dram {tot_b/1e6:.1f} MB  {tot_b/tot_t/1e3:.0f} GB/s')
for i, name, t, b in out:
    print(f'{i:4d} {t:8.2f} us {b/1e6:9.2f} MB {b/max(t,1e-9)/1e3:7.0f} GB/s  {name}')
