"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
n = 0
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d['Metric Name'] != 'gpu__time_duration.sum':
        continue
    name = d['Kernel Name'].split('(')[0].replace('void ', '')
    v = float(d['Metric Value'])
    unit = d['Metric Unit']
    v = {'nsecond': v / 1e3, 'ns': v / 1e3, 'usecond': v, 'us': v, 'msecond': v * 1e3, 'ms': v * 1e3}.get(unit, v)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    n += 1
tot = sum(a[1] for a in agg.values())
print(f'launches: {n}, total device time {tot/1e3:.1f} ms (cold-cache, serialised by ncu)\n')
print('| kernel | launches | total ms | share |')
print('|---|---:|---:|---:|')
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f'| `{k[:70]}` | {c} | {t/1e3:.2f} | {100*t/tot:.1f}% |')
