"""Warp-stall samples per CUDA source line from an ncu source page export
(ncu -i REP --page source --csv --print-source cuda,sass ...)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1], errors='replace')))
fname, hdr, agg, lsb = None, None, {}, {}
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        hdr = r
        continue
    if hdr is None or len(r) < 6 or not r[0]:
        continue
    try:
        s = int(r[hdr.index('Warp Stall Sampling (All Samples)')])
    except Exception:
        continue
    key = (fname, int(r[0]), r[1].strip()[:90])
    agg[key] = agg.get(key, 0) + s
    i = hdr.index('stall_long_sb')
    lsb[key] = lsb.get(key, 0) + (int(r[i]) if r[i].isdigit() else 0)
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f'{100*v/tot:5.1f}% (lsb {100*lsb[k]/tot:4.1f}%)  {k[0]}:{k[1]}  {k[2]}')
