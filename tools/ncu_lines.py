"""Aggregate ncu source-page (cuda,sass) warp-stall samples per source line."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
fname, hdr, agg = None, None, {}
for r in rows:
    if len(r) == 2 and r[0] == 'File Path':
        fname = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No':
        hdr = r; continue
    if hdr is None or len(r) < 5:
        continue
    if r[0]:  # source line row
        key = (fname, r[0], r[1].strip()[:80])
        s = r[4]
        agg[key] = agg.get(key, 0) + (int(s) if s.isdigit() else 0)
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f'{100*v/tot:5.1f}%  {k[0]}:{k[1]}  {k[2]}')
