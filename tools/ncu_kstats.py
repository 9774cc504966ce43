"""Per-launch summary of an ncu report: duration, issue, occupancy,
instructions and the top warp-stall reasons (per issued instruction)."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
units = dict(zip(h, rows[1]))
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}.get(
    units.get('gpu__time_duration.sum', 'ns'), 1e-6)
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d.get('Kernel Name', '')[:48]
    def g(k):
        try:
            return float(d[k].replace(',', ''))
        except Exception:
            return float('nan')
    stalls = {k.split('issue_stalled_')[1].split('_per')[0]: g(k) for k in h
              if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')}
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:6]
    print(f"{d.get('ID')} {name:48s} {g('gpu__time_duration.sum')*scale:8.3f} ms  issue {g('sm__inst_issued.avg.pct_of_peak_sustained_active'):5.1f}%  "
          f"occ {g('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  inst {g('smsp__inst_executed.sum')/1e6:8.1f}M  "
          + ' '.join(f'{k}={v:.2f}' for k, v in top))
