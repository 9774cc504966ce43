"""Refresh the round-2 profile tables from one `tools/round_measure.sh <dir>`
pass: profiles/r02_bench.md (bench lines), r02_vcycle.md (per-level table,
live V-cycle numbers), r02_setup_launches.md (launch list, CUPTI kernel
shares, per-level phases), r02_*_line.json.  usage: update_r02_profiles.py gpurun_out/<dir>"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
F = sys.argv[1]
P = os.path.join(ROOT, 'profiles')


def line(name):
    return json.loads(open(os.path.join(F, name)).read().strip().splitlines()[-1])


def block(s, header, body):
    """Replace the first ``` block after `header`."""
    i = s.index('```', s.index(header))
    j = s.index('```', i + 3)
    return s[:i] + '```\n' + body.rstrip('\n') + '\n' + s[j:]


d, c3 = line('bench.log'), line('bench_c3.log')
for n in ('bench', 'bench_c3'):
    open(os.path.join(P, f'r02_{n}_line.json'), 'w').write(
        open(os.path.join(F, n + '.log')).read().strip().splitlines()[-1] + '\n')

# ---- r02_bench.md
p = os.path.join(P, 'r02_bench.md')
s = open(p).read()
row1 = (f"| configs[1]: 2048² π/4 advection (4.19 M DOFs) | **{d['value'] / 1e6:.2f} M** | "
        f"{d['e2e']['value'] / 1e6:.2f} M | {d['ms_per_step']:.1f} | {d['setup_s']:.3f} | "
        f"{d['solve_s']:.4f} | {d['iterations']} | {d['vcycle_ms']:.3f} | {d['roofline']['frac']:.3f} |")
row3 = (f"| configs[3]: 2048², truncation start 8 (order-100 Newton coarsest, 34.5 k rows) | "
        f"{c3['value'] / 1e6:.2f} M | {c3['e2e']['value'] / 1e6:.2f} M | {c3['ms_per_step']:.1f} | "
        f"{c3['setup_s']:.3f} | {c3['solve_s']:.4f} | {c3['iterations']} | {c3['vcycle_ms']:.2f} | "
        f"{c3['roofline']['frac']:.3f} |")
s = re.sub(r'^\| configs\[1\]: .*$', row1, s, flags=re.M)
s = re.sub(r'^\| configs\[3\]: .*$', row3, s, flags=re.M)
s = re.sub(r'`tools/round_measure.sh r02final\w*`', f'`tools/round_measure.sh {os.path.basename(F)}`', s)
open(p, 'w').write(s)

# ---- r02_vcycle.md
p = os.path.join(P, 'r02_vcycle.md')
s = open(p).read()
vl = open(os.path.join(F, 'vlevels.log')).read().splitlines()
vl = [x for x in vl if not x.lstrip().startswith(('/', '_warn'))]
s = block(s, '## Per level and operation', '\n'.join(vl))
s = re.sub(r'V-cycle \*\*[0-9.]+ ms\*\*; algorithmic bytes [0-9,]+',
           f"V-cycle **{d['vcycle_ms']:.3f} ms**; algorithmic bytes "
           f"{int(d['roofline']['achieved'] * 1e9 * d['vcycle_ms'] * 1e-3):,}", s)
open(p, 'w').write(s)
json.dump(json.load(open(os.path.join(F, 'vlevels.json'))),
          open(os.path.join(P, 'r02_vcycle_levels.json'), 'w'))

# ---- r02_setup_launches.md
p = os.path.join(P, 'r02_setup_launches.md')
s = open(p).read()
lt = subprocess.run([sys.executable, os.path.join(ROOT, 'tools', 'summarize_launches.py'),
                     os.path.join(F, 'launches.csv')], capture_output=True, text=True).stdout.splitlines()
i = s.index('launches: ')
j = s.index('## Warm per-kernel device time')
s = s[:i] + '\n'.join(lt[:32]) + '\n\n' + s[j:]
kp = [x for x in open(os.path.join(F, 'kprof.log')).read().splitlines()
      if 'Warn' not in x and '_warn_once' not in x][:24]
s = block(s, '## Warm per-kernel device time', '\n'.join(kp))
sl = open(os.path.join(F, 'setup_levels.log')).read().splitlines()
k = next(i for i, x in enumerate(sl) if x.startswith('setup wall'))
s = block(s, '## Per level', '\n'.join(sl[k:k + 23]))
open(p, 'w').write(s)
print('updated:', d['value'], d['vcycle_ms'], c3['value'])
