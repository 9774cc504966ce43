#!/bin/bash
# serial 2048^2 setup vs the A*P merge-kernel cutoff (average A row length;
# above it the general hash product runs)
for a in 1000000 300 100 0; do
  echo "AIRG_AP_AVG=$a $(AIRG_AP_AVG=$a timeout 200 python tools/serial_breakdown.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["serial_setup"], d["brk"]["spgemm_coarse"])')"
done
