#!/bin/bash
# polynomial phase (serial 2048^2 setup) per CTA-per-row threshold / thread counts
for cfg in "AIRG_POLY_BLOCK_CAP=256 AIRG_POLY_NT256=128" "AIRG_POLY_BLOCK_CAP=256 AIRG_POLY_NT256=64" "AIRG_POLY_BLOCK_CAP=256 AIRG_POLY_NT256=256" "AIRG_POLY_BLOCK_CAP=128 AIRG_POLY_NT128=64 AIRG_POLY_NT256=64" "AIRG_POLY_BLOCK_CAP=128 AIRG_POLY_NT128=32 AIRG_POLY_NT256=64" "AIRG_POLY_BLOCK_CAP=64 AIRG_POLY_NT128=32 AIRG_POLY_NT256=64"; do
  echo "$cfg $(env $cfg timeout 200 python tools/serial_breakdown.py 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["serial_setup"], d["brk"]["polynomial"])')"
done
