#!/bin/bash
# Setup wall time and breakdown at 2048^2 (tools/serial_breakdown.py) per
# SpGEMM numeric-kernel setting.  Used for the (rejected) column-split
# variant: AIRG_SPLIT=0/1 and AIRG_NWS=<warps per class> selected it; kept
# as the template for A/B runs of the numeric kernels.
for cfg in "AIRG_NT=128,128,256,256,256" "$@"; do
  echo "$cfg $(env $cfg timeout 200 python tools/serial_breakdown.py 2>&1 | tail -1)"
done
