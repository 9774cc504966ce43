#!/bin/bash
# per-kernel device time of one 2048^2 setup+solve under several env settings
for e in "$@"; do
  echo "== $e"
  env $e timeout 300 python tools/kprof.py 2048 6 2>&1 | grep -E "total_ms|spgemm" | head -6
done
