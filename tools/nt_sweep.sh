#!/bin/bash
# Galerkin time of levels 5/7/9 (tools/rap_micro.py) per thread-count table AIRG_NT
for cfg in "128,128,256,256,256" "128,128,128,256,256" "128,128,128,128,256" "128,64,128,128,128" "64,128,128,128,128" "128,128,128,128,128"; do
  echo "NT=$cfg $(for l in 5 7 9; do AIRG_NT=$cfg timeout 200 python tools/rap_micro.py $l 2>&1 | tail -1 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["galerkin_ms"])'; done | tr '\n' ' ')"
done
