#!/bin/bash
# One-GPU measurement pass of a round (run under gpurun from the repo root):
# tests, the driver-contract bench lines, per-level V-cycle / kernel shares,
# and the ncu captures behind profiles/.  Outputs in gpurun_out/$1/.
set -u
D=gpurun_out/${1:-meas}
mkdir -p $D
python -m pytest tests -m gpu -q > $D/gputests.log 2>&1; tail -2 $D/gputests.log
python bench.py > $D/bench.log 2>&1; tail -1 $D/bench.log | cut -c1-400
python bench.py --problem dg --steps 3 --warmup 3 --no-cpu > $D/bench_dg.log 2>&1
python bench.py --truncate-start 8 --steps 3 --warmup 3 --no-cpu > $D/bench_c3.log 2>&1
VLEVELS_OUT=$D/vlevels.json python tools/vlevels.py 2048 9 > $D/vlevels.log 2>&1
python tools/kprof.py 2048 > $D/kprof.log 2>&1
python tools/setup_levels.py 2048 > $D/setup_levels.log 2>&1
# ncu: launch list of the bench, DRAM traffic of one V-cycle, full sets of two new kernels
ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file $D/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu > $D/ncu_launch.log 2>&1
ncu --nvtx --nvtx-include "vcycle/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file $D/vc_launch.csv python tools/vcycle_once.py 2048 > $D/vc_once.log 2>&1
ncu --nvtx --nvtx-include "vcycle/" -k regex:chain_kernel --launch-count 2 --set full --import-source on \
    --clock-control none -o $D/chain python tools/vcycle_once.py 2048 > $D/ncu_chain.log 2>&1
ncu -k regex:spgemm_reg_kernel --launch-count 4 --set full --import-source on --clock-control none \
    -o $D/reg python tools/rap_kernels.py 0 > $D/ncu_reg.log 2>&1
ls $D
