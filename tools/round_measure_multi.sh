#!/bin/bash
# Multi-GPU measurement pass (run under gpurun --gpus 4 from the repo root):
# weak scaling at 4096^2 per GPU (BASELINE configs[2]) N = 1, 2, 4; configs[3]
# (truncation start 8) at N = 1 and 4 with the distributed and the replicated
# coarse solve; distributed setup phases at N = 4.  Outputs in gpurun_out/$1/.
set -u
D=gpurun_out/${1:-multi}
mkdir -p $D
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python bench.py --nx 4096 --steps 3 --warmup 3 --no-cpu > $D/n1_4096.log 2>&1; tail -1 $D/n1_4096.log | cut -c1-200
$R --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 3 --warmup 3 > $D/n2.log 2>&1; tail -1 $D/n2.log | cut -c1-200
$R --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 3 --warmup 3 > $D/n4.log 2>&1; tail -1 $D/n4.log | cut -c1-200
$R --nproc-per-node 4 --master-port 29523 bench.py --gpus 4 --nx 2048 --truncate-start 8 --steps 3 --warmup 3 > $D/c3_n4.log 2>&1
AIRG_DIST_COARSE=0 $R --nproc-per-node 4 --master-port 29524 bench.py --gpus 4 --nx 2048 --truncate-start 8 --steps 3 --warmup 3 > $D/c3_n4_repl.log 2>&1
$R --nproc-per-node 4 --master-port 29525 tools/dist_phases.py 4096 > $D/dist_phases_n4.log 2>&1
$R --nproc-per-node 2 --master-port 29526 tools/dist_phases.py 4096 > $D/dist_phases_n2.log 2>&1
ls $D
