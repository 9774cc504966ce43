"""The reference algorithm (oracle port, pinned bitwise to airmg) at full size
on ONE host core: setup, then two solves, the second timed (cli.py:220-259).
usage: cpu_ref_full.py [nx] -> one JSON line"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from threadpoolctl import threadpool_limits

threadpool_limits(1)
import bench  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
t0 = time.time()
setup_s, solve_s, its = bench.cpu_run(nx, 6)
print(json.dumps({'nx': nx, 'dofs': nx * nx, 'setup_s': setup_s, 'solve_s': solve_s, 'iterations': its,
                  'dof_per_s': nx * nx / (setup_s + solve_s), 'cores': 1, 'host_cpus': os.cpu_count(),
                  'wall_s': time.time() - t0, 'kind': 'port (oracle/airg_oracle.py)'}), flush=True)
