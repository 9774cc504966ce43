"""AIRG setup + solve benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = the hot path over one synthetic problem: ``setup(A, SetupConfig())``
followed by ``richardson_solve`` to rtol 1e-10 (b = 0, x0 = 1), exactly the
reference's benchmark run (cli.py:220-259).  Workload = BASELINE.json
configs[1]: 2D upwind advection, 2048 x 2048 (4.19M DOFs), theta = pi/4,
default AIRG config (order-6 GMRES polynomial smoothers, order-100 Newton
coarse solver, automatic truncation).

value = DOFs / (setup s + solve s).  At N>1 the job is ONE global problem of
4096 x (4096 N) grid points split into N row strips of 4096^2 -- BASELINE.json
configs[2], ~16.8M DOFs per GPU (weak scaling; --nx sets the strip size):
distributed setup + native distributed Richardson with NCCL halo exchanges
(paper_2508_17517_b200/dist.py), step time = max over ranks.  Inputs are
resident in HBM before the timed region; every level operator of the
hierarchy (> 1 GB per GPU) exceeds L2.
"""

import argparse
import glob
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ('AIRG setup+solve throughput, rtol 1e-10 (DOFs / (setup s + solve s)); '
          'solve V-cycle HBM GB/s in roofline')
PI4 = (float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4)))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument('--gpus', type=int, default=1)
    ap.add_argument('--steps', type=int, default=5)
    ap.add_argument('--warmup', type=int, default=3)
    ap.add_argument('--impl', default='ours', choices=['ours', 'reference'])
    ap.add_argument('--nx', type=int, default=None,
                    help='grid points per side per GPU (default: 2048 at N=1, configs[1]; '
                         '4096 at N>1, configs[2]: ~16.8M DOFs per GPU)')
    ap.add_argument('--order', type=int, default=6)
    ap.add_argument('--truncate-start', type=int, default=None,
                    help='SetupConfig.auto_truncate_start_level (configs[3]: a low start, e.g. 4, '
                         'gives a large coarsest grid solved by the order-100 Newton polynomial)')
    ap.add_argument('--cpu-nx', type=int, default=512,
                    help='CPU sample grid (reference arm and cpu_baseline): 512^2, whose per-DOF '
                         'cost is within ~2x of the 2048^2 run; the full 2048^2 reference run '
                         'takes ~19 min (profiles/)')
    ap.add_argument('--no-cpu', action='store_true')
    ap.add_argument('--problem', default='fd', choices=['fd', 'dg'],
                    help='fd: 2-D upwind finite differences (configs[1]); dg: upwind DG Q1 on '
                         'nx x nx cells, 4 unknowns per cell (configs[4], single GPU)')
    return ap.parse_args()


def max_over_ranks(value, dist, device):
    """Max of a per-rank time over all ranks (the step time of the job)."""
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    return (int(os.environ.get('RANK', 0)), int(os.environ.get('WORLD_SIZE', 1)),
            int(os.environ.get('LOCAL_RANK', 0)))


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference (numpy/scipy, same kernels)
# ---------------------------------------------------------------------------

def cpu_run(nx, order, problem='fd'):
    """Reference-style run on the host: setup then two solves, the second
    timed (cli.py:220-259).  Returns (setup_s, solve_s, its)."""
    from oracle import airg_oracle as O
    A = O.advection_dg_q1(nx, nx, *PI4) if problem == 'dg' else O.advection_2d(nx, nx, *PI4)
    t0 = time.perf_counter()
    H = O.setup(A, O.Cfg(poly_order=order))
    t1 = time.perf_counter()
    O.richardson(H, np.zeros(A.nrows), np.ones(A.nrows))
    t2 = time.perf_counter()
    _, hist, conv, its = O.richardson(H, np.zeros(A.nrows), np.ones(A.nrows))
    t3 = time.perf_counter()
    return t1 - t0, t3 - t2, its


def cpu_cores_note():
    try:
        from threadpoolctl import threadpool_info
        blas = [f"{i.get('internal_api')}:{i.get('num_threads')}" for i in threadpool_info()]
    except Exception:
        blas = []
    return os.cpu_count(), blas


def _ref_worker(job):
    """One reference instance: a small warm-up run (module import, caches;
    when W > 0) and `steps` timed setup/solve runs on the sample (one BLAS
    thread; scipy's sparse kernels are single-threaded)."""
    nx, order, problem, warmup, steps = job
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    if warmup:
        cpu_run(min(nx, 64), order, problem)
    setup_s, solve_s, its = [], [], 0
    for _ in range(steps):
        a, b, its = cpu_run(nx, order, problem)
        setup_s.append(a)
        solve_s.append(b)
    return float(np.mean(setup_s)), float(np.mean(solve_s)), its


def reference_arm(args, rank, world):
    """The reference algorithm (oracle port, pinned bitwise to airmg) on ALL
    host cores: the path is single-threaded Python/scipy, so the host's
    throughput is one independent instance per core (AIRG_REF_PROCS to
    override); value = aggregate DOF/s."""
    if rank != 0:
        return 0
    problem = getattr(args, 'problem', 'fd')
    procs = int(os.environ.get('AIRG_REF_PROCS', os.cpu_count() or 1))
    # the K timed steps are spread over the concurrent instances (at least one
    # each), so the run takes about one sample's time, not K of them
    per = max(1, -(-args.steps // procs))
    job = (args.cpu_nx, args.order, problem, args.warmup, per)
    if procs > 1:
        import multiprocessing as mp
        with mp.get_context('fork').Pool(procs) as pool:
            res = pool.map(_ref_worker, [job] * procs)
    else:
        res = [_ref_worker(job)]
    n = args.cpu_nx * args.cpu_nx * (4 if problem == 'dg' else 1)
    step_s = [a + b for a, b, _ in res]
    v = float(sum(n / t for t in step_s))           # aggregate over the instances
    t = float(np.mean(step_s))
    its = res[0][2]
    ncpu, blas = cpu_cores_note()
    line = {
        'impl': 'reference', 'metric': METRIC, 'value': v, 'unit': 'DOF/s',
        # whole-host time per step: the instances run concurrently, so one
        # sample-step of the host takes n / value (each instance's own sample
        # time is instance_ms_per_sample)
        'n_gpus': world, 'steps': args.steps, 'warmup': args.warmup, 'ms_per_step': n / v * 1e3,
        'instance_ms_per_sample': t * 1e3, 'samples_timed': procs * per,
        'higher_is_better': True, 'scaling': 'weak', 'vs_baseline': None, 'dtype': 'f64',
        'data': 'synthetic (2D upwind advection stencil, b=0, x0=1)',
        'config': {'workload': (f'AIRG pi/4 upwind DG Q1 advection {args.nx}x{args.nx} cells'
                                if problem == 'dg' else
                                f'AIRG pi/4 advection {args.nx}x{args.nx}') + f' order {args.order}',
                   'sample': f'{args.cpu_nx}x{args.cpu_nx}', 'rtol': 1e-10},
        'setup_s': float(np.mean([a for a, _, _ in res])),
        'solve_s': float(np.mean([b for _, b, _ in res])), 'iterations': its,
        'cpu_baseline': {'value': v, 'unit': 'DOF/s', 'cores': procs, 'kind': 'port',
                         'sample': f'{procs} concurrent instances (one per host core), {per} timed '
                                   f'setup + solve each at {args.cpu_nx}^2 of the {args.nx}^2 workload '
                                   f'(oracle/airg_oracle.py = numpy/scipy restatement of airmg, '
                                   f'pinned bitwise to it; scipy sparse kernels single-threaded, '
                                   f'1 BLAS thread per instance; host has {ncpu} cpus); value = '
                                   f'aggregate DOF/s'},
        'e2e': {'value': v, 'unit': 'DOF/s', 'h2d_bytes_per_step': 0, 'd2h_bytes_per_step': 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------

class NvmlSampler:
    """SM clock + throttle reasons sampled in-process (NVML) every `period` s
    during the timed region.  nvidia-smi polling at 100 ms slowed the
    synchronisation-heavy setup by ~30%; a few NVML reads do not."""

    NAMES = {'hw_slowdown': 0x8, 'hw_thermal_slowdown': 0x40, 'sw_thermal_slowdown': 0x20,
             'sw_power_cap': 0x4}

    def __init__(self, index, period=0.5):
        self.index = index
        self.period = period
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()
        self.ok = False

    def __enter__(self):
        if os.environ.get('AIRG_BENCH_NO_CLOCKS'):
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.ok = True
        except Exception:
            return self
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def _sample(self):
        nv = self.nv
        self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        self.mx.append(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for k, bit in self.NAMES.items():
            if r & bit:
                self.reasons.add(k)

    def _run(self):
        while True:
            try:
                self._sample()
            except Exception:
                pass
            if self.stop.wait(self.period):
                return

    def __exit__(self, *exc):
        if self.ok:
            self.stop.set()
            self.th.join(timeout=5)

    def summary(self):
        return {'sm_mhz': float(np.median(self.sm)) if self.sm else None,
                'sm_max_mhz': max(self.mx) if self.mx else None,
                'reasons': sorted(self.reasons), 'samples': len(self.sm), 'source': 'nvml'}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get('AIRG_BENCH_NO_CLOCKS'):
            return self
        q = ('clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,'
             'clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,'
             'clocks_event_reasons.sw_power_cap')
        try:
            self.proc = subprocess.Popen(['nvidia-smi', '-i', str(self.index), f'--query-gpu={q}',
                                          '--format=csv,noheader,nounits', '-lms', '1000'],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(',')])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                pass

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace('.', '').isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace('.', '').isdigit()]
        names = ['hw_slowdown', 'hw_thermal_slowdown', 'sw_thermal_slowdown', 'sw_power_cap']
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[3:7]):
                if v.strip().lower() == 'active':
                    reasons.add(nm)
        return {'sm_mhz': float(np.median(sm)) if sm else None,
                'sm_max_mhz': max(mx) if mx else None, 'reasons': sorted(reasons),
                'samples': len(sm)}


def count_launches(step):
    """Kernel launches of one step (CUPTI via torch.profiler), untimed."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    n = 0
    mine = 0
    for e in prof.events():
        if e.device_type.name == 'CUDA' and not e.name.startswith('Memcpy') \
                and not e.name.startswith('Memset'):
            n += 1
            if 'airg' in e.name:
                mine += 1
    return n, mine


def hbm_peak():
    try:
        peaks = json.load(open(os.path.join(ROOT, 'MEASURED_PEAKS.json')))
        return float(peaks['hbm_gbs']), 'MEASURED_PEAKS.json hbm_gbs'
    except Exception:
        return 6650.0, 'fallback (B200_PROFILING.md)'


class SerialWorkload:
    """N=1: the whole 2048^2 problem on one GPU (BASELINE.json configs[1])."""

    def __init__(self, args):
        import torch
        import paper_2508_17517_b200 as G
        self.G, self.args = G, args
        nx = args.nx
        self.cfg = G.SetupConfig(poly_order=args.order, auto_truncate_start_level=args.truncate_start)
        self.scfg = G.SolveConfig()
        prob = G.AdvectionProblem(nx=nx, ny=nx, vx=PI4[0], vy=PI4[1])
        if args.problem == 'dg':
            self.A, self.b = G.build_advection_dg(prob)
            self.workload = (f'AIRG pi/4 upwind DG Q1 advection, {nx}x{nx} cells x 4 unknowns, '
                             f'order {args.order}, default SetupConfig (BASELINE.json configs[4])')
        else:
            self.A, self.b = G.build_advection_2d(prob)
            self.workload = (f'AIRG pi/4 advection {nx}x{nx}, order {args.order}, default '
                             'SetupConfig (BASELINE.json configs[1])')
            if args.truncate_start is not None:
                self.workload = (f'AIRG pi/4 advection {nx}x{nx}, order {args.order}, truncation '
                                 f'start level {args.truncate_start}: order-100 Newton coarse '
                                 'solver on a large coarsest grid (BASELINE.json configs[3])')
        self.n = self.n_total = self.A.nrows
        self.x0 = torch.ones(self.n, dtype=torch.float64, device='cuda')
        self.parallelism = 'single GPU'

    def setup(self):
        return self.G.setup(self.A, self.cfg)

    def solve(self, H):
        return self.G.richardson_solve(H, self.b, self.x0, self.scfg)

    def iteration_ms(self, H):
        """Per-Richardson-iteration time with the solve plan cached (V-cycle +
        residual + norm), the same measurement DistWorkload.roofline makes at
        N > 1, so the solve's weak scaling compares like with like."""
        import torch
        _, st = self.solve(H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        reps = 5
        for _ in range(reps):
            _, st = self.solve(H)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps / max(st.iterations, 1)

    def roofline(self, H):
        """One V-cycle (the solve's kernel chain) timed with CUDA events."""
        import torch
        from paper_2508_17517_b200 import _lib as L
        from paper_2508_17517_b200.amg_solve import count_cycle_bytes, plan_for
        with plan_for(H) as plan:
            # the plan's own staging vectors: the timed call is the V-cycle
            # kernel chain alone (no copy in / out of caller buffers)
            vin, vout = L.C.c_void_p(), L.C.c_void_p()
            L.call('airg_plan_staging', plan.h, L.C.byref(vin), L.C.byref(vout))
            r = torch.randn(self.n, dtype=torch.float64, device='cuda')
            L.call('airg_copy_d2d', vin, L.ptr(r), 8 * self.n, L.stream_handle())
            for _ in range(3):
                L.call('airg_plan_vcycle', plan.h, 0, vin, vout, 1, L.stream_handle())
            nv = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(nv):
                L.call('airg_plan_vcycle', plan.h, 0, vin, vout, 1, L.stream_handle())
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nv
        vbytes = count_cycle_bytes(H, include_top=False)
        self.traffic = None
        src = None
        # ncu DRAM bytes of one V-cycle of this configuration (profiles/, newest round first)
        for fn in sorted(glob.glob(os.path.join(ROOT, 'profiles', 'r*_vcycle_traffic.json')),
                         reverse=True):
            try:
                t = json.load(open(fn))
                if int(t['algorithmic_bytes']) == int(vbytes):
                    self.traffic, src = int(t['dram_total_bytes']), os.path.basename(fn)
                    break
            except Exception:
                pass
        return ms, vbytes, ('one V-cycle (R / A_fc SpMVs, q(A_ff) smoother chains, coarse solve: the path the plan runs); '
                            f'algorithmic bytes {vbytes} (count_cycle_bytes); traffic = ncu '
                            f'dram__bytes_read+write of the same V-cycle (profiles/{src or "r*_vcycle_traffic.json: none matches"})')

    def e2e(self):
        """Step through the public API from pinned host buffers."""
        import torch
        G, n, A = self.G, self.n, self.A
        Ap, Ac, Av = (t.cpu().pin_memory() for t in (A.row_offsets, A.col_indices, A.values))
        bh = torch.zeros(n, dtype=torch.float64).pin_memory()
        xh = torch.ones(n, dtype=torch.float64).pin_memory()
        xout = torch.empty(n, dtype=torch.float64).pin_memory()
        h2d = Ap.numel() * 4 + Ac.numel() * 4 + Av.numel() * 8 + 16 * n

        def step():
            Ad = G.SparseMatrix(n, n, Ap.to('cuda', non_blocking=True),
                                Ac.to('cuda', non_blocking=True), Av.to('cuda', non_blocking=True))
            H = G.setup(Ad, self.cfg)
            x, _ = G.richardson_solve(H, bh.to('cuda', non_blocking=True),
                                      xh.to('cuda', non_blocking=True), self.scfg)
            xout.copy_(x, non_blocking=True)
        return step, h2d, 8 * n

    def extra(self, H, st):
        from paper_2508_17517_b200.amg_setup import setup_compulsory_bytes
        return {'levels': H.num_levels, 'truncated_at': H.truncated_at,
                'cycle_complexity': H.cycle_complexity,
                'setup_breakdown_s': {k: round(v, 4) for k, v in H.setup_breakdown.items()},
                'setup_compulsory_bytes': setup_compulsory_bytes(H)}


class DistWorkload:
    """N>1: ONE global problem of nx x (nx*N) grid points, row strips of
    nx x nx per GPU; setup_distributed + native distributed
    Richardson with NCCL halo exchanges over NVLink."""

    def __init__(self, args, world):
        import torch
        import paper_2508_17517_b200 as G
        from paper_2508_17517_b200 import dist as D
        self.G, self.D, self.args = G, D, args
        self.comm = D.Comm()
        nx = args.nx
        self.cfg = G.SetupConfig(poly_order=args.order, auto_truncate_start_level=args.truncate_start)
        self.scfg = G.SolveConfig()
        # the inflow strip builds ~12 % less work per row (measured at N = 2
        # and 4, tools/dist_kprof.py): it gets proportionally more grid rows
        self.Ad = D.advection_2d_strips(self.comm, nx, nx * world, *PI4,
                                        weights=[float(os.environ.get('AIRG_STRIP_W0', 1.14))]
                                        + [1.0] * (world - 1))
        self.n = self.Ad.M.nrows
        self.n_total = self.Ad.rows.n
        self.b = torch.zeros(self.n, dtype=torch.float64, device='cuda')
        self.x0 = torch.ones(self.n, dtype=torch.float64, device='cuda')
        self.workload = (f'AIRG pi/4 advection {nx}x{nx * world} global grid ({world} row strips '
                         f'of {nx}x{nx}), order {args.order}, '
                         + ('default SetupConfig (BASELINE.json configs[2] weak scaling)'
                            if args.truncate_start is None else
                            f'truncation start level {args.truncate_start} (BASELINE.json configs[3])'))
        self.parallelism = (f'row-strip domain decomposition over {world} GPUs, NCCL halo '
                            'exchanges; replicated coarse tail')

    def setup(self):
        return self.D.setup_distributed(self.comm, self.Ad, self.cfg)

    def solve(self, DH):
        S = self.D.DistSolver(DH)
        x, st = S.solve(self.b, self.x0, self.scfg)
        self.S = S
        return x, st

    def roofline(self, DH):
        """Per-iteration time of the native distributed Richardson (V-cycle +
        residual, halo exchanges included), CUDA events on this rank."""
        import torch
        S = self.S
        S.solve(self.b, self.x0, self.scfg)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        reps = 5
        for _ in range(reps):
            _, st = S.solve(self.b, self.x0, self.scfg)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps / max(st.iterations, 1)
        by = self.D.dist_cycle_bytes(S, include_top=True)
        return ms, by, ('one distributed Richardson iteration per rank (V-cycle over local strips '
                        '+ replicated tail + top residual, NCCL halos inside); algorithmic bytes '
                        f'{by} per rank (dist_cycle_bytes)')

    def e2e(self):
        import torch
        G, D, M = self.G, self.D, self.Ad.M
        Ap, Ac, Av = (t.cpu().pin_memory() for t in (M.row_offsets, M.col_indices, M.values))
        n = self.n
        bh = torch.zeros(n, dtype=torch.float64).pin_memory()
        xh = torch.ones(n, dtype=torch.float64).pin_memory()
        xout = torch.empty(n, dtype=torch.float64).pin_memory()
        h2d = Ap.numel() * 4 + Ac.numel() * 4 + Av.numel() * 8 + 16 * n

        def step():
            Mh = G.SparseMatrix(n, M.ncols, Ap.to('cuda', non_blocking=True),
                                Ac.to('cuda', non_blocking=True), Av.to('cuda', non_blocking=True))
            Ad = D.DMat(Mh, self.Ad.rows, self.Ad.cols)
            DH = D.setup_distributed(self.comm, Ad, self.cfg)
            x, _ = D.DistSolver(DH).solve(bh.to('cuda', non_blocking=True),
                                          xh.to('cuda', non_blocking=True), self.scfg)
            xout.copy_(x, non_blocking=True)
        return step, h2d, 8 * n

    def extra(self, DH, st):
        brk = {}
        for k, v in DH.setup_breakdown.items():  # sub-phases ("spgemm_coarse.RAP") into their phase
            if '@' in k:
                continue
            key = k.split('.')[0]
            brk[key] = brk.get(key, 0.0) + v
        return {'levels': DH.num_levels, 'distributed_levels': len(DH.dlevels),
                'truncated_at': DH.truncated_at,
                'setup_breakdown_s': {k: round(v, 4) for k, v in brk.items()}}


def ours_arm(args, rank, world, local):
    import torch
    import paper_2508_17517_b200 as G

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group('nccl', device_id=torch.device('cuda', local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    if world > 1 and args.problem != 'fd':
        raise SystemExit('the row-strip decomposition generates the FD operator only (--problem fd)')
    W = DistWorkload(args, world) if world > 1 else SerialWorkload(args)
    n = W.n
    # grow both device pools once before warm-up (scaled to the per-GPU
    # problem): the hierarchy's operators live in the library pool (zero-copy
    # results) with the setup scratch; torch holds vectors and small tensors
    G.reserve_memory(library_bytes=n * int(os.environ.get('AIRG_RES_LIB', 5600)),
                     torch_bytes=n * int(os.environ.get('AIRG_RES_TORCH', 600)))
    info = {}

    def release():
        # drop the previous step's hierarchy / solver before building the next
        # (two live 2048^2 hierarchies overflow the pre-grown allocator pool)
        info.pop('H', None)
        info.pop('st', None)
        if hasattr(W, 'S'):
            W.S = None

    def step():
        release()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        H = W.setup()
        ev[1].record()
        x, st = W.solve(H)
        ev[2].record()
        info['H'], info['st'], info['ev'] = H, st, ev
        return H

    for _ in range(args.warmup):
        step()
    barrier()
    setup_ms, solve_ms = [], []
    sampler = ClockSampler if os.environ.get('AIRG_BENCH_CLOCKS') == 'smi' else NvmlSampler
    with sampler(local) as clk:
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        start.record()
        for _ in range(args.steps):
            step()
            ev = info['ev']
            ev[2].synchronize()
            setup_ms.append(ev[0].elapsed_time(ev[1]))
            solve_ms.append(ev[1].elapsed_time(ev[2]))
        stop.record()
        barrier()
    ms = start.elapsed_time(stop) / args.steps
    ms = max_over_ranks(ms, dist, 'cuda')
    H, st = info['H'], info['st']

    # ---- roofline of the solve's kernel chain ----
    vms, vbytes, what = W.roofline(H)
    # per-iteration solve time with the plan cached (the dist roofline already
    # is that measurement); solve_s above includes the first-solve plan build
    it_ms = W.iteration_ms(H) if hasattr(W, 'iteration_ms') else vms
    peak, peak_src = hbm_peak()
    achieved = vbytes / (vms * 1e-3) / 1e9

    # ---- e2e through the public API with pinned host buffers ----
    extra = W.extra(H, st)
    del H
    release()
    e2e_step, h2d, d2h = W.e2e()
    e2e_step()
    k_e2e = max(1, min(args.steps, 3))
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(k_e2e):
        e2e_step()
    f1.record()
    barrier()
    e2e_ms = f0.elapsed_time(f1) / k_e2e
    e2e_ms = max_over_ranks(e2e_ms, dist, 'cuda')

    launches, mine = count_launches(step)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:  # one core: the path is single-threaded Python/scipy (and 1 BLAS thread)
            from threadpoolctl import threadpool_limits
            lim = threadpool_limits(1)
        except Exception:
            lim = None
        a, bs, its = cpu_run(args.cpu_nx, args.order, args.problem)
        if lim is not None:
            lim.restore_original_limits()
        ncpu, blas = cpu_cores_note()
        cpu = {'value': args.cpu_nx ** 2 * (4 if args.problem == 'dg' else 1) / (a + bs), 'unit': 'DOF/s', 'cores': 1, 'kind': 'port',
               'sample': f'one setup + timed second solve at {args.cpu_nx}^2 (of the {args.nx}^2 '
                         f'workload) with oracle/airg_oracle.py (numpy/scipy restatement of airmg; '
                         f'scipy sparse kernels single-threaded, BLAS limited to 1 thread; '
                         f'{ncpu} host cpus); '
                         f'setup {a:.2f} s, solve {bs:.3f} s, {its} its'}

    if rank == 0:
        line = {
            'metric': METRIC, 'value': W.n_total / (ms * 1e-3), 'unit': 'DOF/s', 'n_gpus': world,
            'steps': args.steps, 'warmup': args.warmup, 'ms_per_step': ms,
            'higher_is_better': True, 'scaling': 'weak', 'vs_baseline': None, 'dtype': 'f64',
            'data': 'synthetic (2D upwind advection stencil generated on device, b=0, x0=1)',
            'config': {'workload': W.workload, 'dofs_total': W.n_total, 'dofs_per_gpu': n,
                       'rtol': 1e-10, 'parallelism': W.parallelism,
                       'l2': 'hierarchy operators (>1 GB per GPU) exceed the 126 MB L2'},
            'setup_s': float(np.mean(setup_ms)) / 1e3, 'solve_s': float(np.mean(solve_ms)) / 1e3,
            'iterations': st.iterations,
            'solve_iteration_ms': it_ms,
            'solve_cached_s': it_ms * st.iterations / 1e3,
            **extra,
            'vcycle_ms': vms,
            'setup_roofline': None if 'setup_compulsory_bytes' not in extra else {
                'bound': 'hbm', 'compulsory_bytes': extra['setup_compulsory_bytes'],
                'achieved': extra['setup_compulsory_bytes'] / (np.mean(setup_ms) * 1e-3) / 1e9,
                'peak': peak, 'unit': 'GB/s',
                'frac': extra['setup_compulsory_bytes'] / (np.mean(setup_ms) * 1e-3) / 1e9 / peak,
                'note': 'levels read once + retained operators written once; the setup is '
                        'issue/latency-bound SpGEMM (bitmap / hash) and polynomial assembly '
                        'work, not a streaming kernel'},
            'roofline': {'bound': 'hbm', 'achieved': achieved, 'peak': peak, 'unit': 'GB/s',
                         'frac': achieved / peak, 'traffic': getattr(W, 'traffic', None), 'kernel': what,
                         'peak_source': peak_src},
            'e2e': {'value': W.n_total / (e2e_ms * 1e-3), 'unit': 'DOF/s',
                    'h2d_bytes_per_step': int(h2d), 'd2h_bytes_per_step': int(d2h),
                    'ms_per_step': e2e_ms},
            'gpu_launches': int(mine * args.steps),
            'gpu_launches_all_kernels_per_step': int(launches),
            'clocks': clk.summary(),
            'cpu_baseline': cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.nx is None:  # BASELINE configs[1] on one GPU, configs[2] (weak scaling) on N
        args.nx = 2048 if world == 1 else 4096
    if args.impl == 'reference':
        return reference_arm(args, rank, world)
    return ours_arm(args, rank, world, local)


if __name__ == '__main__':
    sys.exit(main())
