"""``airg-bench``: the reference's benchmark harness (airmg-bench, cli.py)
on the B200 path — same flags, same JSON record (schema v1), same exit codes
(0 converged, 1 configuration / usage / I/O error, 2 non-convergence or
divergence), same CSV/JSON reports.

    python -m paper_2508_17517_b200.cli --n 2048 --output run.json

The setup/solve options are generated from the config dataclasses, so the
flag maps cover ``SetupConfig`` / ``SolveConfig`` exactly (ref: cli.py:28-60;
the only rename is ``lump`` <-> ``--a-lump``).  Timings bracket device work
with a synchronize (the reference times host-synchronous scipy calls).
"""

import argparse
import csv
import dataclasses
import json
import os
import sys
import time

import numpy as np

from .advection import AdvectionProblem, build_advection_1d, build_advection_2d
from .amg_setup import SetupConfig, hierarchy_summary, setup
from .amg_solve import DivergenceError, SolveConfig, richardson_solve
from .csr import diagonal, write_matrix_market

__all__ = ['main', 'run', 'emit_report', 'SETUP_FLAG_MAP', 'SOLVE_FLAG_MAP']

SCHEMA_VERSION = 1
_RENAMED = {'lump': '--a-lump'}
_CHOICES = {'inverse_type': ('arnoldi', 'neumann'),
            'coarsest_inverse_type': ('newton', 'arnoldi', 'neumann')}


def _flag_map(cls):
    return {_RENAMED.get(f.name, '--' + f.name.replace('_', '-')): f.name
            for f in dataclasses.fields(cls)}


SETUP_FLAG_MAP = _flag_map(SetupConfig)
SOLVE_FLAG_MAP = _flag_map(SolveConfig)


def _add_config_flags(group, cls, flag_map):
    types = {f.name: f.type for f in dataclasses.fields(cls)}
    for flag, name in flag_map.items():
        t = types[name]
        t = t if isinstance(t, type) else {'float': float, 'int': int, 'str': str,
                                           'bool': bool}[str(t)]
        dest = flag[2:].replace('-', '_')
        if t is bool:
            group.add_argument(flag, dest=dest, action=argparse.BooleanOptionalAction, default=None)
        else:
            group.add_argument(flag, dest=dest, type=t, default=None, choices=_CHOICES.get(name))


def _build_parser():
    p = argparse.ArgumentParser(prog='airg-bench',
                                description='AIRG reduction multigrid on upwind advection (B200).')
    g = p.add_argument_group('problem')
    g.add_argument('--dim', type=int, choices=(1, 2), default=2)
    g.add_argument('--n', type=int, default=64, help='cells per dimension (square grid)')
    for name in ('nx', 'ny'):
        g.add_argument('--' + name, type=int, default=None)
    for name in ('vx', 'vy'):
        g.add_argument('--' + name, type=float, default=None)
    g.add_argument('--angle', type=float, default=None,
                   help='velocity angle in radians (precedence over --vx/--vy)')
    g.add_argument('--lx', type=float, default=1.0)
    g.add_argument('--ly', type=float, default=1.0)
    su = p.add_argument_group('setup (maps 1:1 onto SetupConfig)')
    _add_config_flags(su, SetupConfig, SETUP_FLAG_MAP)
    su.add_argument('--no-auto-truncate', action='store_true',
                    help='disable hierarchy truncation (auto_truncate_tol=None)')
    so = p.add_argument_group('solve (maps 1:1 onto SolveConfig)')
    _add_config_flags(so, SolveConfig, SOLVE_FLAG_MAP)
    o = p.add_argument_group('execution and output')
    o.add_argument('--second-solve', action=argparse.BooleanOptionalAction, default=True,
                   help='time a second (warm) solve')
    o.add_argument('--repeats', type=int, default=1, help='timed solve repetitions')
    o.add_argument('--compare-inverse-types', action='store_true',
                   help='paired run: arnoldi (AIRG) vs neumann (nAIR)')
    for name in ('output', 'residual-csv', 'report-csv', 'report-json', 'export-matrix',
                 'dump-operators', 'cf-diagnostics'):
        o.add_argument('--' + name, default=None)
    return p


def _config(args, cls, flag_map):
    kw = {}
    for flag, name in flag_map.items():
        v = getattr(args, flag[2:].replace('-', '_'))
        if v is not None:
            kw[name] = v
    return cls(**kw)


def _problem(args):
    if args.angle is not None:
        vx, vy = float(np.cos(args.angle)), float(np.sin(args.angle))
    elif args.vx is not None or args.vy is not None:
        vx, vy = args.vx or 0.0, args.vy or 0.0
    else:
        vx, vy = float(np.cos(np.pi / 4)), float(np.sin(np.pi / 4))
    nx = args.n if args.nx is None else args.nx
    if args.dim == 1:
        return AdvectionProblem(nx=nx, ny=0, vx=vx, vy=0.0, Lx=args.lx)
    ny = args.n if args.ny is None else args.ny
    return AdvectionProblem(nx=nx, ny=ny, vx=vx, vy=vy, Lx=args.lx, Ly=args.ly)


def _system(problem):
    if problem.ny == 0:
        A = build_advection_1d(problem.nx, problem.vx)
        return A, np.zeros(A.nrows)
    return build_advection_2d(problem)


def _timed(fn):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def _one_run(problem, scfg, vcfg, second_solve, repeats):
    A, b = _system(problem)
    x0 = np.ones(A.nrows)
    H, t_setup = _timed(lambda: setup(A, scfg))
    (x, stats), t_first = _timed(lambda: richardson_solve(H, b, x0, vcfg))
    reps = []
    for _ in range(max(repeats, 1) if second_solve else max(repeats - 1, 0)):
        (x, stats), t = _timed(lambda: richardson_solve(H, b, x0, vcfg))
        reps.append(t)
    rec = {
        'schema_version': SCHEMA_VERSION,
        'problem': {'dim': 1 if problem.ny == 0 else 2, 'nx': problem.nx, 'ny': problem.ny,
                    'n': A.nrows, 'vx': problem.vx, 'vy': problem.vy, 'Lx': problem.Lx,
                    'Ly': problem.Ly},
        'setup_config': scfg.to_dict(),
        'solve_config': dataclasses.asdict(vcfg),
        'summary': hierarchy_summary(H),
        'solve': stats.to_dict(),
        'timings': {'setup_seconds': t_setup, 'first_solve_seconds': t_first,
                    'solve_seconds': reps[-1] if reps else t_first, 'repeat_seconds': reps,
                    'setup_breakdown': dict(H.setup_breakdown)},
    }
    return H, stats, rec


def _dump_operators(H, d):
    os.makedirs(d, exist_ok=True)
    write_matrix_market(H.top_A, os.path.join(d, 'top_A.mtx'))
    write_matrix_market(H.coarsest_A, os.path.join(d, 'coarsest_A.mtx'))
    for i, L in enumerate(H.levels):
        for name in ('R', 'P', 'A_ff', 'A_fc'):
            write_matrix_market(getattr(L, name), os.path.join(d, f'level{i}_{name}.mtx'))


def _cf_diagnostics(H, d):
    """Per-level CF labels and 50-bin histograms of the A_ff dominance ratios
    sum_{j != i} |a_ij| / |a_ii| (ref: cli.py:193-217)."""
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, 'cf_labels.csv'), 'w', newline='') as fh:
        w = csv.writer(fh)
        w.writerow(['level', 'node', 'label'])
        for i, L in enumerate(H.levels):
            for node, lab in enumerate(L.split.labels_host()):
                w.writerow([i, node, 'F' if lab == 0 else 'C'])
    with open(os.path.join(d, 'ddc_ratio_histograms.csv'), 'w', newline='') as fh:
        w = csv.writer(fh)
        w.writerow(['level', 'bin_lo', 'bin_hi', 'count'])
        for i, L in enumerate(H.levels):
            p, c, v = L.A_ff.to_host()
            rows = np.repeat(np.arange(L.A_ff.nrows), np.diff(p))
            off = np.abs(np.where(c != rows, v, 0.0))
            ratios = np.bincount(rows, weights=off, minlength=L.A_ff.nrows) / np.abs(
                np.asarray(diagonal(L.A_ff).cpu().numpy()))
            counts, edges = np.histogram(ratios, bins=50)
            for k in range(50):
                w.writerow([i, f'{edges[k]:.6g}', f'{edges[k + 1]:.6g}', int(counts[k])])


def run(args):
    """Run the configured benchmark -> (exit code, record); solver
    non-convergence / divergence is exit code 2, not an exception."""
    problem = _problem(args)
    scfg = _config(args, SetupConfig, SETUP_FLAG_MAP)
    if args.no_auto_truncate:
        scfg = dataclasses.replace(scfg, auto_truncate_tol=None)
    scfg.validate()
    vcfg = _config(args, SolveConfig, SOLVE_FLAG_MAP).validate()
    if args.export_matrix:
        write_matrix_market(_system(problem)[0], args.export_matrix)
    if args.compare_inverse_types:
        rec, code = {'schema_version': SCHEMA_VERSION, 'mode': 'compare_inverse_types'}, 0
        for label, kind in (('airg', 'arnoldi'), ('nair', 'neumann')):
            try:
                _, stats, r = _one_run(problem, dataclasses.replace(scfg, inverse_type=kind),
                                       vcfg, args.second_solve, args.repeats)
            except DivergenceError as e:
                rec[label] = {'diverged': True, 'error': str(e), 'iteration': e.iteration}
                code = 2
                continue
            rec[label] = r
            code = code if stats.converged else 2
        return code, rec
    try:
        H, stats, rec = _one_run(problem, scfg, vcfg, args.second_solve, args.repeats)
    except DivergenceError as e:
        return 2, {'schema_version': SCHEMA_VERSION, 'diverged': True, 'error': str(e),
                   'iteration': e.iteration}
    if args.dump_operators:
        _dump_operators(H, args.dump_operators)
    if args.cf_diagnostics:
        _cf_diagnostics(H, args.cf_diagnostics)
    if args.residual_csv:
        with open(args.residual_csv, 'w', newline='') as fh:
            w = csv.writer(fh)
            w.writerow(['iteration', 'residual_norm'])
            w.writerows([i, f'{r:.17g}'] for i, r in enumerate(stats.residual_history))
    return (0 if stats.converged else 2), rec


REPORT_COLUMNS = [
    'n', 'dim', 'nx', 'ny', 'vx', 'vy', 'strong_threshold', 'poly_order', 'inverse_type',
    'iterations', 'converged', 'num_levels', 'truncated_at', 'cycle_complexity',
    'storage_complexity', 'grid_complexity', 'setup_seconds', 'solve_seconds',
    'setup_cf_split', 'setup_prolongator', 'setup_polynomial', 'setup_spgemm_R',
    'setup_spgemm_coarse', 'setup_extract', 'setup_drop', 'setup_truncation',
]


def _row(rec):
    pr, sc, su, so, tm = (rec['problem'], rec['setup_config'], rec['summary'], rec['solve'],
                          rec['timings'])
    row = {k: pr[k] for k in ('n', 'dim', 'nx', 'ny', 'vx', 'vy')}
    row.update({k: sc[k] for k in ('strong_threshold', 'poly_order', 'inverse_type')})
    row.update(iterations=so['iterations'], converged=so['converged'])
    row.update({k: su[k] for k in ('num_levels', 'truncated_at', 'cycle_complexity',
                                   'storage_complexity', 'grid_complexity')})
    row.update(setup_seconds=tm['setup_seconds'], solve_seconds=tm['solve_seconds'])
    row.update({'setup_' + k: v for k, v in tm['setup_breakdown'].items()})
    return row


def emit_report(results, csv_path=None, json_path=None):
    """Run records -> report rows sorted by problem size, written as CSV
    and/or JSON (ref: cli.py:323-376).  Returns the rows."""
    if not results:
        raise ValueError('need at least one result record')
    rows = sorted((_row(r) for r in results), key=lambda r: r['n'])
    if csv_path:
        with open(csv_path, 'w', newline='') as fh:
            w = csv.DictWriter(fh, fieldnames=REPORT_COLUMNS)
            w.writeheader()
            w.writerows(rows)
    if json_path:
        with open(json_path, 'w') as fh:
            json.dump(rows, fh, indent=2, sort_keys=True)
            fh.write('\n')
    return rows


def main(argv=None):
    try:
        args = _build_parser().parse_args(argv)
    except SystemExit as e:
        return 0 if e.code in (0, None) else 1
    try:
        code, rec = run(args)
    except (ValueError, OSError) as e:
        print(f'error: {e}', file=sys.stderr)
        return 1
    try:
        text = json.dumps(rec, indent=2, sort_keys=True)
        if args.output:
            with open(args.output, 'w') as fh:
                fh.write(text + '\n')
        else:
            print(text)
        if args.report_csv or args.report_json:
            if rec.get('mode') == 'compare_inverse_types':
                src = [rec[k] for k in ('airg', 'nair')
                       if isinstance(rec.get(k), dict) and 'summary' in rec[k]]
            else:
                src = [rec] if 'summary' in rec else []
            if src:
                emit_report(src, csv_path=args.report_csv, json_path=args.report_json)
    except OSError as e:
        print(f'error: {e}', file=sys.stderr)
        return 1
    return code


if __name__ == '__main__':
    sys.exit(main())
