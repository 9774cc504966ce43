"""The airg-bench harness (paper_2508_17517_b200/cli.py) against the reference
harness's contract (airmg cli.py, tests/test_cli.py): flag maps, exit codes,
the schema-v1 record, reports and diagnostics."""

import csv
import json
from dataclasses import fields

import pytest


@pytest.fixture(scope='module')
def cli():
    from paper_2508_17517_b200 import cli
    return cli


def _run(cli, tmp_path, *args, name='out.json'):
    out = tmp_path / name
    code = cli.main([*args, '--output', str(out)])
    return code, (json.loads(out.read_text()) if out.exists() else None)


# ---- CPU: parser and maps ---------------------------------------------------

def test_flag_maps_cover_configs_exactly(cli):
    from paper_2508_17517_b200 import SetupConfig, SolveConfig
    assert set(cli.SETUP_FLAG_MAP.values()) == {f.name for f in fields(SetupConfig)}
    assert set(cli.SOLVE_FLAG_MAP.values()) == {f.name for f in fields(SolveConfig)}
    assert cli.SETUP_FLAG_MAP['--a-lump'] == 'lump'
    known = {o for a in cli._build_parser()._actions for o in a.option_strings}
    for flag in list(cli.SETUP_FLAG_MAP) + list(cli.SOLVE_FLAG_MAP):
        assert flag in known
    # the reference's flag spellings (cli.py:30-60)
    for flag in ('--strong-threshold', '--matrix-free-polys', '--no-matrix-free-polys',
                 '--coarsest-inverse-type', '--auto-truncate-start-level', '--f-smooth-its',
                 '--one-point-classical-prolong', '--inverse-sparsity-order'):
        assert flag in known


def test_unknown_flag_and_bad_choice_exit_code(cli):
    assert cli.main(['--does-not-exist', '3']) == 1
    assert cli.main(['--inverse-type', 'jacobi']) == 1


def test_emit_report_rejects_empty(cli):
    with pytest.raises(ValueError):
        cli.emit_report([])


# ---- GPU: runs --------------------------------------------------------------

@pytest.mark.gpu
def test_cyclic_reduction_example(cli, tmp_path):
    code, res = _run(cli, tmp_path, '--dim', '1', '--n', '256', '--vx', '1',
                     '--strong-threshold', '0.5', '--poly-order', '1')
    assert code == 0 and res['solve']['converged'] and res['solve']['iterations'] <= 2


@pytest.mark.gpu
def test_2d_defaults_schema(cli, tmp_path):
    code, res = _run(cli, tmp_path, '--n', '24', '--angle', '0.7853981633974483')
    assert code == 0 and res['schema_version'] == 1
    assert res['problem']['n'] == 24 * 24
    assert 'cycle_complexity' in res['summary'] and 'storage_complexity' in res['summary']
    assert res['solve']['residual_history'][0] > 0
    for phase in ('cf_split', 'prolongator', 'polynomial', 'spgemm_R', 'spgemm_coarse',
                  'extract', 'drop', 'truncation'):
        assert phase in res['timings']['setup_breakdown']


@pytest.mark.gpu
def test_compare_inverse_types_pairing(cli, tmp_path):
    code, res = _run(cli, tmp_path, '--n', '48', '--compare-inverse-types', '--poly-order', '4',
                     '--max-iters', '200')
    assert code == 0 and res['mode'] == 'compare_inverse_types'
    assert res['airg']['setup_config']['inverse_type'] == 'arnoldi'
    assert res['nair']['setup_config']['inverse_type'] == 'neumann'
    assert res['nair']['solve']['iterations'] >= res['airg']['solve']['iterations']


@pytest.mark.gpu
def test_exit_codes(cli, tmp_path):
    assert _run(cli, tmp_path, '--strong-threshold', '1.5', '--n', '8')[0] == 1
    assert _run(cli, tmp_path, '--smooth-type', 'fcf', '--n', '8')[0] == 1
    assert cli.main(['--n', '8', '--output', str(tmp_path / 'missing' / 'o.json')]) == 1
    code, res = _run(cli, tmp_path, '--n', '48', '--max-iters', '1', '--rtol', '1e-10',
                     '--poly-order', '1')
    assert code == 2 and not res['solve']['converged']


@pytest.mark.gpu
def test_record_deterministic_except_timings(cli, tmp_path):
    _, a = _run(cli, tmp_path, '--n', '32', '--seed', '7', name='a.json')
    _, b = _run(cli, tmp_path, '--n', '32', '--seed', '7', name='b.json')
    a.pop('timings')
    b.pop('timings')
    assert json.dumps(a, sort_keys=True) == json.dumps(b, sort_keys=True)


@pytest.mark.gpu
def test_outputs_reports_and_diagnostics(cli, tmp_path):
    from paper_2508_17517_b200 import read_matrix_market
    res_csv, mtx = tmp_path / 'res.csv', tmp_path / 'a.mtx'
    assert cli.main(['--dim', '1', '--n', '16', '--strong-threshold', '0.5', '--poly-order', '1',
                     '--residual-csv', str(res_csv), '--export-matrix', str(mtx),
                     '--output', str(tmp_path / 'o.json')]) == 0
    rows = list(csv.reader(res_csv.open()))
    assert rows[0] == ['iteration', 'residual_norm'] and len(rows) >= 2
    A = read_matrix_market(mtx)
    assert A.nrows == 16 and A.nnz == 31
    ops, diag = tmp_path / 'ops', tmp_path / 'diag'
    assert cli.main(['--n', '16', '--dump-operators', str(ops), '--cf-diagnostics', str(diag),
                     '--output', str(tmp_path / 'p.json')]) == 0
    for f in ('top_A.mtx', 'coarsest_A.mtx', 'level0_R.mtx'):
        assert (ops / f).exists()
    labels = list(csv.reader((diag / 'cf_labels.csv').open()))
    assert labels[0] == ['level', 'node', 'label'] and {r[2] for r in labels[1:]} <= {'F', 'C'}
    hist = list(csv.reader((diag / 'ddc_ratio_histograms.csv').open()))
    assert hist[0] == ['level', 'bin_lo', 'bin_hi', 'count']
    # reports sorted by size
    recs = [_run(cli, tmp_path, '--n', str(n), name=f'r{n}.json')[1] for n in (48, 16, 32)]
    rows = cli.emit_report(recs, csv_path=str(tmp_path / 'rep.csv'),
                           json_path=str(tmp_path / 'rep.json'))
    assert [r['n'] for r in rows] == sorted(r['n'] for r in rows)
    assert list(csv.reader((tmp_path / 'rep.csv').open()))[0][0] == 'n'


@pytest.mark.gpu
def test_repeats_and_second_solve(cli, tmp_path):
    code, res = _run(cli, tmp_path, '--n', '16', '--repeats', '3')
    assert code == 0 and len(res['timings']['repeat_seconds']) == 3
    assert res['timings']['solve_seconds'] == res['timings']['repeat_seconds'][-1]
    code, res = _run(cli, tmp_path, '--n', '16', '--no-second-solve', name='cold.json')
    assert res['timings']['repeat_seconds'] == []
    assert res['timings']['solve_seconds'] == res['timings']['first_solve_seconds']
