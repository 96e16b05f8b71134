"""Batch driver (paper_2103_07329_b200.cli, the reference cli.py on the device
path): argument handling and error exit codes on CPU; a real run on the GPU."""

import os

import numpy as np
import pytest

from paper_2103_07329_b200 import cli


def test_help_methods(capsys):
    assert cli.main(["--help-methods"]) == 0
    out = capsys.readouterr().out
    assert "MultiGrid  (roles: solver, preconditioner)" in out
    assert "mg_coarse_matrix_size" in out and "Direct" in out


def test_config_required_and_bad_inputs(tmp_path, capsys):
    assert cli.main([]) == 2
    assert cli.main(["--config", str(tmp_path / "missing.yaml")]) == 2
    bad = tmp_path / "bad.yaml"
    bad.write_text("solver: {method: CG}\nsystem: {poisson: [4, 4]}\n")
    assert cli.main(["--config", str(bad)]) == 2
    good = tmp_path / "good.yaml"
    good.write_text("solver: {method: CG}\nsystem: {poisson: [4, 4, 4]}\n")
    assert cli.main(["--config", str(good), "--bench-gain", "x,y"]) == 2


def test_bench_gain_validation():
    from paper_2103_07329_b200.errors import ConfigurationError
    with pytest.raises(ConfigurationError):
        cli.bench_gain(None, None, None, [2, 4])          # m list without 1
    with pytest.raises(ConfigurationError):
        cli.bench_gain(None, None, None, [1, 3])          # unsupported m


def test_csv_schema_matches_reference():
    assert cli.CSV_COLUMNS == ("method", "m", "nnumas", "ncores", "iters",
                               "max_rel_residual", "t_solve_s", "t_setup_s", "P_m")
    sw = cli.GainSweep()
    sw.add(cli.Sample("CG", 1, 10, 1e-9, 2.0, 0.5, True))
    sw.add(cli.Sample("CG", 4, 10, 1e-9, 4.0, 0.5, True))
    sw.finish()
    assert sw.samples[1].gain == pytest.approx(2.0)
    lines = sw.csv_text().splitlines()
    assert lines[0].split(",") == list(cli.CSV_COLUMNS)
    assert lines[2].split(",")[-1] == "2.0000" and len(lines) == 3
    assert sw.converged and "P_m" in sw.table()


@pytest.mark.gpu
def test_cli_run_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = tmp_path / "run.yaml"
    cfg.write_text(
        "solver: {method: CG, rel_tolerance: 1e-8}\n"
        "preconditioner: {method: MultiGrid}\n"
        "pre_smoother: {method: Jacobi, weight: 0.8}\n"
        "post_smoother: {method: Jacobi, weight: 0.8}\n"
        "system: {poisson: [12, 12, 12]}\n"
        "benchmark: {m: [1, 4], repetitions: 2}\n")
    out = tmp_path / "r.csv"
    assert cli.main(["--config", str(cfg), "--csv", str(out)]) == 0
    rows = out.read_text().strip().splitlines()
    assert rows[0].split(",") == list(cli.CSV_COLUMNS)
    assert len(rows) == 3 and rows[2].split(",")[1] == "4"


def test_report_stats_format():
    from paper_2103_07329_b200.solvers import SolveStats
    st = SolveStats(3, np.array([True, False]), np.array([1e-9, 2e-3]),
                    [np.array([1.0, 1.0]), np.array([1e-3, 1e-2]), np.array([1e-9, 2e-3])], "CG")
    out = cli.report_stats(st)
    assert "iterations: 3" in out and "converged: NO (1/2 columns)" in out
    assert "max relative residual: 2.000000e-03" in out
