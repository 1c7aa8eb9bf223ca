"""CLI parity with the reference's ``mgsr`` command line (cli.py:1-397): flags, exit codes, CSV
layouts.  CPU tests cover the usage / configuration errors (exit 2); GPU tests run the solves."""

from __future__ import annotations

import csv
import json

import numpy as np
import pytest


def _main(argv):
    from paper_2403_07936_b200 import cli
    return cli.main(argv)


def test_cli_usage_errors_exit_2(tmp_path, capsys, monkeypatch):
    from paper_2403_07936_b200.grid import Grid, write_grid
    monkeypatch.delenv("MGSR_SEED", raising=False)
    f = tmp_path / "f.mgg"
    write_grid(Grid(np.zeros((16, 16))), f)
    assert _main(["solve", "--rhs", str(tmp_path / "missing.mgg")]) == 2
    assert "RHS file not found" in capsys.readouterr().err
    assert _main(["solve", "--rhs", str(f), "--config", str(tmp_path / "none.json")]) == 2
    assert "config file not found" in capsys.readouterr().err
    (tmp_path / "bad.json").write_text('{"N_iterz": 3}')
    assert _main(["solve", "--rhs", str(f), "--config", str(tmp_path / "bad.json")]) == 2
    assert "bad config" in capsys.readouterr().err
    assert _main(["solve", "--rhs", str(f), "--mode", "sr"]) == 2
    assert "requires --weights" in capsys.readouterr().err
    assert _main(["sweep", "--param", "bogus", "--values", "1", "--out", str(tmp_path / "o.csv")]) == 2
    assert "--param must be one of" in capsys.readouterr().err
    assert _main(["sweep", "--param", "N_smooth", "--values", "1", "--out", str(tmp_path / "o.csv")]) == 2
    assert "--rhs is required" in capsys.readouterr().err
    assert _main(["datagen", "--kind", "windows", "--n", "64", "--out", str(tmp_path / "w")]) == 2
    monkeypatch.setenv("MGSR_SEED", "x")
    assert _main(["solve", "--rhs", str(f)]) == 2
    assert "MGSR_SEED must be an integer" in capsys.readouterr().err


def test_cli_parser_mirrors_reference_flags():
    from paper_2403_07936_b200 import cli
    ap = cli.build_parser()
    sub = next(a for a in ap._actions if a.dest == "command")
    assert set(sub.choices) == {"solve", "sweep", "spectrum", "bench", "datagen"}
    solve_flags = {o for a in sub.choices["solve"]._actions for o in a.option_strings}
    for flag in ("--rhs", "--config", "--weights", "--mode", "--n-iter", "--n-smooth", "--n-gan", "--s-thres",
                 "--tol", "--seed", "--out-grid", "--out-log"):
        assert flag in solve_flags
    assert cli.SWEEP_COLUMNS == ("param", "value", "replicate", "rhs_id", "iters_to_converge", "converged",
                                 "final_diff")


@pytest.mark.gpu
def test_cli_solve_matches_oracle_and_exit_codes(cuda, orc, tmp_path, capsys):
    from paper_2403_07936_b200.grid import Grid, write_grid
    f = orc.sine_modes_rhs(64, 0)
    write_grid(Grid(f), tmp_path / "f.mgg")
    cfg = {"N_step": 1, "r_min": 8, "N_smooth": 2}
    (tmp_path / "c.json").write_text(json.dumps(cfg))
    rc = _main(["solve", "--rhs", str(tmp_path / "f.mgg"), "--config", str(tmp_path / "c.json"),
                "--out-log", str(tmp_path / "log.csv"), "--out-grid", str(tmp_path / "p.mgg")])
    assert rc == 0
    _, log = orc.solve(f, orc.Config(N_step=1, r_min=8, N_smooth=2))
    out = capsys.readouterr().out
    assert f"iterations={log.iterations}" in out and "converged=True" in out
    rows = list(csv.reader(open(tmp_path / "log.csv")))
    assert rows[0][:3] == ["iter", "diff_norm", "residual_norm"] and len(rows) == log.iterations + 1
    rc = _main(["solve", "--rhs", str(tmp_path / "f.mgg"), "--config", str(tmp_path / "c.json"), "--n-iter", "2"])
    assert rc == 3


@pytest.mark.gpu
def test_cli_sweep_batches_and_sorts(cuda, orc, tmp_path):
    from paper_2403_07936_b200.grid import Grid, write_grid
    for s in range(2):
        write_grid(Grid(orc.sine_modes_rhs(64, s)), tmp_path / f"r{s}.mgg")
    (tmp_path / "c.json").write_text(json.dumps({"N_step": 1, "r_min": 8}))
    rc = _main(["sweep", "--param", "N_smooth", "--values", "2,1", "--replicates", "2", "--config",
                str(tmp_path / "c.json"), "--rhs", f"{tmp_path / 'r1.mgg'},{tmp_path / 'r0.mgg'}",
                "--out", str(tmp_path / "s.csv")])
    assert rc == 0
    rows = list(csv.reader(open(tmp_path / "s.csv")))
    assert tuple(rows[0]) == ("param", "value", "replicate", "rhs_id", "iters_to_converge", "converged",
                              "final_diff")
    body = rows[1:]
    assert len(body) == 8
    assert [(r[1], r[2], r[3]) for r in body[:4]] == [("1", "0", "r0"), ("1", "0", "r1"), ("1", "1", "r0"),
                                                      ("1", "1", "r1")]
    _, log = orc.solve(orc.sine_modes_rhs(64, 0), orc.Config(N_step=1, r_min=8, N_smooth=2))
    row = next(r for r in body if r[1] == "2" and r[2] == "0" and r[3] == "r0")
    assert int(row[4]) == log.iterations and row[5] == "1"


@pytest.mark.gpu
def test_cli_spectrum_and_datagen(cuda, tmp_path):
    assert _main(["datagen", "--kind", "mode", "--n", "64", "--mode-k", "3", "--out", str(tmp_path / "m")]) == 0
    assert _main(["spectrum", "--in", str(tmp_path / "m_p.mgg"), "--out", str(tmp_path / "sp.csv")]) == 0
    rows = list(csv.reader(open(tmp_path / "sp.csv")))
    assert rows[0] == ["k", "power"] and len(rows) == 64 // 2 + 2
    power = np.array([float(r[1]) for r in rows[1:]])
    assert int(np.argmax(power)) == 3
