"""Bench-row CLI (reference output contract, cli.py:47-51,336-410)."""

import csv
import io

import pytest

from paper_2508_05958_b200 import cli


def test_usage_errors_exit_2(capsys):
    assert cli.main(["bench-uniform", "--dim", "2", "--kernel", "slp3d", "--n", "16"]) == 2
    assert cli.main(["bench-uniform", "--dim", "2", "--n", "10", "--leaf", "4"]) == 2
    assert cli.main(["bench-quasi", "--n", "7"]) == 2
    assert cli.main(["bench-quasi", "--dim", "3", "--n", "8"]) == 2
    assert "usage error" in capsys.readouterr().err


def test_argparse_errors_exit_nonzero():
    assert cli.main(["bench-uniform"]) != 0
    assert cli.main(["no-such-command"]) != 0


@pytest.mark.gpu
def test_bench_uniform_csv_row(capsys):
    rc = cli.main(["bench-uniform", "--dim", "2", "--kernel", "gaussian", "--n", "64", "--p", "8",
                   "--leaf", "16", "--adm", "weak", "--baseline"])
    assert rc == 0
    rows = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert len(rows) == 2 and list(rows[0]) == cli.UNIFORM_HEADER
    assert [r["variant"] for r in rows] == ["htlr-b200", "hmatrix-b200"]
    assert float(rows[0]["e_apply_rand"]) < 1e-9 and float(rows[1]["e_apply_rand"]) < 1e-9
    assert int(rows[1]["total_scalars"]) > int(rows[0]["total_scalars"])


@pytest.mark.gpu
def test_bench_quasi_rows(capsys):
    rc = cli.main(["bench-quasi", "--n", "128", "--p", "4", "--leaf", "4", "--rho", "2", "--format", "json"])
    assert rc == 0
    import json
    rows = json.loads(capsys.readouterr().out)
    assert rows[0]["variant"] == "htlr-quasi-b200" and rows[0]["n_quasi"] == 128
