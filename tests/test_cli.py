"""Bench-row CLI (reference output contract, cli.py:47-51,336-410)."""

import csv
import io

import pytest

from paper_2508_05958_b200 import cli


def test_usage_errors_exit_2(capsys):
    assert cli.main(["bench-uniform", "--dim", "2", "--kernel", "slp3d", "--n", "16"]) == 2
    assert cli.main(["bench-uniform", "--dim", "2", "--n", "10", "--leaf", "4"]) == 2
    assert cli.main(["bench-uniform", "--dim", "2", "--n", "16", "--baseline"]) == 2
    assert "usage error" in capsys.readouterr().err


def test_argparse_errors_exit_nonzero():
    assert cli.main(["bench-uniform"]) != 0
    assert cli.main(["no-such-command"]) != 0


@pytest.mark.gpu
def test_bench_uniform_csv_row(capsys):
    rc = cli.main(["bench-uniform", "--dim", "2", "--kernel", "gaussian", "--n", "64", "--p", "8",
                   "--leaf", "16", "--adm", "weak"])
    assert rc == 0
    rows = list(csv.DictReader(io.StringIO(capsys.readouterr().out)))
    assert len(rows) == 1 and list(rows[0]) == cli.UNIFORM_HEADER
    assert rows[0]["variant"] == "htlr-b200"
    assert float(rows[0]["e_apply_rand"]) < 1e-9
