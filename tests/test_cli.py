"""The market-eq command line (cli.py): the reference's commands and exit
codes.  `generate` needs no GPU and must write the reference's exact files."""

import json
import os

import pytest

from conftest import GOLDEN

REF = os.path.join(GOLDEN, "fileio")


def _run(argv, capsys):
    from paper_2506_06258_b200.cli import main

    rc = main(argv)
    return rc, capsys.readouterr()


@pytest.mark.parametrize("fmt", ["mtx", "csv"])
def test_generate_writes_the_reference_files(fmt, tmp_path, capsys):
    rc, out = _run(["generate", "--n", "30", "--m", "12", "--sparsity-u", "0.3", "--seed", "4",
                    "--format", fmt, "--out", str(tmp_path / "fisher")], capsys)
    assert rc == 0
    info = json.loads(out.out)
    for p in info["written"]:
        with open(p) as fh, open(os.path.join(REF, os.path.basename(p))) as ref:
            assert fh.read() == ref.read()


def test_usage_and_data_errors(tmp_path, capsys):
    with pytest.raises(SystemExit) as e:
        _run(["solve"], capsys)
    assert e.value.code == 1
    rc, out = _run(["solve", "--instance", str(tmp_path / "missing")], capsys)
    assert rc == 3 and "no utility matrix" in out.err


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["pdhcg", "pdhg"])
def test_solve_then_check(algo, tmp_path, capsys):
    prefix = str(tmp_path / "m")
    assert _run(["generate", "--n", "60", "--m", "25", "--sparsity-u", "0.3", "--seed", "11",
                 "--out", prefix], capsys)[0] == 0
    rc, out = _run(["solve", "--instance", prefix, "--algo", algo, "--tol", "1e-5"], capsys)
    assert rc == 0 and json.loads(out.out)["status"] == "optimal"
    rc, out = _run(["check", "--instance", prefix, "--solution", prefix + ".report.json"],
                   capsys)
    assert rc == 0 and json.loads(out.out)["matches_report"] is True


@pytest.mark.gpu
def test_exchange_command(tmp_path, capsys):
    prefix = str(tmp_path / "e")
    assert _run(["generate", "--kind", "exchange", "--n", "20", "--m", "15", "--sparsity-u",
                 "0.4", "--seed", "2", "--out", prefix], capsys)[0] == 0
    rc, out = _run(["exchange", "--instance", prefix, "--outer-tol", "1e-5"], capsys)
    info = json.loads(out.out)
    assert rc in (0, 2) and info["trace"].endswith(".trace.json")
    assert os.path.exists(info["trace"])
