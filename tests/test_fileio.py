"""Instance files (fileio.py) against the reference's own files and reader
verdicts (tests/golden/fileio/, written by the reference through
oracle/gen_golden.py)."""

import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN

HERE = os.path.join(GOLDEN, "fileio")


def test_reads_reference_files():
    from paper_2506_06258_b200 import ExchangeInstance, FisherInstance
    from paper_2506_06258_b200 import fileio

    a = fileio.load(os.path.join(HERE, "fisher"), "mtx")
    b = fileio.load(os.path.join(HERE, "fisher"), "csv")
    e = fileio.load(os.path.join(HERE, "exch"), "mtx")
    assert isinstance(a, FisherInstance) and isinstance(e, ExchangeInstance)
    for x, y in ((a.utilities, b.utilities),):
        assert np.array_equal(x.row_offsets, y.row_offsets)
        assert np.array_equal(x.col_indices, y.col_indices)
        assert np.array_equal(x.values, y.values)
    assert np.array_equal(a.budgets, b.budgets)


@pytest.mark.parametrize("fmt", ["mtx", "csv"])
def test_writes_byte_identical_files(fmt, tmp_path):
    from paper_2506_06258_b200 import fileio

    inst = fileio.load(os.path.join(HERE, "fisher"), fmt)
    paths = fileio.save(inst, str(tmp_path / "fisher"), fmt)
    for p in paths:
        with open(p) as fh, open(os.path.join(HERE, os.path.basename(p))) as ref:
            assert fh.read() == ref.read(), os.path.basename(p)
    ex = fileio.load(os.path.join(HERE, "exch"), "mtx")
    for p in fileio.save(ex, str(tmp_path / "exch"), "mtx"):
        with open(p) as fh, open(os.path.join(HERE, os.path.basename(p))) as ref:
            assert fh.read() == ref.read()


def test_reader_errors_match_reference(tmp_path):
    from paper_2506_06258_b200 import fileio
    from paper_2506_06258_b200.errors import ParseError

    cases = json.load(open(os.path.join(HERE, "errors.json")))
    for name, want in cases.items():
        path = str(tmp_path / name)
        shutil.copy(os.path.join(HERE, name), path)
        reader = fileio.read_matrix_market if name.endswith(".mtx") else fileio.read_csv_triplets
        if want["ok"]:
            M = reader(path)
            assert M.values.tolist() == want["values"] and M.col_indices.tolist() == want["col"]
            assert M.row_offsets.tolist() == want["rows"]
            continue
        with pytest.raises(ParseError) as ei:
            reader(path)
        assert ei.value.line == want["line"], name
        assert str(ei.value).replace(str(tmp_path) + "/", "") == want["msg"], name


def test_unknown_format_and_missing_files(tmp_path):
    from paper_2506_06258_b200 import fileio
    from paper_2506_06258_b200.errors import ParseError

    with pytest.raises(ValueError):
        fileio.load(str(tmp_path / "x"), "json")
    with pytest.raises(ParseError):
        fileio.load(str(tmp_path / "nothing"), "mtx")
