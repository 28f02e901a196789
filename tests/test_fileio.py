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


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["mtx", "csv"])
def test_streamed_device_ingest_matches_the_host_reader(tmp_path, fmt):
    """fileio.load_device parses the files in chunks straight into device CSR:
    the same market as the host reader (device fingerprint == host
    fingerprint) and the same solve."""
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200 import fileio

    inst = mq.generate_fisher(mq.GeneratorConfig(n=3000, m=700, sparsity_u=0.02, seed=4))
    fileio.save(inst, str(tmp_path / "m"), fmt=fmt)
    dinst = fileio.load_device(str(tmp_path / "m"), fmt=fmt, chunk_entries=4096)
    host = fileio.load(str(tmp_path / "m"), fmt=fmt)
    assert fileio.device_fingerprint(dinst.dm, dinst.budgets) == mq.instance_fingerprint(host)
    a = mq.run_solve(dinst, mq.SolveConfig(tol=1e-5), "pdhcg")
    b = mq.run_solve(host, mq.SolveConfig(tol=1e-5), "pdhcg")
    assert a.inner_iterations == b.inner_iterations and a.restarts == b.restarts
    assert np.array_equal(a.prices, b.prices) and np.array_equal(a.allocation, b.allocation)
    assert a.instance_fingerprint == b.instance_fingerprint


@pytest.mark.gpu
def test_streamed_ingest_reports_the_reference_errors(tmp_path):
    """A malformed file falls back to the host reader: the reference's
    ParseError with its line number."""
    from paper_2506_06258_b200 import fileio
    from paper_2506_06258_b200.errors import ParseError

    (tmp_path / "b.u.mtx").write_text("%%MatrixMarket matrix coordinate real general\n"
                                      "3 2 3\n1 1 0.5\n2 2 x\n3 1 0.25\n")
    (tmp_path / "b.w.txt").write_text("1\n1\n1\n")
    with pytest.raises(ParseError, match="line 4"):
        fileio.load_device(str(tmp_path / "b"))
    (tmp_path / "c.u.mtx").write_text("%%MatrixMarket matrix coordinate real general\n"
                                      "3 2 3\n1 1 0.5\n2 3 1.0\n3 1 0.25\n")
    (tmp_path / "c.w.txt").write_text("1\n1\n1\n")
    with pytest.raises(ParseError, match="outside"):
        fileio.load_device(str(tmp_path / "c"))
