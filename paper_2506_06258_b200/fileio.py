"""Instance files (market_eq/fileio.py): Matrix Market coordinate matrices
(1-based, `%%MatrixMarket matrix coordinate real general`) or CSV triplets
(0-based, `rows,cols,nnz` header), budgets one per line in a sidecar.  A
Fisher instance saved under prefix P is `P.u.<fmt>` + `P.w.txt`, an exchange
instance `P.u.<fmt>` + `P.e.<fmt>`.  Values are written with 17 significant
digits, so a save/load round trip is exact and the files are byte-identical
to the reference's.

Reading is vectorized (one numpy pass over the entry block, then checks on
whole arrays); only a file that fails a check is re-scanned line by line, to
raise the reference's ParseError with the offending line number.
"""

import os

import numpy as np

from .errors import ParseError, StructureError
from .instance import ExchangeInstance, FisherInstance
from .sparse import SparseMatrix

FORMATS = ("mtx", "csv")

_MM_HEADER = "%%MatrixMarket matrix coordinate real general"


# ------------------------------------------------------------------ writing
def _write_entries(path, head, rows, cols, vals, sep):
    with open(path, "w") as fh:
        fh.write(head)
        fh.writelines(f"{r}{sep}{c}{sep}{v:.17g}\n"
                      for r, c, v in zip(rows.tolist(), cols.tolist(), vals.tolist()))


def write_matrix_market(M, path):
    _write_entries(path, f"{_MM_HEADER}\n{M.n_rows} {M.n_cols} {M.nnz}\n", M.row_ids + 1,
                   M.col_indices + 1, M.values, " ")


def write_csv_triplets(M, path):
    _write_entries(path, f"{M.n_rows},{M.n_cols},{M.nnz}\n", M.row_ids, M.col_indices,
                   M.values, ",")


def write_budgets(w, path):
    with open(path, "w") as fh:
        for v in w:
            fh.write(f"{v:.17g}\n")


# ------------------------------------------------------------------ reading
def _scan_entries(lines, first, path, nnz, n_rows, n_cols, sep, base, comments):
    """Line-by-line parse of the entry block (the exact errors)."""
    shape = "'i j value'" if sep is None else "'i,j,value'"
    rows = np.zeros(nnz, dtype=np.int64)
    cols = np.zeros(nnz, dtype=np.int64)
    vals = np.zeros(nnz, dtype=np.float64)
    k = 0
    for lineno in range(first, len(lines)):
        line = lines[lineno].strip()
        if not line or (comments and line.startswith("%")):
            continue
        parts = line.split(sep)
        if len(parts) != 3:
            raise ParseError(f"entry line must be {shape}", path=path, line=lineno + 1)
        if k >= nnz:
            raise ParseError(f"more than the declared {nnz} entries", path=path,
                             line=lineno + 1)
        try:
            i, j, v = int(parts[0]), int(parts[1]), float(parts[2])
        except ValueError:
            raise ParseError("malformed entry", path=path, line=lineno + 1)
        if not (base <= i < n_rows + base and base <= j < n_cols + base):
            raise ParseError(f"index ({i},{j}) outside {n_rows}x{n_cols}", path=path,
                             line=lineno + 1)
        if v < 0:
            raise ParseError(f"negative value {v!r}", path=path, line=lineno + 1)
        rows[k], cols[k], vals[k] = i - base, j - base, v
        k += 1
    if k != nnz:
        raise ParseError(f"declared {nnz} entries but found {k}", path=path, line=len(lines))
    return rows, cols, vals


def _fast_entries(lines, first, nnz, n_rows, n_cols, sep, base, comments):
    """Vectorized parse; None if anything looks off (the scan then reports)."""
    body = lines[first:]
    if comments:
        body = [ln for ln in body if not ln.lstrip().startswith("%")]
    text = "".join(body)
    if sep is not None:
        text = text.replace(sep, " ")
    try:
        tok = np.array(text.split(), dtype=np.float64)
    except ValueError:
        return None
    if tok.size != 3 * nnz or sum(1 for ln in body if ln.strip()) != nnz:
        return None
    tok = tok.reshape(nnz, 3)
    ri, ci, v = tok[:, 0], tok[:, 1], tok[:, 2]
    if (np.any(ri != np.floor(ri)) or np.any(ci != np.floor(ci)) or np.any(v < 0)
            or np.any(ri < base) or np.any(ri >= n_rows + base)
            or np.any(ci < base) or np.any(ci >= n_cols + base)):
        return None
    # integers must also have been written as integers ("1.0" is malformed)
    idx_tokens = [t for ln in body if ln.strip() for t in ln.replace(sep or " ", " ").split()[:2]]
    if any(not t.lstrip("+-").isdigit() for t in idx_tokens):
        return None
    return ri.astype(np.int64) - base, ci.astype(np.int64) - base, v


def _read(path, lines, first, n_rows, n_cols, nnz, sep, base, comments):
    got = _fast_entries(lines, first, nnz, n_rows, n_cols, sep, base, comments)
    if got is None:
        got = _scan_entries(lines, first, path, nnz, n_rows, n_cols, sep, base, comments)
    return SparseMatrix.from_triplets(n_rows, n_cols, *got)


def read_matrix_market(path):
    with open(path) as fh:
        lines = fh.readlines()
    if not lines:
        raise ParseError("empty file", path=path)
    header = lines[0].strip().lower()
    if not header.startswith("%%matrixmarket"):
        raise ParseError("missing MatrixMarket header", path=path, line=1)
    if header.split()[1:5] != ["matrix", "coordinate", "real", "general"]:
        raise ParseError("only 'matrix coordinate real general' is supported", path=path,
                         line=1)
    idx = 1
    while idx < len(lines) and lines[idx].lstrip().startswith("%"):
        idx += 1
    if idx >= len(lines):
        raise ParseError("missing size line", path=path, line=len(lines))
    parts = lines[idx].split()
    if len(parts) != 3:
        raise ParseError("size line must be 'rows cols nnz'", path=path, line=idx + 1)
    try:
        n_rows, n_cols, nnz = (int(p) for p in parts)
    except ValueError:
        raise ParseError("size line must contain three integers", path=path, line=idx + 1)
    return _read(path, lines, idx + 1, n_rows, n_cols, nnz, None, 1, True)


def read_csv_triplets(path):
    with open(path) as fh:
        lines = fh.readlines()
    if not lines:
        raise ParseError("empty file", path=path)
    parts = lines[0].strip().split(",")
    if len(parts) != 3:
        raise ParseError("header must be 'rows,cols,nnz'", path=path, line=1)
    try:
        n_rows, n_cols, nnz = (int(p) for p in parts)
    except ValueError:
        raise ParseError("header must contain three integers", path=path, line=1)
    return _read(path, lines, 1, n_rows, n_cols, nnz, ",", 0, False)


def read_budgets(path):
    vals = []
    with open(path) as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            try:
                vals.append(float(line))
            except ValueError:
                raise ParseError("budget lines must hold one real number", path=path,
                                 line=lineno)
    return np.asarray(vals, dtype=np.float64)


# ------------------------------------------------------------------ instances
def _matrix_io(fmt):
    if fmt == "mtx":
        return write_matrix_market, read_matrix_market
    if fmt == "csv":
        return write_csv_triplets, read_csv_triplets
    raise ValueError(f"unknown format {fmt!r}; expected one of {FORMATS}")


def save(inst, prefix, fmt="mtx"):
    """Write an instance under a path prefix; returns the files written."""
    writer, _ = _matrix_io(fmt)
    paths = [f"{prefix}.u.{fmt}"]
    if isinstance(inst, FisherInstance):
        writer(inst.utilities, paths[0])
        paths.append(f"{prefix}.w.txt")
        write_budgets(inst.budgets, paths[-1])
    elif isinstance(inst, ExchangeInstance):
        writer(inst.utilities, paths[0])
        paths.append(f"{prefix}.e.{fmt}")
        writer(inst.endowments, paths[-1])
    else:
        raise TypeError(f"unsupported instance type {type(inst)!r}")
    return paths


def load(prefix, fmt="mtx"):
    """Load the Fisher (`.w.txt` sidecar) or exchange (`.e.<fmt>`) instance
    saved under a path prefix."""
    _, reader = _matrix_io(fmt)
    u_path = f"{prefix}.u.{fmt}"
    if not os.path.exists(u_path):
        raise ParseError(f"no utility matrix at {u_path}", path=u_path)
    utilities = reader(u_path)
    w_path, e_path = f"{prefix}.w.txt", f"{prefix}.e.{fmt}"
    if os.path.exists(w_path):
        budgets = read_budgets(w_path)
        if budgets.shape != (utilities.n_rows,):
            raise StructureError(f"{w_path} holds {len(budgets)} budgets but U has "
                                 f"{utilities.n_rows} rows")
        return FisherInstance(utilities, budgets)
    if os.path.exists(e_path):
        return ExchangeInstance(utilities, reader(e_path))
    raise ParseError(f"neither {w_path} nor {e_path} exists", path=prefix)


# ------------------------------------------------------- streamed device ingest
class DeviceFisherInstance:
    """A Fisher instance read from its files straight into device CSR
    (load_device): the DeviceMarket and the host budgets.  run_solve accepts
    it like a FisherInstance; no host copy of the utility matrix exists."""

    def __init__(self, dm, budgets, source):
        self.dm = dm
        self.budgets = budgets
        self.source = source

    @property
    def n_buyers(self):
        return self.dm.n

    @property
    def n_goods(self):
        return self.dm.m


def _size_line(path, fmt):
    """(n_rows, n_cols, nnz, lines before the entries) from the header."""
    with open(path) as fh:
        if fmt == "csv":
            parts = fh.readline().strip().split(",")
            return int(parts[0]), int(parts[1]), int(parts[2]), 1
        fh.readline()
        skip = 1
        for line in fh:
            skip += 1
            if not line.lstrip().startswith("%"):
                parts = line.split()
                return int(parts[0]), int(parts[1]), int(parts[2]), skip
    raise ValueError("no size line")


def load_device(prefix, fmt="mtx", device=None, chunk_entries=1 << 24):
    """Fisher instance files (`P.u.<fmt>` + `P.w.txt`) parsed in chunks and
    streamed into device CSR (the reference reader's semantics,
    fileio.py:36-139 + SparseMatrix.from_triplets: zeros dropped, entries
    sorted by (row, column), duplicates rejected).  The host parses chunk
    k+1 (pandas' C tokenizer) while chunk k's H2D copy runs; validation,
    the sort and the row offsets run on the device.  A file the fast path
    cannot take (malformed lines, out-of-range or negative entries, a wrong
    count) is re-read by the host reader, which raises the reference's
    ParseError with its line number."""
    import pandas as pd
    import torch

    from .device import DeviceMarket

    u_path, w_path = f"{prefix}.u.{fmt}", f"{prefix}.w.txt"
    if fmt not in FORMATS:
        raise ValueError(f"unknown format {fmt!r}; expected one of {FORMATS}")
    if not os.path.exists(u_path):
        raise ParseError(f"no utility matrix at {u_path}", path=u_path)
    if not os.path.exists(w_path):
        raise ParseError(f"{w_path} does not exist (device ingest reads Fisher instances)",
                         path=prefix)
    dev = torch.device(device if device is not None else "cuda")

    def host_reader():  # the exact errors
        _, reader = _matrix_io(fmt)
        reader(u_path)
        raise ParseError("unreadable entry block", path=u_path)

    try:
        n, m, nnz, skip = _size_line(u_path, fmt)
    except (ValueError, IndexError):
        host_reader()
    budgets = read_budgets(w_path)
    if budgets.shape != (n,):
        raise StructureError(f"{w_path} holds {len(budgets)} budgets but U has {n} rows")
    base = 1 if fmt == "mtx" else 0
    rows = torch.empty(nnz, dtype=torch.int64, device=dev)
    cols = torch.empty(nnz, dtype=torch.int64, device=dev)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    stage = [None, None]
    ev = [None, None]
    off = 0
    try:
        reader = pd.read_csv(u_path, sep=" " if fmt == "mtx" else ",", header=None,
                             skiprows=skip, comment="%" if fmt == "mtx" else None,
                             names=[0, 1, 2], dtype={0: np.int64, 1: np.int64, 2: np.float64},
                             engine="c", chunksize=chunk_entries, skip_blank_lines=True,
                             float_precision="round_trip")  # correctly rounded, as float()
        for k, df in enumerate(reader):
            c = len(df)
            if off + c > nnz:
                host_reader()
            b = k & 1
            if ev[b] is not None:
                ev[b].synchronize()  # the staging buffer's previous copy is done
            stage[b] = [torch.from_numpy(df[j].to_numpy()).pin_memory() for j in (0, 1, 2)]
            rows[off:off + c].copy_(stage[b][0], non_blocking=True)
            cols[off:off + c].copy_(stage[b][1], non_blocking=True)
            vals[off:off + c].copy_(stage[b][2], non_blocking=True)
            ev[b] = torch.cuda.Event()
            ev[b].record()
            off += c
    except (ValueError, pd.errors.ParserError, OverflowError):
        host_reader()
    if off != nnz:
        host_reader()
    rows -= base
    cols -= base
    bad = ((rows < 0) | (rows >= n) | (cols < 0) | (cols >= m) | (vals < 0)).any()
    if bool(bad.item()):
        host_reader()
    keep = vals != 0.0
    if not bool(keep.all().item()):
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
    del keep
    key = rows * m + cols
    del rows
    if bool((key[1:] < key[:-1]).any().item()):
        key, order = torch.sort(key, stable=True)
        cols, vals = cols[order], vals[order]
        del order
    if key.numel() > 1 and bool((key[1:] == key[:-1]).any().item()):
        raise StructureError("duplicate entry in triplets")
    counts = torch.bincount(torch.div(key, m, rounding_mode="floor"), minlength=n)
    del key
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    dm = DeviceMarket(row_ptr, cols.to(torch.int32), vals, budgets, m, device=dev)
    return DeviceFisherInstance(dm, budgets, prefix)


def device_fingerprint(dm, budgets, chunk=1 << 23):
    """instance_fingerprint (report.py:19-36) of a device-resident Fisher
    instance, its arrays streamed back chunk by chunk: byte-identical to the
    fingerprint of the same instance held on the host."""
    import hashlib

    import torch

    h = hashlib.sha256()
    h.update(np.int64([dm.n, dm.m]).tobytes())
    for t, dt in ((dm.row_ptr, torch.int64), (dm.col, torch.int64), (dm.u_orig, torch.float64)):
        for o in range(0, t.numel(), chunk):
            h.update(t[o:o + chunk].to(dt).cpu().numpy().tobytes())
    h.update(b"fisher")
    h.update(np.ascontiguousarray(budgets, dtype=np.float64))
    return h.hexdigest()
