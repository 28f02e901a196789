"""Host regeneration of the device-generated BASELINE markets — TEST ORACLE.

Test infrastructure only (oracle/__init__.py).  `generate_rows` returns the
same arrays, byte for byte, as paper_2506_06258_b200.generate.generate_rows
builds on the GPU (oracle/market_gen.c restates csrc/generate.cu), without
loading the product's CUDA library: the CPU reference arm of bench.py builds
its instance with it, and tests/test_oracle.py / the -m gpu parity tests
check the byte identity.
"""

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "liborcl_gen.so")
_lib = None
_lock = threading.Lock()

# BASELINE.json configs (same table as paper_2506_06258_b200.generate.CONFIGS)
CONFIGS = {
    "c1": dict(n=1000, m=500, q=1.0),
    "c2": dict(n=100_000, m=10_000, q=0.01),
    "c3": dict(n=1_000_000, m=50_000, powerlaw=2.0, mean_degree=100.0),
    "c4": dict(n=10_000_000, m=100_000, q=1e-3),
    "c5": dict(n=100_000, m=100_000, q=0.01),
}


def _load():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                subprocess.run(["make", "-s", "-C", _HERE], check=True)
            lib = ctypes.CDLL(_LIB_PATH)
            P, i64, f64, cint = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
            u64 = ctypes.c_uint64
            lib.orc_gen_degrees.argtypes = [i64, i64, i64, cint, f64, f64, f64, u64, P, cint]
            lib.orc_gen_fill.argtypes = [i64, i64, i64, cint, f64, f64, f64, u64, P, P, P, P,
                                         cint]
            lib.orc_gm_log.restype = f64
            lib.orc_gm_log.argtypes = [f64]
            lib.orc_gm_exp.restype = f64
            lib.orc_gm_exp.argtypes = [f64]
            _lib = lib
    return _lib


def powerlaw_dmin(m, alpha, mean_degree):
    """dmin with E[min(dmin U^(-1/(alpha-1)), m)] = mean_degree (restates
    generate.powerlaw_dmin: 200 bisection steps on the closed-form mean)."""

    def mean(dmin):
        k = 1.0 / (alpha - 1.0)
        uc = (dmin / m) ** (1.0 / k)
        if abs(k - 1.0) < 1e-12:
            tail = dmin * math.log(1.0 / uc)
        else:
            tail = dmin * (1.0 - uc ** (1.0 - k)) / (1.0 - k)
        return m * uc + tail

    lo, hi = 1e-9, float(m)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if mean(mid) < mean_degree:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def generate_rows(n, m, seed=0, q=None, powerlaw=None, mean_degree=None, row0=0, nrows=None,
                  threads=None):
    """Rows [row0, row0+nrows) of the synthetic n x m market, on the host.

    Returns dict(row_ptr int64 [nrows+1], col int32, u float64, w float64).
    """
    lib = _load()
    threads = int(threads or os.cpu_count() or 1)
    nrows = n - row0 if nrows is None else nrows
    if powerlaw is not None:
        q_mode, alpha, dmin, qq = 1, float(powerlaw), powerlaw_dmin(m, powerlaw, mean_degree), 0.0
    else:
        q_mode, alpha, dmin, qq = 0, 2.0, 1.0, float(q)
    deg = np.empty(nrows, dtype=np.int64)
    lib.orc_gen_degrees(row0, nrows, m, q_mode, qq, alpha, dmin, seed, _ptr(deg), threads)
    row_ptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    del deg
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    w = np.empty(nrows, dtype=np.float64)
    lib.orc_gen_fill(row0, nrows, m, q_mode, qq, alpha, dmin, seed, _ptr(row_ptr), _ptr(col),
                     _ptr(val), _ptr(w), threads)
    return {"row_ptr": row_ptr, "col": col, "u": val, "w": w, "row0": row0, "n": n, "m": m}


def generate_config(name, seed=0, row0=0, nrows=None, threads=None):
    c = dict(CONFIGS[name])
    n, m = c.pop("n"), c.pop("m")
    return generate_rows(n, m, seed=seed, row0=row0, nrows=nrows, threads=threads, **c)


def gm_log(x):
    return _load().orc_gm_log(float(x))


def gm_exp(y):
    return _load().orc_gm_exp(float(y))
