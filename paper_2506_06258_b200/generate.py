"""Device-side synthetic markets for the large BASELINE configs.

The reference's generator (instance.py:141-226) draws n*m host uniforms —
1e12 at config 4 — so configs 3-5 are generated on the GPU instead, row by
row from Philox subsequences (csrc/generate.cu): the same Bernoulli-support /
U(0,1] value law, empty rows repaired with one uniform entry, and any row
range can be produced independently (a rank generates only its shard).
"""

import ctypes
import math

import torch

from . import _native as nat
from .errors import ValidationError

# BASELINE.json configs (n, m, kind, parameter)
CONFIGS = {
    "c1": dict(n=1000, m=500, q=1.0),
    "c2": dict(n=100_000, m=10_000, q=0.01),
    "c3": dict(n=1_000_000, m=50_000, powerlaw=2.0, mean_degree=100.0),
    "c4": dict(n=10_000_000, m=100_000, q=1e-3),
    "c5": dict(n=100_000, m=100_000, q=0.01),
}


def powerlaw_dmin(m, alpha, mean_degree):
    """dmin such that E[min(dmin U^(-1/(alpha-1)), m)] = mean_degree."""

    def mean(dmin):
        k = 1.0 / (alpha - 1.0)
        uc = (dmin / m) ** (1.0 / k)          # below uc the degree is capped at m
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


def generate_rows(n, m, seed=0, q=None, powerlaw=None, mean_degree=None, row0=0, nrows=None,
                  device=None, budgets=True):
    """Rows [row0, row0+nrows) of a synthetic n x m market on the device.

    Returns dict(row_ptr int64 [nrows+1] (local), col int32, u float64, w float64|None).
    """
    lib = nat.lib()
    dev = torch.device(device if device is not None else "cuda")
    nrows = n - row0 if nrows is None else nrows
    if powerlaw is not None:
        q_mode, alpha, dmin, qq = 1, float(powerlaw), powerlaw_dmin(m, powerlaw, mean_degree), 0.0
    else:
        q_mode, alpha, dmin, qq = 0, 2.0, 1.0, float(q)
    s = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    deg = torch.empty(nrows, dtype=torch.int64, device=dev)
    nat.check(lib.mq_gen_degrees(row0, nrows, m, q_mode, qq, alpha, dmin, seed,
                                 nat.ptr(deg), s), "mq_gen_degrees")
    row_ptr = torch.zeros(nrows + 1, dtype=torch.int64, device=dev)
    torch.cumsum(deg, 0, out=row_ptr[1:])
    del deg
    nnz = int(row_ptr[-1].item())
    if nnz >= 2 ** 31:
        raise ValidationError("shard exceeds int32 entry indexing; use more shards")
    col = torch.empty(nnz, dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    w = torch.empty(nrows, dtype=torch.float64, device=dev) if budgets else None
    nat.check(lib.mq_gen_fill(row0, nrows, m, q_mode, qq, alpha, dmin, seed, nat.ptr(row_ptr),
                              nat.ptr(col), nat.ptr(val), nat.ptr(w), s), "mq_gen_fill")
    return {"row_ptr": row_ptr, "col": col, "u": val, "w": w, "row0": row0, "n": n, "m": m}


def generate_config(name, seed=0, row0=0, nrows=None, device=None):
    c = dict(CONFIGS[name])
    n, m = c.pop("n"), c.pop("m")
    return generate_rows(n, m, seed=seed, row0=row0, nrows=nrows, device=device, **c)
