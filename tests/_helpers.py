"""Shared helpers for the parity tests."""

import ctypes

import numpy as np


def instance_from(g, prefix=""):
    from paper_2506_06258_b200 import FisherInstance, SparseMatrix

    u = SparseMatrix(int(g["n"]), int(g["m"]), g[prefix + "indptr"], g[prefix + "col"],
                     g[prefix + "u"])
    return FisherInstance(u, g["w"])


def oracle_market(inst):
    from oracle import solve as orc

    u = inst.utilities
    return orc.Market(u.n_rows, u.n_cols, u.row_offsets, u.col_indices, u.values, inst.budgets)


def stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def device_ksection_chunk(g, state=None, iters=None, subtol=None, sections=None):
    """Run the faithful drop-in mq_pdhcg_chunk on a golden chunk case."""
    import torch

    from paper_2506_06258_b200 import _native as nat

    lib = nat.lib()

    def d(a, dt=torch.float64):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device="cuda")

    st = state or {k: g[f"in_{k}"] for k in ("x", "x_prev", "p", "xbar", "pbar")}
    iters = int(g["iters"]) if iters is None else iters
    X, XP, P, XB, PB = (d(st[k]) for k in ("x", "x_prev", "p", "xbar", "pbar"))
    args = [d(g["indptr"], torch.int64), d(g["col"], torch.int32), d(g["u"]),
            d(g["tperm"], torch.int32), d(g["tindptr"], torch.int64), d(g["w"])]
    nnz = len(g["u"])
    cbuf = torch.empty(max(nnz, 1), dtype=torch.float64, device="cuda")
    pass_out = torch.zeros(iters, dtype=torch.int64, device="cuda")
    navg = ctypes.c_int64(0)
    rc = lib.mq_pdhcg_chunk(int(g["n"]), int(g["m"]), *[nat.ptr(a) for a in args], nat.ptr(X),
                            nat.ptr(XP), nat.ptr(P), nat.ptr(XB), nat.ptr(PB), int(g["navg_in"]),
                            float(g["tau"]), float(g["sigma"]),
                            int(g["sections"]) if sections is None else sections,
                            float(g["subtol"]) if subtol is None else subtol, iters,
                            nat.ptr(cbuf), nat.ptr(pass_out), ctypes.byref(navg), stream())
    nat.check(rc, "mq_pdhcg_chunk")
    out = {k: v.cpu().numpy() for k, v in
           (("x", X), ("x_prev", XP), ("p", P), ("xbar", XB), ("pbar", PB))}
    out["passes"] = pass_out.cpu().numpy()
    out["navg"] = navg.value
    out["faults"] = rc
    return out


def rel_max(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))
