"""Numpy restatement of the reference's restarted PDHCG solve — TEST ORACLE.

Test infrastructure only (see oracle/__init__.py).  Every numpy operation
below is the one the reference issues, in the same order, so results are
bit-identical to the reference on the same inputs:

  normalize / validate       instance.py:87-138
  transpose schedule         sparse.py:130-145
  initial compact state      pdhcg.py:66-72
  op-norm of the selector    driver.py:117-121, sparse.py:213-233
  omega_0 residual norms     driver.py:123-132
  residuals                  kkt.py:29-87, eg_objective kkt.py:126-131
  restart / step controller  adaptive.py:17-118
  solve loop                 driver.py:271-377 (PDHCG branch only)
  Arrow-Debreu outer loop    exchange.py:75-156

The per-iteration work runs in the C restatement of kernels.pdhcg_chunk
(oracle/pdhcg_oracle.c) through ctypes.
"""

import ctypes
import math
import os
import subprocess
import threading
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "lib", "liborcl_pdhcg.so")
_lib = None
_lib_lock = threading.Lock()

OMEGA_BOUND_FACTOR = 16.0          # driver.py:31
ETA_LOWER_FACTOR = 0.01            # adaptive.py:48
ETA_UPPER_FACTOR = 3.0             # adaptive.py:49
OMEGA_CHECK_INTERVAL = 3           # adaptive.py:50
MAX_ROW_PASSES = 200               # kernels.py:16


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load():
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            lib = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            i64, f64, cint = ctypes.c_int64, ctypes.c_double, ctypes.c_int
            lib.orc_pdhcg_chunk.restype = i64
            lib.orc_pdhcg_chunk.argtypes = [i64, i64, P, P, P, P, P, P, P, P, P, P, P,
                                            i64, f64, f64, cint, f64, cint, P, P, P]
            lib.orc_row_root.restype = f64
            lib.orc_row_root.argtypes = [i64, i64, P, P, f64, f64, cint, f64, P]
            lib.orc_set_threads.restype = cint
            lib.orc_set_threads.argtypes = [cint]
            lib.orc_normalize.restype = i64
            lib.orc_normalize.argtypes = [i64, P, P, P, P]
            lib.orc_transpose.restype = cint
            lib.orc_transpose.argtypes = [i64, i64, P, P, P]
            lib.orc_colsums.restype = None
            lib.orc_colsums.argtypes = [i64, P, P, P, P]
            _lib = lib
    return _lib


def set_threads(n):
    """Thread count of the C chunk (results do not depend on it)."""
    return _load().orc_set_threads(int(n))


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _need(a, dtype):
    if a.dtype != dtype or not a.flags.c_contiguous:
        raise TypeError(f"oracle array must be C-contiguous {dtype}")
    return a


def pdhcg_chunk(indptr, colind, uval, tperm, tindptr, w, x, x_prev, p, xbar, pbar,
                navg, tau, sigma, sections, subtol, iters, c_buf, pass_out):
    """Same signature and in-place semantics as kernels.pdhcg_chunk
    (kernels.py:99-145); returns (navg, faults)."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    tindptr = np.ascontiguousarray(tindptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind, dtype=np.int32)
    tperm = np.ascontiguousarray(tperm, dtype=np.int32)
    uval = np.ascontiguousarray(uval, dtype=np.float64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    for a in (x, x_prev, p, xbar, pbar, c_buf):
        _need(a, np.float64)
    _need(pass_out, np.int64)
    faults = ctypes.c_int64(0)
    n = len(indptr) - 1
    m = len(tindptr) - 1
    navg = lib.orc_pdhcg_chunk(n, m, _ptr(indptr), _ptr(colind), _ptr(uval), _ptr(tperm),
                               _ptr(tindptr), _ptr(w), _ptr(x), _ptr(x_prev), _ptr(p),
                               _ptr(xbar), _ptr(pbar), int(navg), float(tau), float(sigma),
                               int(sections), float(subtol), int(iters), _ptr(c_buf),
                               _ptr(pass_out), ctypes.byref(faults))
    return int(navg), int(faults.value)


def row_root(uval, cbuf, tw, s0, sections=32, tol=1e-10):
    """One row's k-section root (kernels.py:33-96): returns (s, passes)."""
    lib = _load()
    uval = np.ascontiguousarray(uval, dtype=np.float64)
    cbuf = np.ascontiguousarray(cbuf, dtype=np.float64)
    passes = ctypes.c_int64(0)
    s = lib.orc_row_root(0, len(uval), _ptr(uval), _ptr(cbuf), float(tw), float(s0),
                         int(sections), float(tol), ctypes.byref(passes))
    return s, int(passes.value)


# ------------------------------------------------- large-market setup (C)

def normalize_rows(indptr, val):
    """(val / row max, row max) as instance.py:118-138 computes them, in C
    (the numpy path needs nnz-sized int64 temporaries at config 4)."""
    lib = _load()
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    n = len(indptr) - 1
    out = np.empty_like(val)
    scales = np.empty(n)
    if lib.orc_normalize(n, _ptr(indptr), _ptr(val), _ptr(out), _ptr(scales)):
        raise ValueError("cannot normalize: some buyer values no good")
    return out, scales


def transpose_int32(col, m):
    """(tperm int32, tindptr int64) = sparse.py:130-145's stable argsort by
    column, as a parallel stable counting sort."""
    lib = _load()
    col = np.ascontiguousarray(col, dtype=np.int32)
    tperm = np.empty(len(col), dtype=np.int32)
    tindptr = np.empty(m + 1, dtype=np.int64)
    if lib.orc_transpose(m, len(col), _ptr(col), _ptr(tperm), _ptr(tindptr)):
        raise MemoryError("orc_transpose scratch")
    return tperm, tindptr


def column_sums_sched(tperm, tindptr, v):
    """np.bincount(col, weights=v) through the transpose schedule."""
    out = np.empty(len(tindptr) - 1)
    _load().orc_colsums(len(out), _ptr(tperm), _ptr(tindptr), _ptr(v), _ptr(out))
    return out


def selector_norm_from_counts(counts, iters=50):
    """The reference's op-norm power iteration (sparse.py:213-233) run on the
    column counts (its iterate is constant within a column): equal to
    op_norm_estimate of the selector to ~1e-15 at O(m) cost."""
    c = np.asarray(counts, dtype=np.float64)
    nnz = float(c.sum())
    if nnz == 0 or len(c) == 0:
        return 0.0
    v = np.full(len(c), 1.0 / np.sqrt(nnz))
    sig = 0.0
    for _ in range(iters):
        wv = c * v
        sig = float(np.sqrt(np.dot(c, wv * wv)))
        if sig == 0.0:
            return 0.0
        v = wv / sig
    return float(np.sqrt(sig))


class ChunkRun:
    """The reference's compact iterate on a large market, set up the way
    _CompactRun (driver.py:94-132) does it: normalized utilities, transpose
    schedule, initial state x = 1/colcount, p = sum(w)/m (pdhcg.py:66-72),
    L from the column counts, omega_0 from the residual norms and the first
    restart window's steps tau = eta/omega, sigma = eta*omega with
    eta = 0.9 / L (adaptive.py).  `step(k)` runs k iterations of the
    restated kernels.pdhcg_chunk and returns their pass counts."""

    def __init__(self, row_ptr, col, val, w, m, sections=32, subtol=1e-10):
        self.indptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.w = np.ascontiguousarray(w, dtype=np.float64)
        self.n, self.m = len(self.indptr) - 1, int(m)
        self.val, _ = normalize_rows(self.indptr, val)
        self.tperm, self.tindptr = transpose_int32(self.col, self.m)
        counts = np.diff(self.tindptr).astype(np.float64)
        self.x = (1.0 / counts)[self.col]
        self.p = np.full(self.m, float(np.sum(self.w)) / self.m)
        self.x_prev, self.xbar, self.pbar = self.x.copy(), self.x.copy(), self.p.copy()
        self.cbuf = np.empty_like(self.x)
        self.navg = 0
        self.L = max(selector_norm_from_counts(counts), np.finfo(float).tiny)
        primal = float(np.linalg.norm(column_sums_sched(self.tperm, self.tindptr, self.x) - 1.0))
        if primal > 1e-8:  # driver.py:123-132 needs the dual residual too
            ux = np.add.reduceat(self.val * self.x, self.indptr[:-1])
            uy = self.val * np.repeat(self.w / ux, np.diff(self.indptr))
            best = np.full(self.m, -np.inf)
            np.maximum.at(best, self.col, uy)
            dual = float(np.linalg.norm(np.minimum(self.p - best, 0.0)))
            self.omega0 = max(1.0, dual / primal) if dual > 1e-8 else 1.0
        else:
            self.omega0 = 1.0
        eta = 0.9 / self.L
        self.tau, self.sigma = eta / self.omega0, eta * self.omega0
        self.sections, self.subtol = sections, subtol

    def step(self, iters=1):
        passes = np.zeros(iters, dtype=np.int64)
        self.navg, faults = pdhcg_chunk(self.indptr, self.col, self.val, self.tperm,
                                        self.tindptr, self.w, self.x, self.x_prev, self.p,
                                        self.xbar, self.pbar, self.navg, self.tau, self.sigma,
                                        self.sections, self.subtol, iters, self.cbuf, passes)
        if faults:
            raise RuntimeError(f"{faults} row subproblems exceeded {MAX_ROW_PASSES} passes")
        return passes


# ---------------------------------------------------------------- market data

class Market:
    """CSR utilities + budgets (the oracle's own minimal container)."""

    def __init__(self, n, m, indptr, col, val, w):
        self.n, self.m = int(n), int(m)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int64)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        self.w = np.ascontiguousarray(w, dtype=np.float64)
        self.row_ids = np.repeat(np.arange(self.n), np.diff(self.indptr))

    @property
    def nnz(self):
        return len(self.val)

    @classmethod
    def from_dense(cls, dense, w):
        dense = np.asarray(dense, dtype=np.float64)
        rows, cols = np.nonzero(dense)
        indptr = np.zeros(dense.shape[0] + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=dense.shape[0]), out=indptr[1:])
        return cls(dense.shape[0], dense.shape[1], indptr, cols, dense[rows, cols], w)

    def with_values(self, val, w=None):
        return Market(self.n, self.m, self.indptr, self.col, val,
                      self.w if w is None else w)

    # storage-order accumulations (sparse.py:147-171, 200-210)
    def row_sums(self, v):
        return np.bincount(self.row_ids, weights=v, minlength=self.n)

    def col_sums(self, v):
        return np.bincount(self.col, weights=v, minlength=self.m)

    def apply(self, dense):
        return np.bincount(self.row_ids, weights=self.val * dense[self.col], minlength=self.n)


def validate(mk):
    bad = []
    if np.any(np.diff(mk.indptr) == 0):
        bad.append("buyer values no good")
    if np.any(np.bincount(mk.col, minlength=mk.m) == 0):
        bad.append("good unvalued")
    if np.any(mk.w <= 0):
        bad.append("nonpositive budget")
    return bad


def normalize(mk):
    scales = np.zeros(mk.n)
    np.maximum.at(scales, mk.row_ids, mk.val)
    if np.any(scales == 0):
        raise ValueError("cannot normalize: some buyer values no good")
    return mk.with_values(mk.val / scales[mk.row_ids]), scales


def transpose_schedule(mk):
    tperm = np.argsort(mk.col, kind="stable").astype(np.int64)
    tindptr = np.zeros(mk.m + 1, dtype=np.int64)
    np.cumsum(np.bincount(mk.col, minlength=mk.m), out=tindptr[1:])
    return tperm, tindptr


def selector_op_norm(mk, tperm, iters=50):
    """op_norm_estimate of the m x nnz column selector, through the same
    bincount/norm sequence the reference runs on it (sparse.py:213-233)."""
    nnz = mk.nnz
    if nnz == 0 or mk.m == 0:
        return 0.0
    sel_rows = mk.col[tperm]           # selector row ids in storage order
    sel_cols = tperm                   # selector column indices
    ones = np.ones(nnz)
    v = np.full(nnz, 1.0 / np.sqrt(nnz))
    sig = 0.0
    for _ in range(iters):
        u = np.bincount(sel_rows, weights=ones * v[sel_cols], minlength=mk.m)
        wv = np.bincount(sel_cols, weights=ones * u[sel_rows], minlength=nnz)
        sig = np.linalg.norm(wv)
        if sig == 0.0:
            return 0.0
        v = wv / sig
    return float(np.sqrt(sig))


# ------------------------------------------------------------------ residuals

def residuals_lifted(mk, x, t, p, y):
    """(r_primal, r_dual, r_gap, rel_kkt) — kkt.py:29-76."""
    if np.any(t <= 0):
        raise ValueError("residuals require strictly positive t")
    cs = mk.col_sums(x)
    ux = mk.row_sums(mk.val * x)
    row_gap = np.max(np.abs(t - ux)) if len(t) else 0.0
    col_gap = np.max(np.abs(cs - 1.0)) if len(cs) else 0.0
    r_primal = max(col_gap, row_gap) / (1.0 + max(np.max(np.abs(cs), initial=0.0), row_gap, 1.0))
    wt = mk.w / t
    dual_t = np.max(np.abs(wt - y), initial=0.0)
    uy = mk.val * y[mk.row_ids]
    best = np.full(mk.m, -np.inf)
    np.maximum.at(best, mk.col, uy)
    slack = p - best
    dual_p = np.max(np.maximum(-slack, 0.0), initial=0.0)
    r_dual = max(dual_t, dual_p) / (1.0 + max(np.max(np.abs(wt), initial=0.0),
                                             np.max(np.abs(y), initial=0.0),
                                             np.max(slack, initial=0.0)))
    es = np.maximum(p[mk.col] - uy, 0.0)
    r_gap = np.max(x * es, initial=0.0) / (1.0 + max(np.max(np.abs(x), initial=0.0),
                                                    np.max(es, initial=0.0)))
    rel = max(r_primal, r_dual, r_gap)
    return (float(r_primal), float(r_dual), float(r_gap), float(rel))


def residuals_compact(mk, x, p):
    """kkt.py:79-87: t = u.x per buyer, y = w / t."""
    x = np.asarray(x, dtype=np.float64)
    ux = mk.row_sums(mk.val * x)
    if np.any(ux <= 0):
        i = int(np.nonzero(ux <= 0)[0][0])
        raise ValueError(f"buyer {i} has zero utility value; state is not a "
                         "valid compact iterate")
    return residuals_lifted(mk, x, ux, p, mk.w / ux)


def eg_objective(mk, x):
    """-sum_i w_i log(u_i . x_i) on the given instance (kkt.py:126-131)."""
    ux = mk.row_sums(mk.val * np.asarray(x, dtype=np.float64))
    if np.any(ux <= 0):
        return np.inf
    return float(-np.dot(mk.w, np.log(ux)))


# ----------------------------------------------------------------- controller

def should_restart(now, at_restart, prev, inner_len, total, beta=(0.2, 0.8, 0.2)):
    """adaptive.py:29-45."""
    b_suff, b_nec, b_art = beta
    if now < 0 or at_restart < 0 or prev < 0:
        raise ValueError("metrics must be nonnegative")
    if now <= b_suff * at_restart:
        return True
    if now <= b_nec * at_restart and now > prev:
        return True
    return inner_len >= b_art * total


class Steps:
    """eta/omega controller: tau = eta/omega, sigma = eta*omega (adaptive.py:53-118)."""

    def __init__(self, eta0, omega0, eta_max, omega_lo, omega_hi, theta=0.2):
        self.eta0, self.omega0 = eta0, omega0
        self.eta, self.omega = eta0, omega0
        self.eta_max, self.lo, self.hi, self.theta = eta_max, omega_lo, omega_hi, theta
        self.since = 0

    @property
    def tau(self):
        return self.eta / self.omega

    @property
    def sigma(self):
        return self.eta * self.omega

    def update(self, primal_move, dual_move, eta_obs):
        th = self.theta
        if primal_move > 0.0 and dual_move > 0.0:
            self.omega = math.exp(th * math.log(dual_move / primal_move)
                                  + (1.0 - th) * math.log(self.omega))
        self.since += 1
        if self.since >= OMEGA_CHECK_INTERVAL:
            self.since = 0
            if not self.lo <= self.omega <= self.hi:
                self.omega = self.omega0
        if eta_obs is not None and eta_obs > 0.0:
            self.eta = math.exp(th * math.log(eta_obs) + (1.0 - th) * math.log(self.eta))
        lo = ETA_LOWER_FACTOR * self.eta0
        hi = min(ETA_UPPER_FACTOR * self.eta0, self.eta_max)
        self.eta = min(max(self.eta, lo), hi)


# ---------------------------------------------------------------- solve loop

def solve(mk, tol=1e-4, max_iters=100_000, sections=32, subtol=1e-10,
          check_every=40, warm_start=None, step_mode="adaptive", adapt_eta=True,
          restart="adaptive", restart_k=0, beta=(0.2, 0.8, 0.2), threads=None):
    """Restarted PDHCG (driver.py:271-377, algo="pdhcg"); returns a dict
    with the SolveReport fields (plus "objective")."""
    if threads is not None:
        set_threads(threads)
    bad = validate(mk)
    if bad:
        raise ValueError("; ".join(bad))
    nm, _ = normalize(mk)
    tperm, tindptr = transpose_schedule(nm)
    col32 = nm.col.astype(np.int32)
    tperm32 = tperm.astype(np.int32)
    if warm_start is not None:
        x = np.array(warm_start["x"], dtype=np.float64)
        p = np.array(warm_start["p"], dtype=np.float64)
        if x.shape != (nm.nnz,) or p.shape != (nm.m,):
            raise ValueError("warm start shapes do not match the instance")
        if np.any(nm.row_sums(nm.val * x) <= 0):
            raise ValueError("warm start gives some buyer zero utility")
    else:
        counts = np.bincount(nm.col, minlength=nm.m)
        x = 1.0 / counts[nm.col].astype(np.float64)
        p = np.full(nm.m, float(np.sum(nm.w)) / nm.m)
    x_prev = x.copy()
    xbar, pbar = x.copy(), p.copy()
    navg = 0
    cbuf = np.empty(nm.nnz)
    passes = []
    L = max(selector_op_norm(nm, tperm), np.finfo(float).tiny)

    if step_mode == "theory":
        steps = None
        tau = sigma = 1.0 / (2.0 * L)
    else:
        primal = np.linalg.norm(nm.col_sums(x) - 1.0)
        ux = nm.row_sums(nm.val * x)
        uy = nm.val * (nm.w / ux)[nm.row_ids]
        best = np.full(nm.m, -np.inf)
        np.maximum.at(best, nm.col, uy)
        dual = np.linalg.norm(np.minimum(p - best, 0.0))
        primal, dual = float(primal), float(dual)
        omega0 = max(1.0, dual / primal) if (primal > 1e-8 and dual > 1e-8) else 1.0
        steps = Steps(0.9 / L, omega0, 0.95 / L, omega0 / OMEGA_BOUND_FACTOR,
                      omega0 * OMEGA_BOUND_FACTOR)
        tau, sigma = steps.tau, steps.sigma

    res_avg = residuals_compact(mk, xbar, pbar)
    at_restart = prev_check = res_avg[3]
    snap = (x.copy(), p.copy())
    history = []
    total = restarts = 0
    t0 = time.perf_counter()
    while True:
        chunk = min(check_every, max_iters - total)
        if restart == "fixed":
            chunk = min(chunk, restart_k - navg)
        pass_out = np.zeros(chunk, dtype=np.int64)
        navg, faults = pdhcg_chunk(nm.indptr, col32, nm.val, tperm32, tindptr, nm.w,
                                   x, x_prev, p, xbar, pbar, navg, tau, sigma,
                                   sections, subtol, chunk, cbuf, pass_out)
        if faults:
            raise RuntimeError(f"{faults} row subproblems exceeded {MAX_ROW_PASSES} passes")
        passes.extend(int(v) for v in pass_out)
        total += chunk
        res_last = residuals_compact(mk, x, p)
        res_avg = residuals_compact(mk, xbar, pbar)
        metric = min(res_last[3], res_avg[3])
        history.append((total, metric))
        if metric <= tol or total >= max_iters:
            if res_avg[3] < res_last[3]:
                x, p = xbar.copy(), pbar.copy()
                final = res_avg
            else:
                final = res_last
            status = "optimal" if metric <= tol else "max-iters"
            break
        if restart == "fixed":
            do_restart = navg >= restart_k
        else:
            do_restart = should_restart(res_avg[3], at_restart, prev_check, navg, total, beta)
        prev_check = res_avg[3]
        if do_restart:
            if steps is not None:
                dx = xbar - snap[0]
                dp = pbar - snap[1]
                inter = abs(float(np.dot(nm.col_sums(dx), dp)))
                pm, dm = float(np.linalg.norm(dx)), float(np.linalg.norm(dp))
                psq, dsq = float(np.dot(dx, dx)), float(np.dot(dp, dp))
                eta_obs = None
                if adapt_eta and inter > 0.0:
                    eta_obs = (steps.omega * psq + dsq / steps.omega) / (2.0 * inter)
                steps.update(pm, dm, eta_obs)
                tau, sigma = steps.tau, steps.sigma
            x[:] = xbar
            p[:] = pbar
            x_prev[:] = x
            navg = 0
            restarts += 1
            snap = (x.copy(), p.copy())
            at_restart = prev_check = res_avg[3]
    wall = time.perf_counter() - t0
    ux = mk.row_sums(mk.val * x)
    return {
        "status": status, "inner_iterations": total, "restarts": restarts,
        "wall_time_seconds": wall, "final_residuals": final,
        "residual_history": history, "prices": p.copy(), "allocation": x.copy(),
        "utility_values": ux, "dual_values": mk.w / ux, "subproblem_passes": passes,
        "objective": eg_objective(mk, x), "op_norm": L, "tau_sigma": (tau, sigma),
    }


# ------------------------------------------------------------ lifted PDHG

def pdhg_chunk(nm, x, x_prev, t, t_prev, p, y, xbar, tbar, pbar, ybar, navg, tau, sigma,
               iters):
    """kernels.py:146-197 (pdhg_chunk) in numpy, same operations in the same
    order: the column sums accumulate each column in ascending row order and
    the row sums each row in storage order (np.bincount is sequential), every
    elementwise step rounds as numba's (no contraction).  In place; returns
    the new navg."""
    count = navg
    for _ in range(iters):
        ext = 2.0 * x - x_prev
        p += sigma * (nm.col_sums(ext) - 1.0)
        acc = nm.row_sums(nm.val * ext)
        y += sigma * ((2.0 * t - t_prev) - acc)
        x_prev[:] = x
        t_prev[:] = t
        d = tau * y - t_prev
        root = np.sqrt(d * d + 4.0 * tau * nm.w)
        with np.errstate(divide="ignore", invalid="ignore"):
            conj = 2.0 * tau * nm.w / (d + root)
        t[:] = np.where(d > 0.0, conj, 0.5 * (root - d))
        xv = x_prev - tau * (p[nm.col] - nm.val * y[nm.row_ids])
        x[:] = np.where(xv > 0.0, xv, 0.0)
        count += 1
        wold = (count - 1.0) / count
        wnew = 1.0 / count
        xbar[:] = wold * xbar + wnew * x
        tbar[:] = wold * tbar + wnew * t
        ybar[:] = wold * ybar + wnew * y
        pbar[:] = wold * pbar + wnew * p
    return count


def lifted_op_norm(nm, iters=50):
    """pdhg.py:144-166: power iteration on (x, t) -> (colsum x, t - u.x)."""
    nnz, n = nm.nnz, nm.n
    v = np.full(nnz + n, 1.0 / np.sqrt(nnz + n))
    sig = 0.0
    for _ in range(iters):
        vx, vt = v[:nnz], v[nnz:]
        out_p = nm.col_sums(vx)
        out_y = vt - nm.row_sums(nm.val * vx)
        back_x = out_p[nm.col] - nm.val * out_y[nm.row_ids]
        wv = np.concatenate([back_x, out_y])
        sig = np.linalg.norm(wv)
        if sig == 0.0:
            return 0.0
        v = wv / sig
    return float(np.sqrt(sig))


def solve_lifted(mk, tol=1e-4, max_iters=100_000, check_every=40, step_mode="adaptive",
                 adapt_eta=True, restart="adaptive", restart_k=0, beta=(0.2, 0.8, 0.2)):
    """Restarted lifted PDHG (driver.py:184-268 _LiftedRun inside the loop of
    driver.py:271-377, algo="pdhg"); returns a dict with the SolveReport
    fields (plus "objective")."""
    bad = validate(mk)
    if bad:
        raise ValueError("; ".join(bad))
    nm, scales = normalize(mk)
    counts = np.bincount(nm.col, minlength=nm.m)
    x = 1.0 / counts[nm.col].astype(np.float64)          # pdhg.py:60-68
    t = nm.row_sums(nm.val * x)
    p = np.full(nm.m, float(np.sum(nm.w)) / nm.m)
    y = nm.w / t
    x_prev, t_prev = x.copy(), t.copy()
    xbar, tbar, pbar, ybar = x.copy(), t.copy(), p.copy(), y.copy()
    navg = 0
    L = max(lifted_op_norm(nm), np.finfo(float).tiny)

    if step_mode == "theory":
        steps = None
        tau = sigma = 1.0 / (2.0 * L)
    else:
        primal = np.linalg.norm(np.concatenate([nm.col_sums(x) - 1.0,
                                                t - nm.row_sums(nm.val * x)]))
        uy = nm.val * y[nm.row_ids]
        best = np.full(nm.m, -np.inf)
        np.maximum.at(best, nm.col, uy)
        dual = np.linalg.norm(np.concatenate([nm.w / t - y, np.minimum(p - best, 0.0)]))
        primal, dual = float(primal), float(dual)
        omega0 = max(1.0, dual / primal) if (primal > 1e-8 and dual > 1e-8) else 1.0
        steps = Steps(0.9 / L, omega0, 0.95 / L, omega0 / OMEGA_BOUND_FACTOR,
                      omega0 * OMEGA_BOUND_FACTOR)
        tau, sigma = steps.tau, steps.sigma

    def res(xx, tt, pp, yy):
        return residuals_lifted(mk, xx, tt * scales, pp, yy / scales)

    res_avg = res(xbar, tbar, pbar, ybar)
    at_restart = prev_check = res_avg[3]
    snap = (x.copy(), t.copy(), p.copy(), y.copy())
    history = []
    total = restarts = 0
    t0 = time.perf_counter()
    while True:
        chunk = min(check_every, max_iters - total)
        if restart == "fixed":
            chunk = min(chunk, restart_k - navg)
        navg = pdhg_chunk(nm, x, x_prev, t, t_prev, p, y, xbar, tbar, pbar, ybar, navg,
                          tau, sigma, chunk)
        total += chunk
        res_last = res(x, t, p, y)
        res_avg = res(xbar, tbar, pbar, ybar)
        metric = min(res_last[3], res_avg[3])
        history.append((total, metric))
        if metric <= tol or total >= max_iters:
            if res_avg[3] < res_last[3]:
                x, t, p, y = xbar.copy(), tbar.copy(), pbar.copy(), ybar.copy()
                final = res_avg
            else:
                final = res_last
            status = "optimal" if metric <= tol else "max-iters"
            break
        if restart == "fixed":
            do_restart = navg >= restart_k
        else:
            do_restart = should_restart(res_avg[3], at_restart, prev_check, navg, total, beta)
        prev_check = res_avg[3]
        if do_restart:
            if steps is not None:
                dx, dt = xbar - snap[0], tbar - snap[1]
                dp, dy = pbar - snap[2], ybar - snap[3]
                k_dx_p = float(np.dot(nm.col_sums(dx), dp))
                k_dt_y = float(np.dot(dt - nm.row_sums(nm.val * dx), dy))
                psq = float(np.dot(dx, dx) + np.dot(dt, dt))
                dsq = float(np.dot(dp, dp) + np.dot(dy, dy))
                inter = abs(k_dx_p + k_dt_y)
                eta_obs = None
                if adapt_eta and inter > 0.0:
                    eta_obs = (steps.omega * psq + dsq / steps.omega) / (2.0 * inter)
                steps.update(float(np.sqrt(psq)), float(np.sqrt(dsq)), eta_obs)
                tau, sigma = steps.tau, steps.sigma
            x[:], t[:], p[:], y[:] = xbar, tbar, pbar, ybar
            x_prev[:] = x
            t_prev[:] = t
            navg = 0
            restarts += 1
            snap = (x.copy(), t.copy(), p.copy(), y.copy())
            at_restart = prev_check = res_avg[3]
    wall = time.perf_counter() - t0
    return {
        "status": status, "inner_iterations": total, "restarts": restarts,
        "wall_time_seconds": wall, "final_residuals": final,
        "residual_history": history, "prices": p.copy(), "allocation": x.copy(),
        "utility_values": t * scales, "dual_values": y / scales,
        "objective": eg_objective(mk, x), "op_norm": L, "tau_sigma": (tau, sigma),
    }


# ---------------------------------------------------------- Arrow-Debreu loop

def apply_T(U, E, w, tol=1e-6, warm_start=None, **kw):
    """w -> E p(w) / sum (exchange.py:75-93); returns (w_next, report)."""
    w = np.asarray(w, dtype=np.float64)
    if np.any(w <= 0):
        raise ValueError("budgets must be strictly positive")
    rep = solve(U.with_values(U.val, w), tol=tol, warm_start=warm_start, **kw)
    w_next = E.apply(rep["prices"])
    total = float(np.sum(w_next))
    if total <= 0:
        raise ValueError("endowment application produced no budget mass")
    return w_next / total, rep


def inner_tolerance(prev_gap, outer_tol):
    """exchange.py:96-101."""
    if prev_gap < 10.0 * outer_tol:
        return outer_tol / 10.0
    return max(outer_tol / 10.0, min(1e-5, prev_gap / 20.0))


def solve_exchange(U, E, outer_tol=1e-6, max_outer=100, **kw):
    """Fixed-point iteration on budgets (exchange.py:104-156); U carries any w."""
    n = U.n
    w = np.full(n, 1.0 / n)
    warm = None
    prev_gap = np.inf
    rises = 0
    gaps, inner_iters = [], []
    status = "max-outer"
    prices = None
    for k in range(max_outer):
        tol_k = inner_tolerance(prev_gap, outer_tol)
        w_next, rep = apply_T(U, E, w, tol=tol_k, warm_start=warm, **kw)
        warm = {"x": rep["allocation"], "p": rep["prices"]}
        gap = float(np.linalg.norm(w_next - w))
        gaps.append(gap)
        inner_iters.append(rep["inner_iterations"])
        prices = rep["prices"]
        if abs(float(np.sum(w_next)) - 1.0) > 1e-8:
            raise AssertionError("budget mass drifted")
        if rep["status"] != "optimal":
            status = "inner-failure"
            w = w_next
            break
        w = w_next
        if gap <= outer_tol:
            status = "converged"
            break
        if gap > prev_gap:
            rises += 1
            if rises >= 5:
                status = "diverging"
                break
        else:
            rises = 0
        prev_gap = gap
    return {"status": status, "outer_iterations": len(gaps), "budget_gaps": gaps,
            "final_budgets": w, "final_prices": prices, "inner_iterations": inner_iters}
