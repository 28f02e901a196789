"""CPU stand-in for the engine's device operations — TEST ONLY.

Lets tests drive the real PdhcgEngine orchestration (chunk loop, all-reduce
placement, distributed residual/restart reductions, driver loop) on CPU ranks
with the gloo backend.  Row solves use the oracle's k-section at subtol=0 (the
same root the CUDA exact solver computes, to ~1e-15).
"""

import types

import numpy as np
import torch

from oracle import solve as orc


class CpuMarket:
    """A row shard [row0, row0 + nrows) of a FisherInstance on the CPU."""

    def __init__(self, inst, row0=0, nrows=None):
        u = inst.utilities
        nrows = u.n_rows - row0 if nrows is None else nrows
        a, b = u.row_offsets[row0], u.row_offsets[row0 + nrows]
        rp = u.row_offsets[row0:row0 + nrows + 1] - a
        col = u.col_indices[a:b]
        val = u.values[a:b]
        w = inst.budgets[row0:row0 + nrows]
        mk = orc.Market(nrows, u.n_cols, rp, col, val, w)
        nm, scales = orc.normalize(mk)
        self.n, self.m, self.nnz = nrows, u.n_cols, int(b - a)
        self.row_begin = row0
        self.nblk = 0
        self.device = torch.device("cpu")
        self.row_ptr = torch.from_numpy(rp.astype(np.int64))
        self.col = torch.from_numpy(col.astype(np.int32))
        self.u = torch.from_numpy(nm.val.copy())
        self.u_orig = torch.from_numpy(val.astype(np.float64).copy())
        self.w = torch.from_numpy(w.astype(np.float64).copy())
        self.scales = torch.from_numpy(scales)
        self.col_counts = torch.bincount(self.col.to(torch.int64), minlength=self.m)
        self.row_ids = np.repeat(np.arange(nrows), np.diff(rp))


class OracleOps:
    supports_graphs = False

    def __init__(self, dm, engine):
        self.dm, self.e = dm, engine

    def _avg(self, it):
        count = int(self.e.navg_dev.item()) + it + 1
        return (count - 1.0) / count, 1.0 / count

    def colsum(self, v, out):
        out.copy_(torch.from_numpy(np.bincount(self.dm.col.numpy(), weights=v.numpy(),
                                               minlength=self.dm.m)))

    def dual(self, it):
        e = self.e
        wold, wnew = self._avg(it)
        sigma = float(e.steps[1])
        acc = 2.0 * e.cs - e.cs_prev
        e.p += sigma * (acc - 1.0)
        e.pbar.copy_(wold * e.pbar + wnew * e.p)
        e.cs_prev.copy_(e.cs)

    def primal(self, it, rebuild=False):
        e, dm = self.e, self.dm
        wold, wnew = self._avg(it)
        tau = float(e.steps[0])
        rp, col = dm.row_ptr.numpy(), dm.col.numpy()
        u, w, p = dm.u.numpy(), dm.w.numpy(), e.p.numpy()
        x, xb = e.x.numpy(), e.xbar.numpy()
        passes = 0
        for i in range(dm.n):
            a, b = rp[i], rp[i + 1]
            if b == a:
                continue
            c = x[a:b] - tau * p[col[a:b]]
            s0 = float(np.dot(u[a:b], x[a:b]))
            s, np_ = orc.row_root(u[a:b], c, tau * w[i], s0, 32, 0.0)
            passes += max(np_, 0)
            xn = np.maximum(c + (tau * w[i] * u[a:b]) / s, 0.0)
            x[a:b] = xn
            xb[a:b] = wold * xb[a:b] + wnew * xn
        e.pass_buf[it] += passes
        self.colsum(e.x, e.cs)  # the fused kernel's tile column sums

    def colsum_rest(self, it, finalize):
        if finalize:
            self.finalize(it)

    def finalize(self, it):
        wold, wnew = self._avg(it)
        self.e.csbar.copy_(wold * self.e.csbar + wnew * self.e.cs)

    def chunk_end(self, iters):
        self.e.navg_dev += iters

    def resid_rows(self, x, p, use_norm, colbest, t_out, out, scratch):
        dm = self.dm
        U = (dm.u if use_norm else dm.u_orig).numpy()
        xv, pv, col = x.numpy(), p.numpy(), dm.col.numpy()
        t = np.bincount(dm.row_ids, weights=U * xv, minlength=dm.n)
        bad = np.flatnonzero(~(t > 0))
        with np.errstate(divide="ignore"):
            y = np.where(t > 0, dm.w.numpy() / np.where(t > 0, t, 1.0), 0.0)
        uy = U * y[dm.row_ids]
        best = np.zeros(dm.m)
        np.maximum.at(best, col, uy)
        colbest.copy_(torch.maximum(colbest, torch.from_numpy(best)))
        es = np.maximum(pv[col] - uy, 0.0)
        good = t > 0
        ge = good[dm.row_ids]
        vals = [np.max(y, initial=0.0), np.max((xv * es)[ge], initial=0.0),
                np.max(np.abs(xv)[ge], initial=0.0), np.max(es[ge], initial=0.0),
                float(bad[0] + dm.row_begin) if len(bad) else -1.0,
                float(np.sum(dm.w.numpy()[good] * np.log(t[good]))), float(len(bad)), 0.0]
        out.copy_(torch.tensor(vals, dtype=torch.float64))
        if t_out is not None:
            t_out.copy_(torch.from_numpy(t))

    def resid_cols(self, cs, p, colbest, out, scratch):
        c, sl = cs.numpy(), p.numpy() - colbest.numpy()
        vals = [np.max(np.abs(c - 1.0), initial=0.0), np.max(np.abs(c), initial=0.0),
                np.max(np.maximum(-sl, 0.0), initial=0.0), np.max(sl, initial=0.0),
                float(np.sum((c - 1.0) ** 2)), float(np.sum(np.minimum(sl, 0.0) ** 2))]
        out.copy_(torch.tensor(vals, dtype=torch.float64))

    def restart_moves(self, xbar, x0, pbar, p0, csbar, cs0, out, scratch):
        dx, dp = (xbar - x0).numpy(), (pbar - p0).numpy()
        vals = [float(np.dot(dx, dx)), float(np.dot(dp, dp)),
                float(np.dot((csbar - cs0).numpy(), dp)), 0.0]
        out.copy_(torch.tensor(vals, dtype=torch.float64))


def cpu_session(dm, group=None):
    """A driver DeviceSession equivalent built on a CpuMarket."""
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.sparse import selector_norm_from_counts

    eng = PdhcgEngine(dm, group=group, ops_factory=OracleOps)
    return types.SimpleNamespace(dm=dm, engine=eng, op_norm=selector_norm_from_counts(
        eng._global_counts().numpy()))
