"""Restarted lifted PDHG on the device (algo="pdhg").

The reference's second solver (`market_eq/kernels.py:146-197` pdhg_chunk,
`market_eq/driver.py:184-268` _LiftedRun, `market_eq/pdhg.py:60-166`) on the
same DeviceMarket as the PDHCG path: state x (nnz), t, y (n), p (m) and
their running averages live on the device; one iteration is one
`mq_pdhg_step` (price step, per-buyer y/t/x updates, fixed-point column
sums); chunks are CUDA-graph captured; residuals, omega_0 norms, restart
moves and the lifted operator norm are device reductions.  The engine
exposes the interface `driver.solve_on_device` drives, so the restarted loop
is shared with PDHCG.
"""

import math

import numpy as np
import torch

from . import _native as nat
from .engine import _cur_stream, to_host
from .kkt import Residuals


class LiftedEngine:
    def __init__(self, dm, use_graphs=True, group=None):
        self.dm = dm
        self.lib = dm.lib
        if self.lib.mq_fixed_colsum() != 1:
            raise RuntimeError("lifted PDHG needs the fixed-point column-sum build")
        self.group = group
        self.world = 1
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
        self.use_graphs = bool(use_graphs) and self.world == 1
        dev = dm.device
        f64 = dict(dtype=torch.float64, device=dev)
        nnz, n, m = dm.nnz, dm.n, dm.m
        self.x, self.xbar, self.x0 = (torch.zeros(nnz, **f64) for _ in range(3))
        (self.t, self.t_prev, self.tbar, self.t0, self.y, self.ybar, self.y0, self.ru,
         self.ru_prev) = (torch.zeros(n, **f64) for _ in range(9))
        (self.p, self.pbar, self.p0, self.cs, self.cs_prev, self.csbar,
         self.cs0) = (torch.zeros(m, **f64) for _ in range(7))
        self.fix = torch.zeros(max(1, m), dtype=torch.int64, device=dev)
        self.colbest = torch.zeros(2, m, **f64)
        self.steps = torch.zeros(2, **f64)
        self.navg_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        self.faults = torch.zeros(1, dtype=torch.int64, device=dev)
        nscr = int(self.lib.mq_scratch_doubles())
        self.scratch = torch.zeros(nscr, **f64)
        self.out = torch.zeros(64, **f64)
        self.navg = 0
        self.tau = self.sigma = None
        self._graphs = {}
        if self.world > 1:
            from .device import fixed_point_scale

            gmax = int(self._global_counts().max().item()) if m else 1
            dm.struct.cs_scale, dm.struct.cs_xmax = fixed_point_scale(gmax)
        s = nat.MqLState()
        for k in ("x", "xbar", "t", "t_prev", "tbar", "y", "ybar", "ru", "ru_prev", "p", "pbar",
                  "cs", "cs_prev", "csbar", "fix", "steps", "faults"):
            setattr(s, k, getattr(self, k).data_ptr())
        s.navg = self.navg_dev.data_ptr()
        self.state = s

    # ------------------------------------------------------------ plumbing
    def _c(self, rc, what):
        return nat.check(rc, what)

    def _allreduce(self, t, op="sum"):
        if self.world > 1:
            import torch.distributed as dist

            red = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX}[op]
            dist.all_reduce(t, op=red, group=self.group)
        return t

    def _global_counts(self):
        return self._allreduce(self.dm.col_counts.clone())

    def colsum(self, v, out):
        self._c(self.lib.mq_colsum(self.dm.struct, nat.ptr(v), nat.ptr(out), _cur_stream()),
                "mq_colsum")
        return self._allreduce(out)

    def row_dot(self, x, out, use_norm=1):
        self._c(self.lib.mq_row_dot(self.dm.struct, nat.ptr(x), int(use_norm), nat.ptr(out),
                                    _cur_stream()), "mq_row_dot")
        return out

    # ------------------------------------------------------------ state
    def initial_state(self, w_sum=None):
        """pdhg.py:60-68: x = 1/colcount, t = u.x, p = sum(w)/m, y = w/t."""
        counts = self._global_counts()
        self.x.copy_(1.0 / counts.to(torch.float64)[self.dm.col.to(torch.int64)])
        self.row_dot(self.x, self.t)
        if w_sum is None:
            w_sum = float(self._allreduce(self.dm.w.sum().reshape(1)).item())
        self.p.fill_(w_sum / self.dm.m)
        torch.div(self.dm.w, self.t, out=self.y)
        self.t_prev.copy_(self.t)
        self.ru.copy_(self.t)  # u.x of x^k and of x_prev = x
        self.ru_prev.copy_(self.t)
        self.xbar.copy_(self.x)
        self.tbar.copy_(self.t)
        self.pbar.copy_(self.p)
        self.ybar.copy_(self.y)
        self.colsum(self.x, self.cs)
        self.cs_prev.copy_(self.cs)
        self.csbar.copy_(self.cs)
        self.navg = 0
        self.navg_dev.zero_()
        self.snapshot()

    def load_state(self, x, p):
        raise NotImplementedError("the lifted solver ignores warm starts (driver.py:271-276)")

    def set_steps(self, tau, sigma):
        if (tau, sigma) != (self.tau, self.sigma):
            self.tau, self.sigma = float(tau), float(sigma)
            self.steps.copy_(torch.tensor([self.tau, self.sigma], dtype=torch.float64))

    def snapshot(self):
        for a, b in ((self.x0, self.x), (self.t0, self.t), (self.p0, self.p), (self.y0, self.y),
                     (self.cs0, self.cs)):
            a.copy_(b)

    def restart(self):
        """driver.py:254-261: x, t, p, y <- averages, x_prev <- x, t_prev <- t."""
        self.x.copy_(self.xbar)
        self.t.copy_(self.tbar)
        self.p.copy_(self.pbar)
        self.y.copy_(self.ybar)
        self.t_prev.copy_(self.t)
        self.row_dot(self.x, self.ru)
        self.ru_prev.copy_(self.ru)
        self.cs.copy_(self.csbar)
        self.cs_prev.copy_(self.csbar)
        self.navg = 0
        self.navg_dev.zero_()

    def adopt_average(self):
        self.x.copy_(self.xbar)
        self.t.copy_(self.tbar)
        self.p.copy_(self.pbar)
        self.y.copy_(self.ybar)
        self.cs.copy_(self.csbar)

    # ------------------------------------------------------------ chunks
    def run_chunk(self, iters):
        """`iters` lifted iterations (kernels.py:146-197); returns [] (the
        lifted solver reports no sub-problem passes)."""
        if iters <= 0:
            return []
        self.faults.zero_()
        if self.use_graphs:
            g = self._graphs.get(iters)
            if g is None:
                g = self._capture(iters)
            g.replay()
        else:
            self._launch_chunk(iters)
        if int(self.faults.item()):
            raise RuntimeError("allocation entries beyond the fixed-point column-sum range")
        self.navg += iters
        return []

    def _launch_chunk(self, iters):
        lib, mk, st = self.lib, self.dm.struct, self.state
        for it in range(iters):
            if self.world > 1:
                self._c(lib.mq_pdhg_colsum_only(mk, st, it, _cur_stream()), "mq_pdhg_step")
                self._allreduce(self.fix)
                self._c(lib.mq_pdhg_finish_colsum(mk, st, it, _cur_stream()), "mq_pdhg_step")
            else:
                self._c(lib.mq_pdhg_step(mk, st, it, _cur_stream()), "mq_pdhg_step")
        self._c(lib.mq_pdhg_chunk_end(st, iters, _cur_stream()), "mq_pdhg_chunk_end")

    def _capture(self, iters):
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.dm.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=side):
            self._launch_chunk(iters)
        torch.cuda.current_stream().wait_stream(side)
        self._graphs[iters] = g
        return g

    # ------------------------------------------------------------ reductions
    def _rows(self, x, t, y, p, use_norm, k):
        o = self.out[16 * k: 16 * k + 10]
        self._c(self.lib.mq_pdhg_resid_rows(self.dm.struct, nat.ptr(self.dm.scales), nat.ptr(x),
                                            nat.ptr(t), nat.ptr(y), nat.ptr(p), int(use_norm),
                                            nat.ptr(self.colbest[k]), nat.ptr(o),
                                            nat.ptr(self.scratch), _cur_stream()),
                "mq_pdhg_resid_rows")
        if self.world > 1:
            self._allreduce(self.colbest[k], "max")
            mx = o[0:7].clone()
            self._allreduce(mx, "max")
            o[0:7].copy_(mx)
            sm = o[7:10].clone()
            self._allreduce(sm, "sum")
            o[7:10].copy_(sm)

    def _cols(self, cs, p, k):
        self._c(self.lib.mq_resid_cols(self.dm.m, nat.ptr(cs), nat.ptr(p),
                                       nat.ptr(self.colbest[k]),
                                       nat.ptr(self.out[16 * k + 10: 16 * k + 16]),
                                       nat.ptr(self.scratch), _cur_stream()), "mq_resid_cols")

    @staticmethod
    def _assemble(v):
        """residuals_lifted (kkt.py:29-76) from the row and column maxima."""
        row_gap, wtmax, ymax, dual_t, gap, xmax, emax, nbad = v[0:8]
        col_gap, csmax, dual_p, slmax = v[10:14]
        if nbad > 0:
            raise ValueError("residuals require strictly positive t")
        r_primal = max(col_gap, row_gap) / (1.0 + max(csmax, row_gap, 1.0))
        r_dual = max(dual_t, dual_p) / (1.0 + max(wtmax, ymax, slmax))
        r_gap = gap / (1.0 + max(xmax, emax))
        return Residuals(float(r_primal), float(r_dual), float(r_gap),
                         float(max(r_primal, r_dual, r_gap)))

    def residuals_pair(self):
        """(last, avg) residuals on the ORIGINAL instance (driver.py:230-236)."""
        self._rows(self.x, self.t, self.y, self.p, 0, 0)
        self._cols(self.cs, self.p, 0)
        self._rows(self.xbar, self.tbar, self.ybar, self.pbar, 0, 1)
        self._cols(self.csbar, self.pbar, 1)
        v = self.out[:32].cpu().numpy()
        return self._assemble(v[0:16]), self._assemble(v[16:32])

    def residuals_avg(self):
        self._rows(self.xbar, self.tbar, self.ybar, self.pbar, 0, 1)
        self._cols(self.csbar, self.pbar, 1)
        return self._assemble(self.out[16:32].cpu().numpy())

    def omega_norms(self):
        """driver.py:216-226: || [colsum x - 1, t - u.x] ||, || [w/t - y,
        min(p - colbest, 0)] || on the normalized instance."""
        self._rows(self.x, self.t, self.y, self.p, 1, 0)
        self._cols(self.cs, self.p, 0)
        v = self.out[0:16].cpu().numpy()
        return math.sqrt(v[8] + v[14]), math.sqrt(v[9] + v[15])

    def restart_moves(self):
        """driver.py:242-252 for the lifted state."""
        o = self.out[32:40]
        self._c(self.lib.mq_restart_moves(self.dm.struct, nat.ptr(self.xbar), nat.ptr(self.x0),
                                          nat.ptr(self.pbar), nat.ptr(self.p0),
                                          nat.ptr(self.csbar), nat.ptr(self.cs0), nat.ptr(o),
                                          nat.ptr(self.scratch), _cur_stream()),
                "mq_restart_moves")
        self._c(self.lib.mq_pdhg_moves(self.dm.struct, nat.ptr(self.xbar), nat.ptr(self.x0),
                                       nat.ptr(self.tbar), nat.ptr(self.t0), nat.ptr(self.ybar),
                                       nat.ptr(self.y0), nat.ptr(o[4:7]), nat.ptr(self.scratch),
                                       _cur_stream()), "mq_pdhg_moves")
        if self.world > 1:
            sx = torch.cat([o[0:1], o[4:7]])
            self._allreduce(sx, "sum")
            o[0:1].copy_(sx[0:1])
            o[4:7].copy_(sx[1:4])
        dxx, dpp, kxp, _, dtt, dyy, kty = (float(v) for v in o[0:7].cpu().numpy())
        psq, dsq = dxx + dtt, dpp + dyy
        return math.sqrt(psq), math.sqrt(dsq), psq, dsq, abs(kxp + kty)

    def op_norm(self, iters=50):
        """pdhg.py:144-166: power iteration on (x, t) -> (colsum x, t - u.x)."""
        dm = self.dm
        nnz, n = dm.nnz, dm.n
        total = int(self._allreduce(torch.tensor([nnz + n], dtype=torch.int64,
                                                 device=dm.device)).item())
        vx = torch.full((nnz,), 1.0 / math.sqrt(total), dtype=torch.float64, device=dm.device)
        vt = torch.full((n,), 1.0 / math.sqrt(total), dtype=torch.float64, device=dm.device)
        out_p = torch.zeros(dm.m, dtype=torch.float64, device=dm.device)
        out_y = torch.zeros(n, dtype=torch.float64, device=dm.device)
        wx = torch.zeros(nnz, dtype=torch.float64, device=dm.device)
        sums = self.out[48:50]
        sig = 0.0
        for _ in range(iters):
            self.colsum(vx, out_p)
            self._c(self.lib.mq_pdhg_opnorm_step(dm.struct, nat.ptr(vx), nat.ptr(vt),
                                                 nat.ptr(out_p), nat.ptr(out_y), nat.ptr(wx),
                                                 nat.ptr(sums), nat.ptr(self.scratch),
                                                 _cur_stream()), "mq_pdhg_opnorm_step")
            s2 = self._allreduce(sums.clone())
            sig = math.sqrt(float(s2.sum().item()))
            if sig == 0.0:
                return 0.0
            torch.div(wx, sig, out=vx)
            torch.div(out_y, sig, out=vt)
        return math.sqrt(sig)

    def final_payload(self, gather=False):
        """prices, allocation, t and y on the original instance, objective
        (gather=True on N ranks: the whole market's rows, in row order)."""
        ux = torch.zeros(self.dm.n, dtype=torch.float64, device=self.dm.device)
        self.row_dot(self.x, ux, use_norm=0)
        if bool((ux <= 0).any().item()):
            obj = math.inf
        else:
            part = -(self.dm.w * torch.log(ux)).sum().reshape(1)
            obj = float(self._allreduce(part).item())
        scales = self.dm.scales
        x, t, y = self.x, self.t * scales, self.y / scales
        if gather and self.world > 1:
            from .engine import gather_rows

            x, t, y = (gather_rows(v, self.group, self.world) for v in (x, t, y))
        return {"prices": self.p.cpu().numpy(), "allocation": to_host(x),
                "utility_values": t.cpu().numpy(), "dual_values": y.cpu().numpy(),
                "objective": obj}
