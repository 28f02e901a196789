"""PDHCG iterate on the device: chunks, residuals, restarts.

`PdhcgEngine` owns the iterate of driver._CompactRun (driver.py:91-181) as
torch buffers and runs everything through the native library:

* row_solver="exact" (default): one iteration = mq_dual_step +
  mq_primal_step + mq_colsum_step, all scalars device-resident, a chunk of
  `iters` iterations captured once per length as a CUDA graph and replayed;
  on N GPUs the column sums are all-reduced between colsum and the next price
  step (NCCL over NVLink), everything else stays rank-local.
* row_solver="ksection": the bit-faithful drop-in mq_pdhcg_chunk (literal
  k-section search, serial reference sums), single GPU.

Residuals (kkt.py:29-87), the omega_0 norms (driver.py:123-132) and restart
moves (driver.py:156-162) are device reductions that hand back a handful of
scalars per check.
"""

import math
import os
import weakref

import numpy as np
import torch

from . import _native as nat
from .errors import FixedPointRangeError, SubproblemError
from .kkt import Residuals

MAX_ROW_PASSES = 200  # kernels.py:16 (k-section fault threshold)


def _cur_stream():
    import ctypes

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_STAGE_ELEMS = 1 << 24  # 128 MB of float64 per pinned staging buffer


def to_host(t):
    """Device tensor -> numpy, through two pinned staging buffers: the D2H
    copy of one chunk overlaps the host copy of the previous one (a plain
    .cpu() of 8 GB goes through pageable memory at a few GB/s)."""
    n = t.numel()
    if n * t.element_size() <= (64 << 20):
        return t.cpu().numpy()
    t = t.reshape(-1)
    out = np.empty(n, dtype=torch.empty(0, dtype=t.dtype).numpy().dtype)
    stage = [torch.empty(_STAGE_ELEMS, dtype=t.dtype, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    prev = None
    for i, off in enumerate(range(0, n, _STAGE_ELEMS)):
        c = min(_STAGE_ELEMS, n - off)
        buf = stage[i & 1]
        buf[:c].copy_(t[off:off + c], non_blocking=True)
        evs[i & 1].record()
        if prev is not None:
            poff, pc, pi = prev
            evs[pi & 1].synchronize()
            _pcopy(out[poff:poff + pc], stage[pi & 1][:pc].numpy())
        prev = (off, c, i)
    poff, pc, pi = prev
    evs[pi & 1].synchronize()
    _pcopy(out[poff:poff + pc], stage[pi & 1][:pc].numpy())
    return out


def to_device(a, device):
    """numpy -> device tensor (same dtype) through two pinned staging buffers,
    the host copy of one chunk overlapping the H2D copy of the previous."""
    a = np.ascontiguousarray(a).reshape(-1)
    if a.nbytes <= (64 << 20):
        return torch.from_numpy(a if a.flags.writeable else a.copy()).to(device)
    out = torch.empty(a.shape[0], dtype=torch.from_numpy(a[:0].copy()).dtype, device=device)
    stage = [torch.empty(_STAGE_ELEMS * 8 // a.itemsize, dtype=out.dtype, pin_memory=True)
             for _ in range(2)]
    ce = stage[0].numel()
    evs = [None, None]
    with torch.cuda.device(out.device):
        for i, off in enumerate(range(0, a.shape[0], ce)):
            c = min(ce, a.shape[0] - off)
            b = i & 1
            if evs[b] is not None:
                evs[b].synchronize()  # its previous H2D copy has finished
            _pcopy(stage[b].numpy()[:c], a[off:off + c])
            out[off:off + c].copy_(stage[b][:c], non_blocking=True)
            evs[b] = torch.cuda.Event()
            evs[b].record()
        torch.cuda.current_stream().synchronize()
    return out


_POOL = None


def gather_rows(t, group, world):
    """Concatenation of every rank's `t` in rank order (all-gather of
    variable-length row shards, padded to the longest)."""
    import torch.distributed as dist

    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(v.item()) for v in sizes]
    buf = torch.zeros(max(sizes), dtype=t.dtype, device=t.device)
    buf[:t.numel()] = t
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:k] for p, k in zip(parts, sizes)])


def _pcopy(dst, src, piece=1 << 21):
    """np.copyto over threads (numpy drops the GIL; first-touch page faults
    of a fresh output array dominate a single-threaded copy)."""
    global _POOL
    if _POOL is None:
        import concurrent.futures
        import os

        _POOL = concurrent.futures.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1))
    n = dst.shape[0]
    list(_POOL.map(lambda o: np.copyto(dst[o:o + piece], src[o:o + piece]), range(0, n, piece)))


class NativeOps:
    """The engine's device operations, each one call into libmarket_eq_b200.so
    on the current CUDA stream (include/market_eq_b200.h)."""

    supports_graphs = True

    def __init__(self, dm, engine):
        # a weak reference: no engine <-> ops cycle, so a dropped engine frees
        # its device memory at once (config 4 holds tens of GB)
        self.lib, self.dm, self.eng = dm.lib, dm, weakref.proxy(engine)

    def _c(self, rc, what):
        return nat.check(rc, what)

    def colsum(self, v, out):
        self._c(self.lib.mq_colsum(self.dm.struct, nat.ptr(v), nat.ptr(out), _cur_stream()),
                "mq_colsum")

    def dual(self, it):
        self._c(self.lib.mq_dual_step(self.dm.struct, self.eng.state, it, _cur_stream()),
                "mq_dual_step")

    def primal(self, it, rebuild=False):
        st = self.eng.state_rebuild if rebuild else self.eng.state
        self._c(self.lib.mq_primal_step(self.dm.struct, st, it, None, _cur_stream()),
                "mq_primal_step")

    def colsum_rest(self, it, finalize):
        self._c(self.lib.mq_colsum_step(self.dm.struct, self.eng.state, it, int(finalize),
                                        _cur_stream()), "mq_colsum_step")

    def finalize(self, it):
        self._c(self.lib.mq_colsum_finalize(self.dm.struct, self.eng.state, it, _cur_stream()),
                "mq_colsum_finalize")

    def chunk_end(self, iters):
        self._c(self.lib.mq_chunk_end(self.eng.state, iters, _cur_stream()), "mq_chunk_end")
        if self.eng.sparse:  # x from the slots; xbar is formed on demand (PdhcgEngine.xbar)
            self._c(self.lib.mq_ws_flush(self.dm.struct, self.eng.state, _cur_stream()),
                    "mq_ws_flush")

    def avg_xbar(self):
        self._c(self.lib.mq_avg_xbar(self.dm.struct, self.eng.state, _cur_stream()),
                "mq_avg_xbar")

    def resid_rows(self, x, p, use_norm, colbest, t_out, out, scratch):
        work = self.eng.resid_work
        self._c(self.lib.mq_resid_rows(self.dm.struct, nat.ptr(x), nat.ptr(p), int(use_norm),
                                       nat.ptr(colbest), nat.ptr(work), nat.ptr(t_out), None,
                                       nat.ptr(out), nat.ptr(scratch), _cur_stream()),
                "mq_resid_rows")

    def resid_pair(self, cb_last, cb_avg, out_last, out_avg):
        e = self.eng
        self._c(self.lib.mq_resid_rows_pair(self.dm.struct, e.state, nat.ptr(cb_last),
                                            nat.ptr(cb_avg), nat.ptr(e.resid_work),
                                            nat.ptr(out_last), nat.ptr(out_avg),
                                            nat.ptr(e.scratch), nat.ptr(e.scratch2),
                                            _cur_stream()), "mq_resid_rows_pair")

    def resid_cols(self, cs, p, colbest, out, scratch):
        self._c(self.lib.mq_resid_cols(self.dm.m, nat.ptr(cs), nat.ptr(p), nat.ptr(colbest),
                                       nat.ptr(out), nat.ptr(scratch), _cur_stream()),
                "mq_resid_cols")

    def restart_moves(self, xbar, x0, pbar, p0, csbar, cs0, out, scratch):
        self._c(self.lib.mq_restart_moves(self.dm.struct, nat.ptr(xbar), nat.ptr(x0),
                                          nat.ptr(pbar), nat.ptr(p0), nat.ptr(csbar),
                                          nat.ptr(cs0), nat.ptr(out), nat.ptr(scratch),
                                          _cur_stream()), "mq_restart_moves")

    def ksection_chunk(self, iters):
        """mq_pdhcg_chunk on the engine's buffers -> (faults, navg)."""
        import ctypes

        e, dm = self.eng, self.dm
        tperm, tptr = dm.global_schedule()
        navg_out = ctypes.c_int64(0)
        rc = self.lib.mq_pdhcg_chunk(
            dm.n, dm.m, nat.ptr(dm.row_ptr), nat.ptr(dm.col), nat.ptr(dm.u), nat.ptr(tperm),
            nat.ptr(tptr), nat.ptr(dm.w), nat.ptr(e.x), nat.ptr(e.x_prev), nat.ptr(e.p),
            nat.ptr(e.xbar), nat.ptr(e.pbar), e.navg, e.tau, e.sigma, e.sections, e.subtol,
            iters, nat.ptr(e.c_buf), nat.ptr(e.pass_buf), ctypes.byref(navg_out), _cur_stream())
        self._c(rc, "mq_pdhcg_chunk")
        return rc, int(navg_out.value)


class PdhcgEngine:
    def __init__(self, dm, row_solver="exact", sections=32, subproblem_tol=1e-10,
                 use_graphs=True, group=None, ops_factory=None, working_set=True,
                 force_collectives=False, colsum_fp64=False):
        if row_solver not in ("exact", "ksection"):
            raise ValueError("row_solver must be 'exact' or 'ksection'")
        self.dm = dm
        self.mode = row_solver
        # validation mode: the price step's column sums recomputed in fp64 in
        # the reference's ascending-row order (mq_colsum) instead of the
        # fixed-point atomics (tests/test_gpu_baseline_markets.py)
        self.colsum_fp64 = bool(colsum_fp64)
        self.sections = int(sections)
        self.subtol = float(subproblem_tol)
        self.group = group
        self.world = 1
        backend = None
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
            backend = dist.get_backend(group)
        # the N-rank step (collectives between the kernels); force_collectives
        # runs it on one rank too (tests of the captured collectives on 1 GPU)
        self.distributed = self.world > 1 or (bool(force_collectives) and group is not None)
        if self.mode == "ksection" and self.distributed:
            raise ValueError("the k-section drop-in runs on a single GPU")
        self.ops = (ops_factory or NativeOps)(dm, self)
        # N ranks: the chunk graph captures the NCCL all-reduces with the
        # kernels (gloo collectives are host-side and cannot be captured)
        self.use_graphs = (bool(use_graphs) and getattr(self.ops, "supports_graphs", False)
                           and (not self.distributed or backend == "nccl")
                           and os.environ.get("MQ_GRAPH_COLLECTIVES", "1") != "0")
        dev = dm.device
        f64 = dict(dtype=torch.float64, device=dev)
        nnz, m = dm.nnz, dm.m
        # x / xbar are read by TMA bulk copies: nat.PAD readable elements past nnz
        self._x_buf = torch.zeros(nnz + nat.PAD, **f64)
        self._xbar_buf = torch.zeros(nnz + nat.PAD, **f64)
        self.x = self._x_buf[:nnz]
        self._xbar_t = self._xbar_buf[:nnz]
        self._xbar_stale = False  # sparse iterate: xbar not yet formed from xsum
        self.x0 = torch.zeros(nnz, **f64)
        # sparse iterate: x > 0 flags and the running sum of x
        self.sparse = bool(hasattr(dm, "lib") and dm.lib.mq_x_sparse() == 1
                           and self.mode != "ksection")
        self._xflag_buf = torch.ones(nnz + nat.PAD if self.sparse else 16, dtype=torch.uint8,
                                     device=dev)
        self.xflag = self._xflag_buf
        self.xsum = torch.zeros(nnz if self.sparse else 1, **f64)
        # per-buyer utility of the last prox: the fused row solve's warm start
        self._srow_buf = torch.zeros(dm.n + nat.PAD, **f64)
        self.srow = self._srow_buf[:dm.n]
        # the primal kernels' dynamic work counters (tiles, long rows, medium
        # rows, full-solve list length and claims)
        self.blk_done = torch.zeros(8, dtype=torch.int32, device=dev)
        # working sets of the screened row solve: -3 marks the
        # rows the medium / long kernels solve, -1 "no working set yet"
        # (the fp64 validation mode sums x itself mid-chunk: no slot-resident x)
        self.working_set = bool(working_set and self.sparse and hasattr(dm, "lib")
                                and not colsum_fp64)
        if self.working_set:
            K = int(dm.lib.mq_ws_slots())  # nat.WS_SLOTS in the shipped build
            lens = dm.row_ptr[1:] - dm.row_ptr[:-1]
            self.ws_init = torch.where(lens > nat.WS_MAX_ROW, -3, -1).to(torch.int32)
            if dm.long_rows.numel():
                self.ws_init[dm.long_rows.to(torch.int64)] = -3
            npad = -(-max(1, dm.n) // 32) * 32
            # per row (h, theta, P, C): h in ws_len (a view), the rest float bits
            self.ws_hdr = torch.zeros(npad, 4, dtype=torch.int32, device=dev)
            self.ws_hdr[:, 0] = -3
            self.ws_len = self.ws_hdr[:dm.n, 0]
            self.ws_len.copy_(self.ws_init)
            self.ws_kmax = torch.zeros(npad // 32, dtype=torch.int32, device=dev)
            ns = npad * K  # slot k of row i: ((i/32)K + k)32 + i%32
            self.ws_u = torch.zeros(ns, **f64)
            self.ws_x = torch.zeros(ns, **f64)
            self.ws_col = torch.zeros(ns, dtype=torch.int32, device=dev)
            self.ws_pos = torch.zeros(ns, dtype=torch.uint8, device=dev)
            self.ws_list = torch.zeros(max(1, dm.n), dtype=torch.int32, device=dev)
            # long rows (> 1024 entries): one working-set pool of LONG_CAP
            # entries per row, in dm.long_rows order
            nl = int(dm.long_rows.numel())
            self.pool = nl > 0
            if self.pool:
                C = nat.LONG_CAP
                self.pl_hdr = torch.zeros(nl, 4, dtype=torch.int32, device=dev)
                self.pl_hdr[:, 0] = -1
                self.pl_u = torch.zeros(nl * C, **f64)
                self.pl_x = torch.zeros(nl * C, **f64)
                self.pl_col = torch.zeros(nl * C, dtype=torch.int32, device=dev)
                self.pl_pos = torch.zeros(nl * C, dtype=torch.int32, device=dev)
                self.pl_list = torch.zeros(nl, dtype=torch.int32, device=dev)
            # medium rows longer than WS_MAX_ROW (the leading nmed_long of
            # dm.med_rows): a pool of MED_CAP entries each
            nml = int(dm.struct.nmed_long) if dm.struct.nmed else 0
            self.mpool = nml > 0
            if self.mpool:
                C = nat.MED_CAP
                self.pm_hdr = torch.zeros(nml, 4, dtype=torch.int32, device=dev)
                self.pm_hdr[:, 0] = -1
                self.pm_u = torch.zeros(nml * C, **f64)
                self.pm_x = torch.zeros(nml * C, **f64)
                self.pm_col = torch.zeros(nml * C, dtype=torch.int32, device=dev)
                self.pm_pos = torch.zeros(nml * C, dtype=torch.int32, device=dev)
            self.drift = torch.zeros(2, **f64)
            # per-row working-set width level (kept across invalidations)
            self.ws_lvl = torch.zeros(max(1, dm.n), dtype=torch.uint8, device=dev)
        # fixed-point column sums: m u64 accumulators, zero between iterations
        fixed = getattr(getattr(dm, "lib", None), "mq_fixed_colsum", None)
        self.fixed = bool(fixed is not None and fixed() == 1 and self.mode != "ksection")
        self.bucket = torch.zeros(max(1, m if self.fixed else 1), **f64)
        self.p = torch.zeros(m, **f64)
        self.pbar = torch.zeros(m, **f64)
        self.p0 = torch.zeros(m, **f64)
        self.cs = torch.zeros(m, **f64)
        self.cs_prev = torch.zeros(m, **f64)
        self.csbar = torch.zeros(m, **f64)
        self.cs0 = torch.zeros(m, **f64)
        self.colbest = torch.zeros(2, m, **f64)
        # (p, column max[, pbar, column max]) interleaved per good
        self.resid_work = torch.zeros(4 * max(1, m), **f64)
        self.steps = torch.zeros(2, **f64)
        self.navg_dev = torch.zeros(1, dtype=torch.int64, device=dev)
        # [0] rows whose solve did not settle, [1] entries beyond the
        # fixed-point column-sum range
        self.faults = torch.zeros(2, dtype=torch.int64, device=dev)
        self.pass_buf = torch.zeros(1024, dtype=torch.int64, device=dev)
        nscr = int(dm.lib.mq_scratch_doubles()) if hasattr(dm, "lib") else 16
        self.scratch = torch.zeros(nscr, **f64)
        self.scratch2 = torch.zeros(nscr, **f64)
        self.out = torch.zeros(32, **f64)
        self.t_buf = torch.zeros(dm.n, **f64)
        if self.mode == "ksection":
            self.x_prev = torch.zeros(nnz, **f64)
            self.c_buf = torch.zeros(nnz, **f64)
        self.navg = 0
        self.tau = self.sigma = None
        self._graphs = {}
        if self.fixed and self.distributed:
            # one fixed-point scale on every rank (from the global column
            # counts), so the ranks' integer column sums add exactly: the
            # all-reduce runs on the u64 accumulators and the N-rank column
            # sums are bitwise the 1-rank ones
            from .device import fixed_point_scale

            gmax = int(self._global_counts().max().item()) if m else 1
            dm.struct.cs_scale, dm.struct.cs_xmax = fixed_point_scale(gmax)
        self.state = self._make_state()
        # the same state with ws_rebuild set: the tile kernel rebuilds every
        # working set (first iteration after the host wrote x or p)
        self.state_rebuild = None
        if self.state is not None and self.working_set:
            self.state_rebuild = self._make_state()
            self.state_rebuild.ws_rebuild = 1
        self._rebuild = True

    # ------------------------------------------------------------ plumbing
    def _make_state(self):
        if not isinstance(self.ops, NativeOps):
            return None
        s = nat.MqState()
        for name in ("x", "xbar", "p", "pbar", "cs", "cs_prev", "csbar", "blk_done",
                     "steps", "faults", "srow", "bucket", "xflag", "xsum"):
            setattr(s, name, getattr(self, name).data_ptr())
        if self.working_set:
            for name in ("ws_hdr", "ws_kmax", "ws_u", "ws_x", "ws_col", "ws_pos", "ws_list",
                         "drift", "ws_lvl"):
                setattr(s, name, getattr(self, name).data_ptr())
            if self.pool:
                for name in ("pl_hdr", "pl_u", "pl_x", "pl_col", "pl_pos", "pl_list"):
                    setattr(s, name, getattr(self, name).data_ptr())
            if self.mpool:
                for name in ("pm_hdr", "pm_u", "pm_x", "pm_col", "pm_pos"):
                    setattr(s, name, getattr(self, name).data_ptr())
        s.navg = self.navg_dev.data_ptr()
        s.pass_out = self.pass_buf.data_ptr()
        return s

    def _allreduce(self, t, op="sum"):
        if self.distributed:
            import torch.distributed as dist

            red = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX,
                   "min": dist.ReduceOp.MIN}[op]
            dist.all_reduce(t, op=red, group=self.group)
        return t

    def colsum(self, v, out):
        self.ops.colsum(v, out)
        return self._allreduce(out)

    # ------------------------------------------------------------ state
    def _sparse_sync(self):
        """After the host wrote x, xbar or navg: every x may be nonzero, the
        running sum restarts from navg * xbar and no working set is valid."""
        if self.working_set:
            self.ws_len.copy_(self.ws_init)
            self.ws_kmax.zero_()
            if self.pool:
                self.pl_hdr[:, 0] = -1
            if self.mpool:
                self.pm_hdr[:, 0] = -1
            self._rebuild = True
        if self.sparse:
            self.xflag.fill_(1)
            if self.navg:
                torch.mul(self.xbar, float(self.navg), out=self.xsum)
            else:
                self.xsum.zero_()

    def load_state(self, x, p):
        """Start (or warm start) from allocation x and prices p."""
        self.x.copy_(torch.as_tensor(x, dtype=torch.float64))
        self.p.copy_(torch.as_tensor(p, dtype=torch.float64))
        self.srow.zero_()  # cold row-solve start: results depend only on (x, p)
        self.xbar.copy_(self.x)
        self.pbar.copy_(self.p)
        if self.mode == "ksection":
            self.x_prev.copy_(self.x)
        self.colsum(self.x, self.cs)
        self.cs_prev.copy_(self.cs)
        self.csbar.copy_(self.cs)
        self.navg = 0
        self.navg_dev.zero_()
        self._sparse_sync()
        self.snapshot()

    def load_full_state(self, x, x_prev, p, xbar, pbar, navg):
        """Mid-run state of kernels.pdhcg_chunk's argument list (lockstep tests)."""
        f = lambda a: torch.as_tensor(np.asarray(a), dtype=torch.float64)  # noqa: E731
        self.x.copy_(f(x))
        self.srow.zero_()
        self.p.copy_(f(p))
        self.xbar.copy_(f(xbar))
        self.pbar.copy_(f(pbar))
        self.colsum(self.x, self.cs)
        self.colsum(self.xbar, self.csbar)
        if self.mode == "ksection":
            self.x_prev.copy_(f(x_prev))
            self.colsum(self.x_prev, self.cs_prev)
        else:
            xp = torch.as_tensor(np.asarray(x_prev), dtype=torch.float64, device=self.x.device)
            self.colsum(xp, self.cs_prev)
        self.navg = int(navg)
        self.navg_dev.fill_(self.navg)
        self._sparse_sync()
        self.snapshot()

    def initial_state(self, w_sum=None):
        """x_ij = 1/colcount_j, p_j = sum(w)/m (pdhcg.py:66-72)."""
        counts = self._global_counts()
        x = 1.0 / counts.to(torch.float64)[self.dm.col.to(torch.int64)]
        if w_sum is None:
            w_sum = float(self._allreduce(self.dm.w.sum().reshape(1)).item())
        p = torch.full((self.dm.m,), w_sum / self.dm.m, dtype=torch.float64,
                       device=self.dm.device)
        self.load_state(x, p)

    def _global_counts(self):
        return self._allreduce(self.dm.col_counts.clone())

    def set_steps(self, tau, sigma):
        if (tau, sigma) != (self.tau, self.sigma):
            self.tau, self.sigma = float(tau), float(sigma)
            self.steps.copy_(torch.tensor([self.tau, self.sigma], dtype=torch.float64))

    def snapshot(self):
        self.x0.copy_(self.x)
        self.p0.copy_(self.p)
        self.cs0.copy_(self.cs)

    def restart(self):
        """x <- xbar, p <- pbar, x_prev <- x, navg <- 0 (driver.py:164-168)."""
        self.x.copy_(self.xbar)
        self.p.copy_(self.pbar)
        self.cs.copy_(self.csbar)
        self.cs_prev.copy_(self.csbar)
        if self.mode == "ksection":
            self.x_prev.copy_(self.x)
        self.navg = 0
        self.navg_dev.zero_()
        self._sparse_sync()

    def adopt_average(self):
        self.x.copy_(self.xbar)
        self.p.copy_(self.pbar)
        self.cs.copy_(self.csbar)
        if self.sparse:
            self.xflag.fill_(1)
        if self.working_set:
            self.ws_len.copy_(self.ws_init)
            self.ws_kmax.zero_()
            if self.pool:
                self.pl_hdr[:, 0] = -1
            if self.mpool:
                self.pm_hdr[:, 0] = -1
            self._rebuild = True

    # ------------------------------------------------------------ chunks
    def run_chunk(self, iters):
        """`iters` PDHCG iterations; returns the per-iteration work counts.
        Raises SubproblemError on faulted rows (driver.py:142-144)."""
        if self.mode == "ksection":
            return self._run_chunk_ksection(iters)
        if iters > self.pass_buf.numel():
            raise ValueError("chunk longer than the pass buffer")
        rebuild = self.working_set and self._rebuild
        if self.use_graphs:
            g = self._graphs.get((iters, rebuild))
            if g is None:
                try:
                    g = self._capture(iters, rebuild)
                except Exception as exc:  # capture unsupported: eager launches
                    if not self.distributed:
                        raise
                    import warnings

                    warnings.warn(f"chunk capture with collectives failed ({exc}); "
                                  "launching eagerly")
                    self.use_graphs = False
            if g is not None:
                g.replay()
            else:
                self._launch_chunk(iters, rebuild)
        else:
            self._launch_chunk(iters, rebuild)
        self._rebuild = False
        self.navg += iters
        self._xbar_stale = self.sparse
        vals = torch.cat([self.pass_buf[:iters], self.faults]).cpu().numpy()
        if vals[-1]:
            raise FixedPointRangeError(
                f"{int(vals[-1])} allocation entries reached the fixed-point column-sum "
                f"range (x >= cs_xmax = {self.dm.struct.cs_xmax:g}); the iterate diverged")
        if vals[-2]:
            raise SubproblemError(f"{int(vals[-2])} row subproblems failed to converge")
        return [int(v) for v in vals[:-2]]

    def _launch_chunk(self, iters, rebuild=False):
        """One chunk: per iteration price step, fused prox + column sums, and on
        N ranks the all-reduce of the m-length column sums before the running
        average of colsum(xbar) is updated.  rebuild: the first iteration
        rebuilds every working set (after the host invalidated them)."""
        ops = self.ops
        self.pass_buf[:iters].zero_()
        self.faults.zero_()
        single = not self.distributed
        exact = self.fixed and not single
        for it in range(iters):
            ops.dual(it)
            ops.primal(it, rebuild=rebuild and it == 0)
            if exact:  # integer all-reduce of the fixed-point sums, then convert
                self._allreduce(self.bucket.view(torch.int64)[:self.dm.m])
                ops.colsum_rest(it, True)
                continue
            if self.colsum_fp64 and single:
                ops.colsum_rest(it, False)  # zeroes the accumulators, advances the drift
                ops.colsum(self.x, self.cs)
                ops.finalize(it)
                continue
            ops.colsum_rest(it, single)
            if not single:
                self._allreduce(self.cs)
                ops.finalize(it)
        if not single:
            self._allreduce(self.pass_buf[:iters])
            self._allreduce(self.faults)
        ops.chunk_end(iters)

    def _capture(self, iters, rebuild=False):
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=self.dm.device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            torch.cuda.synchronize(self.dm.device)
        with torch.cuda.graph(g, stream=side):
            self._launch_chunk(iters, rebuild)
        torch.cuda.current_stream().wait_stream(side)
        self._graphs[(iters, rebuild)] = g
        return g

    def _run_chunk_ksection(self, iters):
        rc, navg = self.ops.ksection_chunk(iters)
        if rc > 0:
            raise SubproblemError(f"{rc} row subproblems exceeded {MAX_ROW_PASSES} passes")
        self.navg = navg
        self.navg_dev.fill_(self.navg)
        # column sums of the iterates for residuals / restart moves
        self.colsum(self.x, self.cs)
        self.colsum(self.x_prev, self.cs_prev)
        self.colsum(self.xbar, self.csbar)
        return [int(v) for v in self.pass_buf[:iters].cpu().numpy()]

    # ------------------------------------------------------------ reductions
    def _rows(self, x, p, use_norm, k, t_out=None):
        self.colbest[k].zero_()
        self.ops.resid_rows(x, p, use_norm, self.colbest[k], t_out, self.out[16 * k: 16 * k + 8],
                            self.scratch if k == 0 else self.scratch2)
        self._reduce_rows(k)

    def _reduce_rows(self, k):
        if self.distributed:
            o = self.out[16 * k: 16 * k + 8]
            self._allreduce(self.colbest[k], "max")
            mx = o[0:4].clone()
            self._allreduce(mx, "max")
            o[0:4].copy_(mx)
            bad = torch.where(o[4:5] < 0, torch.full_like(o[4:5], math.inf), o[4:5])
            self._allreduce(bad, "min")
            o[4:5].copy_(torch.where(torch.isinf(bad), torch.full_like(bad, -1.0), bad))
            sm = o[5:7].clone()
            self._allreduce(sm, "sum")
            o[5:7].copy_(sm)

    def _cols(self, cs, p, k):
        self.ops.resid_cols(cs, p, self.colbest[k], self.out[16 * k + 8: 16 * k + 14],
                            self.scratch if k == 0 else self.scratch2)

    @staticmethod
    def _assemble(v):
        ymax, gmax, xmax, emax, bad, _obj, nbad = v[0:7]
        colgap, csmax, dualp, slmax = v[8:12]
        if nbad > 0:
            raise ValueError(f"buyer {int(bad)} has zero utility value; state is not a "
                             "valid compact iterate")
        r_primal = colgap / (1.0 + max(csmax, 0.0, 1.0))
        r_dual = max(0.0, dualp) / (1.0 + max(ymax, ymax, slmax))
        r_gap = gmax / (1.0 + max(xmax, emax))
        return Residuals(float(r_primal), float(r_dual), float(r_gap),
                         float(max(r_primal, r_dual, r_gap)))

    @property
    def xbar(self):
        """The running average x̄.  With the sparse iterate a chunk leaves it
        as xsum / navg unformed (the residual check reads the sum directly);
        it is formed here, once, when anything else reads it."""
        if self._xbar_stale:
            self._xbar_stale = False
            self.ops.avg_xbar()
        return self._xbar_t

    def residuals_pair(self):
        """(last, avg) residuals on the ORIGINAL instance with one sync; with
        the sparse iterate both row passes run as one sweep (mq_resid_rows_pair),
        reading x̄ as xsum / navg when it has not been formed."""
        if self.sparse and isinstance(self.ops, NativeOps):
            self.colbest.zero_()
            self.state.xbar_lazy = int(self._xbar_stale)
            try:
                self.ops.resid_pair(self.colbest[0], self.colbest[1], self.out[0:8],
                                    self.out[16:24])
            finally:
                self.state.xbar_lazy = 0
            self._reduce_rows(0)
            self._reduce_rows(1)
        else:
            self._rows(self.x, self.p, 0, 0)
            self._rows(self.xbar, self.pbar, 0, 1)
        self._cols(self.cs, self.p, 0)
        self._cols(self.csbar, self.pbar, 1)
        v = self.out.cpu().numpy()
        return self._assemble(v[0:16]), self._assemble(v[16:32])

    def residuals_avg(self):
        self._rows(self.xbar, self.pbar, 0, 1)
        self._cols(self.csbar, self.pbar, 1)
        return self._assemble(self.out[16:32].cpu().numpy())

    def omega_norms(self):
        """(||colsum(x)-1||_2, ||min(p - max_col u y, 0)||_2) on the normalized
        instance (driver.py:123-132)."""
        self._rows(self.x, self.p, 1, 0)
        self._cols(self.cs, self.p, 0)
        v = self.out[0:16].cpu().numpy()
        if v[6] > 0:
            raise ValueError("warm start gives some buyer zero utility")
        return math.sqrt(v[12]), math.sqrt(v[13])

    def restart_moves(self):
        """(||dx||, ||dp||, ||dx||^2, ||dp||^2, |colsum(dx).dp|) of the average
        against the last restart point (driver.py:156-162)."""
        o = self.out[24:28]
        self.ops.restart_moves(self.xbar, self.x0, self.pbar, self.p0, self.csbar, self.cs0, o,
                               self.scratch)
        if self.distributed:
            sx = o[0:1].clone()
            self._allreduce(sx, "sum")
            o[0:1].copy_(sx)
        dxx, dpp, inter = (float(v) for v in o[0:3].cpu().numpy())
        return math.sqrt(dxx), math.sqrt(dpp), dxx, dpp, abs(inter)

    def _gather(self, t):
        return gather_rows(t, self.group, self.world)

    def final_payload(self, gather=False):
        """prices, allocation, utility values, dual values, objective.  On N
        ranks the allocation and the per-buyer values are this rank's rows,
        or (gather=True) the whole market's in row order."""
        self._rows(self.x, self.p, 0, 0, t_out=self.t_buf)
        v = self.out[0:8].cpu().numpy()
        x, t, w = self.x, self.t_buf, self.dm.w
        if gather and self.world > 1:
            x, t, w = self._gather(x), self._gather(t), self._gather(w)
        t = t.cpu().numpy()
        w = w.cpu().numpy()
        with np.errstate(divide="ignore"):
            y = w / t
        obj = -float(v[5]) if v[6] == 0 else math.inf
        return {"prices": self.p.cpu().numpy(), "allocation": to_host(x),
                "utility_values": t, "dual_values": y, "objective": obj}
