"""Restarted PDHCG solve on the B200 (market_eq/driver.py:35-377, PDHCG branch).

The control flow is the reference's, decision for decision: validate,
normalize, initial (or warm) state, operator norm L, omega_0 from the
residual norms, StepController(eta 0.9/L, cap 0.95/L, omega band x16),
chunks of `check_every` iterations, residuals of the last and the averaged
iterate on the original instance, metric = min of the two, stop at tol or the
iteration cap (adopting the better iterate), adaptive restart test, restart
moves -> controller update -> restart to the average.

What moved to the device: every nnz- or m-sized operation (the chunk, the
column sums, residuals, omega_0 norms, restart moves, normalization, the
transpose schedule).  The host keeps only scalars.
"""

import logging
import time
from dataclasses import dataclass, field, replace

import numpy as np

from .adaptive import RestartParams, StepController, should_restart, update_weights
from .errors import ValidationError
from .instance import FisherInstance
from .report import SolveReport, instance_fingerprint
from .sparse import selector_norm_from_counts

log = logging.getLogger("market_eq")

OMEGA_BOUND_FACTOR = 16.0  # driver.py:31


@dataclass
class SolveConfig:
    tol: float = 1e-4
    max_iters: int = 100_000
    restart: str = "adaptive"          # "adaptive" or "fixed"
    restart_k: int = 0                 # inner length when restart == "fixed"
    sections: int = 32                 # k-section grid (row_solver="ksection")
    subproblem_tol: float = 1e-10      # k-section bracket width (row_solver="ksection")
    step_mode: str = "adaptive"        # "theory" or "adaptive"
    adapt_eta: bool = True
    check_every: int = 40
    threads: int = None                # accepted for API compatibility (no CPU threads)
    restart_params: RestartParams = field(default_factory=RestartParams)
    # B200 additions
    row_solver: str = "exact"          # "exact" (active-set closed form) or "ksection"
    device: object = None              # torch device / index; default current CUDA device
    use_graphs: bool = True            # CUDA-graph capture of chunks
    working_set: bool = True           # screened row solves (exact)
    group: object = None               # torch.distributed group: buyers row-sharded over
                                       # its ranks (one GPU each), NCCL all-reduces

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tol must be positive")
        if self.restart not in ("adaptive", "fixed"):
            raise ValueError("restart must be 'adaptive' or 'fixed'")
        if self.restart == "fixed" and self.restart_k < 1:
            raise ValueError("fixed restart needs restart_k >= 1")
        if self.step_mode not in ("theory", "adaptive"):
            raise ValueError("step_mode must be 'theory' or 'adaptive'")
        if self.sections < 2:
            raise ValueError("sections must be >= 2")
        if self.check_every < 1:
            raise ValueError("check_every must be >= 1")
        if self.row_solver not in ("exact", "ksection"):
            raise ValueError("row_solver must be 'exact' or 'ksection'")

    def with_overrides(self, **kw):
        return replace(self, **kw)

    def as_dict(self):
        rp = self.restart_params
        return {
            "tol": self.tol, "max_iters": self.max_iters,
            "restart": f"fixed:{self.restart_k}" if self.restart == "fixed" else "adaptive",
            "sections": self.sections, "subproblem_tol": self.subproblem_tol,
            "step_mode": self.step_mode, "adapt_eta": self.adapt_eta,
            "check_every": self.check_every, "threads": self.threads,
            "beta_sufficient": rp.beta_sufficient, "beta_necessary": rp.beta_necessary,
            "beta_artificial": rp.beta_artificial, "row_solver": self.row_solver,
            **({} if self.group is None else {"ranks": _world(self.group)}),
        }


class _Fingerprint:
    """instance_fingerprint computed on a side thread (hashlib releases the
    GIL on large buffers), overlapped with the device solve."""

    def __init__(self, inst):
        import threading

        self.value = ""
        if inst is None:
            self.thread = None
            return
        self.thread = threading.Thread(target=self._run, args=(inst,), daemon=True)
        self.thread.start()

    def _run(self, inst):
        self.value = instance_fingerprint(inst)

    def get(self):
        if self.thread is not None:
            self.thread.join()
        return self.value


class _DeviceFingerprint(_Fingerprint):
    """instance_fingerprint of a device-resident instance (fileio.load_device),
    streamed back on a side thread and its own CUDA stream."""

    def __init__(self, dm, budgets):
        import threading

        import torch

        self.value = ""
        dev = dm.device
        stream = torch.cuda.Stream(device=dev)
        stream.wait_stream(torch.cuda.current_stream(dev))

        def run():
            from .fileio import device_fingerprint

            with torch.cuda.device(dev), torch.cuda.stream(stream):
                self.value = device_fingerprint(dm, budgets)

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()


def device_violations(dm):
    """validate() (instance.py:87-115) evaluated on the device copy."""
    import torch

    lens = dm.row_ptr[1:] - dm.row_ptr[:-1]
    out = [f"buyer {int(i)} values no good" for i in torch.nonzero(lens == 0).flatten().tolist()]
    counts = dm.col_counts
    out += [f"good {int(j)} unvalued" for j in torch.nonzero(counts == 0).flatten().tolist()]
    out += [f"nonpositive budget for buyer {int(i)}"
            for i in torch.nonzero(dm.w <= 0).flatten().tolist()]
    return out


class DeviceSession:
    """Device market + engine kept alive across solves of the same utilities
    (Arrow-Debreu re-solves with new budgets; benchmarks)."""

    def __init__(self, inst, cfg, group=None, dm=None, algo="pdhcg"):
        from .device import DeviceMarket
        from .engine import PdhcgEngine

        self.dm = dm if dm is not None else DeviceMarket.from_instance(inst, device=cfg.device)
        if algo == "pdhg":  # lifted PDHG (driver.py:184-268), lifted operator norm
            from .lifted import LiftedEngine

            self.engine = LiftedEngine(self.dm, use_graphs=cfg.use_graphs, group=group)
            self.op_norm = self.engine.op_norm()
            return
        self.engine = PdhcgEngine(self.dm, row_solver=cfg.row_solver, sections=cfg.sections,
                                  subproblem_tol=cfg.subproblem_tol, use_graphs=cfg.use_graphs,
                                  group=group, working_set=cfg.working_set)
        counts = self.engine._global_counts().cpu().numpy()
        self.op_norm = selector_norm_from_counts(counts)


def _world(group):
    import torch.distributed as dist

    return dist.get_world_size(group)


def split_rows(row_offsets, world):
    """Contiguous buyer ranges balanced by entries: rank r owns rows
    [cuts[r], cuts[r+1]) (the partition of bench.shard_rows)."""
    ro = np.asarray(row_offsets, dtype=np.int64)
    n, nnz = len(ro) - 1, int(ro[-1])
    targets = [nnz * r // world for r in range(1, world)]
    cuts = [0] + [min(n, int(np.searchsorted(ro[1:], t)) + 1) for t in targets] + [n]
    return [min(c, n) for c in cuts]


def solve_on_device(session, cfg, warm_start=None, w_sum=None, inst=None, algo="pdhcg",
                    fingerprint=None, gather=False):
    """The restarted loop of driver.py:271-377 against a DeviceSession."""
    eng = session.engine
    if fingerprint is None:
        fingerprint = _Fingerprint(inst)
    if algo == "pdhg":
        warm_start = None  # the lifted solver ignores warm starts (driver.py:271-276)
    if warm_start is not None:
        import torch

        x, p = warm_start["x"], warm_start["p"]
        if not isinstance(x, torch.Tensor):  # device tensors stay on the device
            x = np.asarray(x, dtype=np.float64)
        if not isinstance(p, torch.Tensor):
            p = np.asarray(p, dtype=np.float64)
        if tuple(x.shape) != (session.dm.nnz,) or tuple(p.shape) != (session.dm.m,):
            raise ValueError("warm start shapes do not match the instance")
        eng.load_state(x, p)
    else:
        eng.initial_state(w_sum=w_sum)

    L = max(session.op_norm, np.finfo(float).tiny)
    if cfg.step_mode == "theory":
        controller = None
        tau = sigma = 1.0 / (2.0 * L)
        if warm_start is not None:
            eng.omega_norms()  # zero-utility check of the warm start
    else:
        primal_res, dual_res = eng.omega_norms()
        if primal_res > 1e-8 and dual_res > 1e-8:
            omega0 = max(1.0, dual_res / primal_res)
        else:
            omega0 = 1.0
        controller = StepController(eta_initial=0.9 / L, omega_initial=omega0, eta_max=0.95 / L,
                                    omega_lower=omega0 / OMEGA_BOUND_FACTOR,
                                    omega_upper=omega0 * OMEGA_BOUND_FACTOR)
        tau, sigma = controller.tau, controller.sigma
    eng.set_steps(tau, sigma)
    log.info("%s solve on %s: n=%d m=%d nnz=%d L=%.3g tau=%.3g sigma=%.3g", algo,
             session.dm.device, session.dm.n, session.dm.m, session.dm.nnz, L, tau, sigma)

    res_avg = eng.residuals_avg()
    metric_last_restart = metric_prev_check = res_avg.rel_kkt
    history, passes = [], []
    total = restarts = 0
    chunk_time = 0.0
    t0 = time.perf_counter()
    while True:
        chunk = min(cfg.check_every, cfg.max_iters - total)
        if cfg.restart == "fixed":
            chunk = min(chunk, cfg.restart_k - eng.navg)
        tc = time.perf_counter()
        passes.extend(eng.run_chunk(chunk))
        chunk_time += time.perf_counter() - tc
        total += chunk
        res_last, res_avg = eng.residuals_pair()
        metric = min(res_last.rel_kkt, res_avg.rel_kkt)
        history.append((total, metric))
        if metric <= cfg.tol or total >= cfg.max_iters:
            if res_avg.rel_kkt < res_last.rel_kkt:
                eng.adopt_average()
                final = res_avg
            else:
                final = res_last
            status = "optimal" if metric <= cfg.tol else "max-iters"
            break
        if cfg.restart == "fixed":
            do_restart = eng.navg >= cfg.restart_k
        else:
            do_restart = should_restart(res_avg.rel_kkt, metric_last_restart, metric_prev_check,
                                        eng.navg, total, cfg.restart_params)
        metric_prev_check = res_avg.rel_kkt
        if do_restart:
            if controller is not None:
                pm, dm_, psq, dsq, inter = eng.restart_moves()
                eta_obs = None
                if cfg.adapt_eta and inter > 0.0:
                    eta_obs = (controller.omega * psq + dsq / controller.omega) / (2.0 * inter)
                update_weights(controller, pm, dm_, eta_obs)
                eng.set_steps(controller.tau, controller.sigma)
            eng.restart()
            restarts += 1
            eng.snapshot()
            metric_last_restart = metric_prev_check = res_avg.rel_kkt
    wall = time.perf_counter() - t0
    log.info("%s finished: status=%s iters=%d restarts=%d rel_kkt=%.3g (%.2fs)", algo, status,
             total, restarts, final.rel_kkt, wall)
    payload = eng.final_payload(gather=gather)
    echo = cfg.as_dict()
    echo["algo"] = algo
    objective = payload.pop("objective")
    return SolveReport(
        solver=algo, status=status, inner_iterations=total, restarts=restarts,
        wall_time_seconds=wall, final_residuals=final, residual_history=history,
        instance_fingerprint=fingerprint.get(),
        config_echo=echo, subproblem_passes=None if algo == "pdhg" else passes,
        objective=objective,
        device_stats={"chunk_seconds": chunk_time,
                      "iters_per_second": total / chunk_time if chunk_time > 0 else None,
                      "op_norm": L, "device": str(session.dm.device)},
        **payload)


def run_solve(inst, cfg, algo, warm_start=None):
    """Restarted solve of a Fisher instance on the GPU; returns a SolveReport.

    `warm_start`, when given, is a dict {"x": entry-aligned allocation,
    "p": prices} used by the compact solver; algo="pdhg" (lifted PDHG)
    ignores it, as the reference does.

    With cfg.group (a torch.distributed group of N > 1 ranks, one GPU each,
    every rank calling run_solve), buyers are row-sharded: `inst` is either
    the whole FisherInstance on every rank (each rank uploads its
    entry-balanced rows; the report carries the whole allocation) or this
    rank's FisherShard (the report carries this rank's rows).
    """
    if algo not in ("pdhcg", "pdhg"):
        raise ValueError(f"unknown algorithm {algo!r}")
    from .instance import FisherShard

    world = 1 if cfg.group is None else _world(cfg.group)
    if isinstance(inst, FisherShard) or world > 1:
        if not isinstance(inst, (FisherInstance, FisherShard)):
            raise TypeError(f"unsupported instance type {type(inst)!r}")
        if cfg.group is None:
            raise ValueError("a FisherShard is solved with SolveConfig.group set")
        return _run_solve_sharded(inst, cfg, algo, warm_start, world)
    from .fileio import DeviceFisherInstance

    if isinstance(inst, DeviceFisherInstance):  # streamed into device CSR (fileio)
        dm = inst.dm
        violations = device_violations(dm)
        if violations:
            raise ValidationError("; ".join(violations))
        fp = _DeviceFingerprint(dm, inst.budgets)
        session = DeviceSession(None, cfg, dm=dm, algo=algo)
        return solve_on_device(session, cfg, warm_start=warm_start,
                               w_sum=float(np.sum(inst.budgets)), fingerprint=fp, algo=algo)
    if not isinstance(inst, FisherInstance):
        raise TypeError(f"unsupported instance type {type(inst)!r}")
    from .device import DeviceMarket

    fp = _Fingerprint(inst)
    dm = DeviceMarket.from_instance(inst, device=cfg.device)
    violations = device_violations(dm)
    if violations:
        raise ValidationError("; ".join(violations))
    session = DeviceSession(inst, cfg, dm=dm, algo=algo)
    return solve_on_device(session, cfg, warm_start=warm_start,
                           w_sum=float(np.sum(inst.budgets)), inst=inst, fingerprint=fp,
                           algo=algo)


def _run_solve_sharded(inst, cfg, algo, warm_start, world):
    """run_solve on this rank's rows (see run_solve)."""
    import torch
    import torch.distributed as dist

    from .device import DeviceMarket
    from .instance import FisherShard

    rank = dist.get_rank(cfg.group)
    dev = cfg.device if cfg.device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    u = inst.utilities
    if isinstance(inst, FisherShard):
        lo, rows = inst.row_begin, inst.n_buyers
        e_lo, e_hi = 0, u.nnz
        rp, col, val, w = u.row_offsets, u.col_indices, u.values, inst.budgets
        fp = _Fingerprint(None)
        gather = False
    else:
        cuts = split_rows(u.row_offsets, world)
        lo, hi = cuts[rank], cuts[rank + 1]
        rows = hi - lo
        e_lo, e_hi = int(u.row_offsets[lo]), int(u.row_offsets[hi])
        rp = u.row_offsets[lo:hi + 1] - e_lo
        col, val, w = u.col_indices[e_lo:e_hi], u.values[e_lo:e_hi], inst.budgets[lo:hi]
        fp = _Fingerprint(inst)
        gather = True
    dm = DeviceMarket(rp, col, val, w, u.n_cols, device=dev, row_begin=lo)
    # validate() across the ranks: empty rows / budgets locally, goods globally
    lens = dm.row_ptr[1:] - dm.row_ptr[:-1]
    bad = [f"buyer {lo + int(i)} values no good" for i in torch.nonzero(lens == 0).flatten()]
    bad += [f"nonpositive budget for buyer {lo + int(i)}"
            for i in torch.nonzero(dm.w <= 0).flatten()]
    counts = dm.col_counts.clone()
    dist.all_reduce(counts, group=cfg.group)
    bad += [f"good {int(j)} unvalued" for j in torch.nonzero(counts == 0).flatten()]
    nbad = torch.tensor([len(bad)], dtype=torch.int64, device=dm.device)
    dist.all_reduce(nbad, group=cfg.group)
    if int(nbad.item()):
        raise ValidationError("; ".join(bad) if bad else "invalid rows on another rank")
    wsum = torch.tensor([float(np.sum(w))], dtype=torch.float64, device=dm.device)
    dist.all_reduce(wsum, group=cfg.group)
    local_warm = None
    if warm_start is not None and algo == "pdhcg":
        x = np.asarray(warm_start["x"], dtype=np.float64)
        local_warm = {"x": x if isinstance(inst, FisherShard) else x[e_lo:e_hi],
                      "p": warm_start["p"]}
    session = DeviceSession(None, cfg, group=cfg.group, dm=dm, algo=algo)
    return solve_on_device(session, cfg, warm_start=local_warm, w_sum=float(wsum.item()),
                           inst=None, fingerprint=fp, algo=algo, gather=gather)
