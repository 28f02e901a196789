"""Time to 1e-4 relative KKT on a BASELINE config, market generated on device.

    python tools/ttt.py [c4] [--max-iters N] [--tol 1e-4]

Writes one JSON line (iterations, restarts, seconds, residual history, it/s).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_06258_b200.device import DeviceMarket  # noqa: E402
from paper_2506_06258_b200.driver import DeviceSession, SolveConfig, solve_on_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c4")
ap.add_argument("--max-iters", type=int, default=40000)
ap.add_argument("--tol", type=float, default=1e-4)
ap.add_argument("--solver", default="exact")
a = ap.parse_args()
t0 = time.perf_counter()
shard = bench.shard_rows(a.config, 0, 1, 0)
dm = DeviceMarket(shard["row_ptr"], shard["col"], shard["u"], shard["w"], shard["m"])
cfg = SolveConfig(tol=a.tol, max_iters=a.max_iters, row_solver=a.solver)
sess = DeviceSession(None, cfg, dm=dm)
setup = time.perf_counter() - t0
torch.cuda.synchronize()
t1 = time.perf_counter()
rep = solve_on_device(sess, cfg, w_sum=float(dm.w.sum().item()))
wall = time.perf_counter() - t1
print(json.dumps({
    "config": a.config, "n": dm.n, "m": dm.m, "nnz": dm.nnz, "status": rep.status,
    "iterations": rep.inner_iterations, "restarts": rep.restarts, "seconds": round(wall, 3),
    "setup_seconds": round(setup, 3), "rel_kkt": rep.final_residuals.rel_kkt,
    "objective": rep.objective, "iters_per_second_device": rep.device_stats["iters_per_second"],
    "mean_sweeps_per_row": sum(rep.subproblem_passes) / max(1, rep.inner_iterations) / dm.n,
    "history": rep.residual_history[::5] + rep.residual_history[-1:],
}))
