"""Where the end-to-end run_solve time goes outside the iterations (config 4).

    python tools/e2e_profile.py [--iters 200]
"""
import argparse
import functools
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2506_06258_b200 as mq  # noqa: E402
from paper_2506_06258_b200 import device, driver, engine, report  # noqa: E402

T0 = [0.0]
LOG = []


def timed(mod, name):
    f = getattr(mod, name)

    @functools.wraps(f)
    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize()
        LOG.append((t - T0[0], time.perf_counter() - t, f"{mod.__name__.split('.')[-1]}.{name}"))
        return r
    setattr(mod, name, g)


def timed_method(cls, name):
    f = getattr(cls, name)

    @functools.wraps(f)
    def g(self, *a, **k):
        t = time.perf_counter()
        r = f(self, *a, **k)
        torch.cuda.synchronize()
        LOG.append((t - T0[0], time.perf_counter() - t, f"{cls.__name__}.{name}"))
        return r
    setattr(cls, name, g)


ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--config", default="c4")
a = ap.parse_args()
shard = bench.shard_rows(a.config, 0, 1, 0)
rp = shard["row_ptr"].cpu().numpy()
col = shard["col"].cpu().numpy().astype(np.int64)
u = shard["u"].cpu().numpy()
w = shard["w"].cpu().numpy()
inst = mq.FisherInstance(mq.SparseMatrix(shard["n"], shard["m"], rp, col, u), w)
del col, u, shard
timed(engine, "to_device")
timed(engine, "to_host")
timed(report, "instance_fingerprint")
timed(device, "build_tiles")
timed(device, "build_blocked_schedule")
timed_method(device.DeviceMarket, "__init__")
timed_method(engine.PdhcgEngine, "__init__")
timed_method(engine.PdhcgEngine, "final_payload")
timed_method(engine.PdhcgEngine, "omega_norms")
timed_method(engine.PdhcgEngine, "initial_state")
timed_method(engine.PdhcgEngine, "residuals_pair")
timed_method(engine.PdhcgEngine, "restart_moves")
timed_method(engine.PdhcgEngine, "restart")
timed_method(engine.PdhcgEngine, "run_chunk")
timed_method(driver._Fingerprint, "get")
timed(driver, "device_violations")
torch.cuda.synchronize()
T0[0] = time.perf_counter()
rep = mq.run_solve(inst, mq.SolveConfig(tol=1e-4, max_iters=a.iters), "pdhcg")
wall = time.perf_counter() - T0[0]
print(f"wall {wall:.2f} s for {rep.inner_iterations} iterations; device loop "
      f"{rep.device_stats.get('chunk_seconds', 0):.2f} s")
from collections import defaultdict  # noqa: E402

agg = defaultdict(lambda: [0, 0.0])
for t, d, nm in sorted(LOG):
    agg[nm][0] += 1
    agg[nm][1] += d
    if agg[nm][0] <= 2:
        print(f"  start {t:7.3f}  took {d:7.3f}  {nm}")
print("totals:")
for nm, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {nm:40s} calls {c:6d}  total {d:8.3f} s  mean {1e3 * d / c:8.3f} ms")
