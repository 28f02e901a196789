"""Lifted PDHG iteration rate on a BASELINE config (device-generated market).

    python tools/pdhg_rate.py [c4] [--iters 200]
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
from paper_2506_06258_b200.lifted import LiftedEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c4")
ap.add_argument("--iters", type=int, default=200)
a = ap.parse_args()
shard = bench.shard_rows(a.config, 0, 1, 0)
dm = DeviceMarket(shard["row_ptr"], shard["col"], shard["u"], shard["w"], shard["m"])
eng = LiftedEngine(dm)
t0 = time.perf_counter()
L = eng.op_norm()
t_norm = time.perf_counter() - t0
eng.initial_state()
eng.set_steps(0.9 / L, 0.9 / L)
eng.run_chunk(40)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters // 40):
    eng.run_chunk(40)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (40 * (a.iters // 40))
print(json.dumps({"config": a.config, "nnz": dm.nnz, "algo": "pdhg", "ms_per_iter": round(ms, 3),
                  "iters_per_second": round(1e3 / ms, 2), "op_norm": L,
                  "op_norm_seconds": round(t_norm, 2),
                  "x_nonzero_fraction": float((eng.x > 0).double().mean().item())}))
