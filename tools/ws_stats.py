"""Working-set statistics along a solve (design / tuning aid).

    python tools/ws_stats.py [c4] [--iters 400] [--every 20]

Prints, every `every` iterations of the restarted solve: rows solved in full
in that iteration, working-set entries (sum of ws_len >= 0), rows whose
working set overflows the slots, nonzero entries, and the iteration time.
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

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="c4")
ap.add_argument("--iters", type=int, default=400)
ap.add_argument("--every", type=int, default=20)
a = ap.parse_args()

shard = bench.shard_rows(a.config, 0, 1, 0)
dm, eng = bench.make_session(shard, None)
rows = []
done = 0
while done < a.iters:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run_chunk(1)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    done += 1
    if done % a.every == 0 or done <= 5:
        h = eng.ws_len
        r = {"it": done, "ms": round(dt * 1e3, 3), "full_rows": int(eng.blk_done[3].item()),
             "ws_entries": int(h.clamp(min=0).sum().item()),
             "overflow_rows": int((h == -2).sum().item()),
             "nonzero": int(eng.xflag[:dm.nnz].sum().item()),
             "drift_C": float(eng.drift[0].item())}
        rows.append(r)
        print(json.dumps(r), flush=True)
print(json.dumps({"config": a.config, "n": dm.n, "nnz": dm.nnz,
                  "tile_rows": int((eng.ws_init == -1).sum().item())}))
