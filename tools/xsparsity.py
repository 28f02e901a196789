"""Fraction of allocation entries that are nonzero along a config-4 run."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv += ["--no-cpu", "--no-e2e"]
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c4"
shard = bench.shard_rows(cfg, 0, 1, 0)
dm, eng = bench.make_session(shard, None)
done = 0
for target in [0, 1, 5, 20, 40, 100, 200, 400, 1000, 2000, 4000]:
    if target > done:
        bench.run_iters(eng, target - done)
        done = target
    torch.cuda.synchronize()
    nz = int((eng.x > 0).sum().item())
    print(f"iter {done:5d}: nonzero x {nz / dm.nnz:.4f}", flush=True)
