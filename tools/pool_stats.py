"""Working-set pool sizes of the long (> 1024 entries) and medium (257-1024)
rows on config 3 after 400 iterations.

    python tools/pool_stats.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv += ["--no-cpu", "--no-e2e"]
import torch
import bench
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
shard = bench.shard_rows(cfg, 0, 1, 0)
dm, eng = bench.make_session(shard, None)
bench.run_iters(eng, 400)
torch.cuda.synchronize()
h = eng.pl_hdr[:, 0].cpu()
import numpy as np
h = h.numpy()
print("long rows", len(h), "none", (h == -1).sum(), "overfull", (h == -2).sum(), "h<=32", ((h >= 0) & (h <= 32)).sum(), "h<=128", ((h >= 0) & (h <= 128)).sum(), "h<=256", ((h >= 0) & (h <= 256)).sum(), "max", h.max(), "mean", h[h >= 0].mean())
lens = (dm.row_ptr[1:] - dm.row_ptr[:-1])[dm.long_rows.to(torch.int64)].cpu().numpy()
print("len mean", lens.mean(), "max", lens.max())
hm = eng.pm_hdr[:, 0].cpu().numpy()
print("med pools", len(hm), "none", (hm == -1).sum(), "overfull", (hm == -2).sum(),
      "mean", hm[hm >= 0].mean() if (hm >= 0).any() else None, "max", hm.max())
