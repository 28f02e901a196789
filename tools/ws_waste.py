"""Slots copied per iteration (per-block kmax x 32) against slots used
(sum of h) by the screened kernel, after a few hundred iterations.

    python tools/ws_waste.py [c4|c3|c2] [iters]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv += ["--no-cpu", "--no-e2e"]
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 400
shard = bench.shard_rows(cfg, 0, 1, 0)
dm, eng = bench.make_session(shard, None)
bench.run_iters(eng, iters)
torch.cuda.synchronize()
h = eng.ws_hdr[:, 0].clamp(min=0).to(torch.int64)
used = int(h.sum())
copied = int(eng.ws_kmax.to(torch.int64).sum()) * 32
lvl = torch.bincount(eng.ws_lvl.to(torch.int64), minlength=4).tolist()
hist = torch.bincount(h, minlength=11).tolist()
print(f"{cfg} after {iters}: slots used {used:,} copied {copied:,} ratio {copied / max(used, 1):.2f}; "
      f"levels {lvl}; h histogram {hist}")
