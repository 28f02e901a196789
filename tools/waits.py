"""Debug: wait-cycle breakdown of the fused primal kernel (build with
python -m paper_2506_06258_b200._build --profile-waits)."""
import ctypes
import sys

import numpy as np
import torch

sys.argv += ["--no-cpu", "--no-e2e"]
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import bench
from paper_2506_06258_b200 import _native as nat

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c4"
shard = bench.shard_rows(cfg, 0, 1, 0)
dm, eng = bench.make_session(shard, None)
lib = nat.load_library()
lib.mq_debug_counters.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 16)()
bench.run_iters(eng, 3)
torch.cuda.synchronize()
lib.mq_debug_counters(buf)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
bench.run_iters(eng, 10)
e1.record()
torch.cuda.synchronize()
lib.mq_debug_counters(buf)
ms = e0.elapsed_time(e1) / 10
cyc = ms * 1e-3 * 1.965e9
nsm = dm.prim_grid
names = ["solver wait tile", "(unused)", "producer wait stage", "(unused)", "(unused)",
         "solver loads + c", "solver root", "solver stores", "solver claim",
         "solver row meta", "solver tile end"]
print(f"{cfg}: {ms:.3f} ms/iter, kernel-cycles/SM ~{cyc:.3e}")
NSW = 19  # solver warps of the default build (fast.cu MQ_NSW)
per_warp = {i: NSW for i in range(11)}
per_warp[2] = 1
for i, nm in enumerate(names):
    if nm == "(unused)":
        continue
    v = buf[i] / 10 / nsm / per_warp[i]
    print(f"  {nm:22s} {v:.3e} cycles per warp per iter ({100 * v / cyc:.1f}% of iter)")
print(f"  row pairs per warp per iter {buf[12] / 10 / nsm / NSW:.0f}, "
      f"tile visits {buf[13] / 10 / nsm / NSW:.0f}")
