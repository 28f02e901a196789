"""Time the per-check reductions (residuals of x and x̄, restart moves) on
a BASELINE config after a few chunks."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.argv += ["--no-cpu", "--no-e2e"]
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "c4"
shard = bench.shard_rows(cfg, 0, 1, 0)
dm, eng = bench.make_session(shard, None)
bench.run_iters(eng, 80)
torch.cuda.synchronize()
for name, fn in (("residuals_pair", eng.residuals_pair), ("restart_moves", eng.restart_moves),
                 ("run_chunk(40)", lambda: eng.run_chunk(40))):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms", flush=True)
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
eng._rows(eng.x, eng.p, 0, 0)
e[1].record()
torch.cuda.synchronize()
print(f"resid_rows(x) device: {e[0].elapsed_time(e[1]):.2f} ms")
e[0].record()
eng._rows(eng.xbar, eng.pbar, 0, 1)
e[1].record()
torch.cuda.synchronize()
print(f"resid_rows(xbar) device: {e[0].elapsed_time(e[1]):.2f} ms")
