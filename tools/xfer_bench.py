"""Host <-> device transfer rates of engine.to_device / to_host (8 GB) against
plain torch copies.

    python tools/xfer_bench.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_06258_b200 import engine
a = np.random.default_rng(0).random(1 << 30)  # 8 GB
torch.cuda.synchronize()
for k in range(2):
    t = time.perf_counter(); d = engine.to_device(a, torch.device("cuda", 0)); torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter(); h = engine.to_host(d); t2 = time.perf_counter() - t
    print(f"to_device {a.nbytes/t1/1e9:.1f} GB/s  to_host {a.nbytes/t2/1e9:.1f} GB/s", flush=True)
    del d, h
t = time.perf_counter(); d = torch.from_numpy(a).to("cuda"); torch.cuda.synchronize(); print(f"plain .to {a.nbytes/(time.perf_counter()-t)/1e9:.1f} GB/s")
t = time.perf_counter(); h = d.cpu(); print(f"plain .cpu {a.nbytes/(time.perf_counter()-t)/1e9:.1f} GB/s")
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip(), os.cpu_count())
