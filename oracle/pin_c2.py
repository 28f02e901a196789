"""Pin the oracle at BASELINE config 2 scale (build container only, ~1-2 h).

    python oracle/pin_c2.py

Runs the oracle's restated solve loop (oracle/solve.py + the C chunk) on
config 2 (generate_fisher(100k, 10k, 0.01, seed 0), subproblem_tol=0) and
compares it with the reference's own run frozen in
tests/golden/solve_c2_tol0.npz: iteration and restart counts, residual
history, prices and allocation bit for bit.  Writes
profiles/oracle_c2_pin.json.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import solve as orc  # noqa: E402
import paper_2506_06258_b200 as mq  # noqa: E402  (host generator only)

orc.set_threads(os.cpu_count() or 1)
g = np.load(os.path.join(ROOT, "tests", "golden", "solve_c2_tol0.npz"))
inst = mq.generate_fisher(mq.GeneratorConfig(n=100_000, m=10_000, sparsity_u=0.01, seed=0))
assert mq.instance_fingerprint(inst) == str(g["fingerprint"])
u = inst.utilities
mk = orc.Market(u.n_rows, u.n_cols, u.row_offsets, u.col_indices, u.values, inst.budgets)
t = time.time()
o = orc.solve(mk, tol=1e-4, subtol=0.0)
secs = time.time() - t
res = {
    "iterations": o["inner_iterations"], "ref_iterations": int(g["iters"]),
    "restarts": o["restarts"], "ref_restarts": int(g["restarts"]),
    "prices_bitwise": bool(np.array_equal(o["prices"], g["prices"])),
    "allocation_sha_equal": hashlib.sha256(o["allocation"].tobytes()).hexdigest()
    == str(g["allocation_sha"]),
    "history_equal": bool(np.array_equal(np.asarray(o["residual_history"], dtype=np.float64),
                                         g["history"])),
    "objective": o["objective"], "ref_objective": float(g["objective"]),
    "oracle_seconds": round(secs, 1), "ref_seconds": float(g["ref_seconds"]),
    "threads": os.cpu_count(),
}
print(json.dumps(res), flush=True)
with open(os.path.join(ROOT, "profiles", "oracle_c2_pin.json"), "w") as fh:
    json.dump(res, fh, indent=1)
