"""BASELINE config 1 (dense 1000 x 500, U(0,1) from default_rng(0), w = 1):
the reference's own solve (tests/golden/solve_c1.npz, run on the build
container's CPU) against run_solve on the GPU, same instance.

    python tools/c1_solve.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2506_06258_b200 as mq  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "solve_c1.npz"))
U = np.random.default_rng(0).random((1000, 500))
U[U == 0.0] = 0.5
inst = mq.FisherInstance(mq.SparseMatrix.from_dense(U), np.ones(1000))
assert mq.instance_fingerprint(inst) == str(g["fingerprint"])
kw = dict(tol=float(g["tol"]), subproblem_tol=float(g["subtol"]), sections=int(g["sections"]))
if "restart" in g.files:
    kw.update(restart=str(g["restart"]), restart_k=int(g["restart_k"]),
              step_mode=str(g["step_mode"]), max_iters=int(g["max_iters"]))
mq.run_solve(inst, mq.SolveConfig(tol=1e-2), "pdhcg")  # library load, first graphs
out = {}
for solver in ("exact", "ksection"):
    t = time.perf_counter()
    rep = mq.run_solve(inst, mq.SolveConfig(**kw, row_solver=solver), "pdhcg")
    out[solver] = {"seconds": round(time.perf_counter() - t, 3), "iterations": rep.inner_iterations,
                   "restarts": rep.restarts,
                   "price_rel_diff": float(np.max(np.abs(rep.prices - g["prices"]) / g["prices"]))}
out["reference"] = {"seconds": float(g["ref_seconds"]), "iterations": int(g["iters"]),
                    "restarts": int(g["restarts"])}
print(json.dumps(out))
