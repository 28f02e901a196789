"""Arrow-Debreu exchange market at BASELINE config 5 scale (n = m = 1e5,
U and E each Bernoulli(0.01)), generated on device, solved through the
public solve_exchange API (warm-started PDHCG inner solves on the B200).

    python tools/exchange_c5.py [--n 100000] [--q 0.01] [--inner-max-iters 100000]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_06258_b200 as mq  # noqa: E402
from paper_2506_06258_b200.generate import generate_rows  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--q", type=float, default=0.01)
ap.add_argument("--inner-max-iters", type=int, default=100_000)  # the reference default
ap.add_argument("--max-outer", type=int, default=40)
ap.add_argument("--outer-tol", type=float, default=1e-6)
a = ap.parse_args()


def host_csr(d, n, m):
    rp = d["row_ptr"].cpu().numpy()
    col = d["col"].cpu().numpy().astype(np.int64)
    val = d["u"].cpu().numpy()
    return rp, col, val


t0 = time.perf_counter()
U = generate_rows(a.n, a.n, seed=5, q=a.q, budgets=False)
E = generate_rows(a.n, a.n, seed=6, q=a.q, budgets=False)
urp, ucol, uval = host_csr(U, a.n, a.n)
erp, ecol, evals = host_csr(E, a.n, a.n)
cs = np.bincount(ecol, weights=evals, minlength=a.n)
if np.any(cs == 0):
    raise SystemExit("empty endowment column; pick another seed")
evals = evals / cs[ecol]
inst = mq.ExchangeInstance(mq.SparseMatrix(a.n, a.n, urp, ucol, uval),
                           mq.SparseMatrix(a.n, a.n, erp, ecol, evals))
gen_s = time.perf_counter() - t0
t0 = time.perf_counter()
tr = mq.solve_exchange(inst, outer_tol=a.outer_tol, max_outer=a.max_outer,
                       inner_config=mq.SolveConfig(max_iters=a.inner_max_iters))
wall = time.perf_counter() - t0
print(json.dumps({
    "n": a.n, "m": a.n, "nnz_u": int(len(uval)), "nnz_e": int(len(evals)),
    "status": tr.status, "outer_iterations": tr.outer_iterations,
    "budget_gaps": tr.budget_gaps,
    "inner": [(r.status, r.inner_iterations, r.restarts, round(r.wall_time_seconds, 2))
              for r in tr.inner_reports],
    "seconds": round(wall, 2), "generate_seconds": round(gen_s, 2)}))
