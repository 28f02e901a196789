"""Search generated exchange instances on which the reference's fixed-point
loop (solve_exchange with its default inner configuration) converges — to pin
a converged Arrow-Debreu case against the reference itself.

    python tools/ad_search.py [--max-n 200]
"""
import argparse
import itertools
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_06258_b200 as mq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-n", type=int, default=200)
ap.add_argument("--solver", default="exact")
a = ap.parse_args()
sizes = [(n, m) for n, m in [(10, 6), (20, 10), (40, 30), (60, 20), (100, 50), (200, 80)]
         if n <= a.max_n]
for (n, m), qu, qe, seed in itertools.product(sizes, (0.3, 0.6, 1.0), (0.5, 1.0), range(3)):
    ex = mq.generate_exchange(mq.GeneratorConfig(n=n, m=m, sparsity_u=qu, sparsity_e=qe,
                                                 seed=seed))
    t = time.time()
    try:
        tr = mq.solve_exchange(ex, outer_tol=1e-6, max_outer=40,
                               inner_config=mq.SolveConfig(row_solver=a.solver))
        r = {"n": n, "m": m, "qu": qu, "qe": qe, "seed": seed, "status": tr.status,
             "outer": tr.outer_iterations, "inner": [rep.inner_iterations
                                                     for rep in tr.inner_reports][:8],
             "last_gap": tr.budget_gaps[-1] if tr.budget_gaps else None,
             "seconds": round(time.time() - t, 2)}
    except Exception as e:  # noqa: BLE001
        r = {"n": n, "m": m, "qu": qu, "qe": qe, "seed": seed, "error": repr(e)[:200]}
    print(json.dumps(r), flush=True)
