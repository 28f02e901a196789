"""Arrow-Debreu inner configurations on SPEC acceptance 6's instance
(generate_exchange(n=1000, m=400, sparsity_u=0.2, sparsity_e=0.5, seed),
outer_tol 1e-6): which documented SolveConfig knobs let the
reference's fixed-point loop converge.

    python tools/ad_explore.py [--seeds 0,1,2] [--solver exact|ksection]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_06258_b200 as mq  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seeds", default="0")
ap.add_argument("--solver", default="exact")
ap.add_argument("--max-outer", type=int, default=40)
ap.add_argument("--only", default=None)
a = ap.parse_args()

CONFIGS = {
    "default": dict(),
    "theory": dict(step_mode="theory"),
    "no_adapt_eta": dict(adapt_eta=False),
    "fixed_200": dict(restart="fixed", restart_k=200),
    "fixed_1000": dict(restart="fixed", restart_k=1000),
    "check_10": dict(check_every=10),
    "max_iters_20k": dict(max_iters=20_000),
    "max_iters_1m": dict(max_iters=1_000_000),
    "theory_1m": dict(step_mode="theory", max_iters=1_000_000),
    "check_10_1m": dict(check_every=10, max_iters=1_000_000),
    "beta_art_05": dict(restart_params=mq.RestartParams(0.2, 0.8, 0.5)),
}
for seed in [int(s) for s in a.seeds.split(",")]:
    ex = mq.generate_exchange(mq.GeneratorConfig(n=1000, m=400, sparsity_u=0.2, sparsity_e=0.5,
                                                 seed=seed))
    for name, kw in CONFIGS.items():
        if a.only and name not in a.only.split(","):
            continue
        cfg = mq.SolveConfig(row_solver=a.solver, **kw)
        t = time.time()
        tr = mq.solve_exchange(ex, outer_tol=1e-6, max_outer=a.max_outer, inner_config=cfg)
        r = {"seed": seed, "config": name, "status": tr.status, "outer": tr.outer_iterations,
             "gaps": [float(f"{g:.3e}") for g in tr.budget_gaps],
             "inner_iters": [rep.inner_iterations for rep in tr.inner_reports],
             "inner_status": [rep.status for rep in tr.inner_reports][-3:],
             "seconds": round(time.time() - t, 2)}
        if tr.status == "converged":
            res, _ = mq.verify_fixed_point(ex, tr.budgets_history[-1], inner_tol=1e-8,
                                           inner_config=mq.SolveConfig(row_solver=a.solver,
                                                                       **kw))
            r["verify_residual"] = res
        print(json.dumps(r), flush=True)
