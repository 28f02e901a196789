"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py

Touches every kernel family of the library on small markets: the unscreened
tile kernel, the screened solve (working sets: rebuild, screened, full-solve
list), medium and long rows (power-law market), the k-section drop-in, the
residual / restart reductions, the lifted PDHG step, the theory diagnostics,
the device generator and E.p.  Exits 0 after printing "sanitize workload ok".
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.generate import generate_rows

    # power-law market: short tile rows, medium rows (129..1024), long rows (> 1024)
    d = generate_rows(6000, 3000, seed=4, powerlaw=2.0, mean_degree=60.0)
    lens = np.diff(d["row_ptr"].cpu().numpy())
    assert lens.max() > 1024 and ((lens > 128) & (lens <= 1024)).any()
    for ws in (True, False):
        dm = DeviceMarket(d["row_ptr"], d["col"], d["u"], d["w"], d["m"])
        eng = PdhcgEngine(dm, working_set=ws, use_graphs=False)
        eng.initial_state()
        eng.set_steps(0.05, 0.05)
        for _ in range(3):
            eng.run_chunk(8)
        eng.residuals_pair()
        eng.restart_moves()
        eng.restart()
        eng.run_chunk(4)
        eng.final_payload()
    torch.cuda.synchronize()
    # k-section drop-in and a full solve through the public API
    inst = mq.generate_fisher(mq.GeneratorConfig(n=200, m=80, sparsity_u=0.2, seed=1))
    mq.run_solve(inst, mq.SolveConfig(tol=1e-4, row_solver="ksection", use_graphs=False,
                                      max_iters=400), "pdhcg")
    mq.run_solve(inst, mq.SolveConfig(tol=1e-4, use_graphs=False, max_iters=400), "pdhcg")
    # lifted PDHG and the theory diagnostics
    mq.run_solve(inst, mq.SolveConfig(tol=1e-3, use_graphs=False, max_iters=400), "pdhg")
    rep = mq.run_solve(inst, mq.SolveConfig(tol=1e-4, max_iters=400), "pdhcg")
    mq.smoothed_gap(inst, (rep.allocation, rep.prices), (rep.allocation, rep.prices), 1.0)
    # exchange (E.p on the device)
    ex = mq.generate_exchange(mq.GeneratorConfig(n=60, m=30, sparsity_u=0.3, sparsity_e=0.5,
                                                 seed=2))
    mq.solve_exchange(ex, outer_tol=1e-4, max_outer=3,
                      inner_config=mq.SolveConfig(use_graphs=False, max_iters=400))
    torch.cuda.synchronize()
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()
