"""Solver entry points: restarted PDHCG (market_eq/pdhcg.py:204-208) and
lifted PDHG (market_eq/pdhg.py:169-173)."""


def solve_fisher_pdhcg(inst, config=None):
    """Solve a Fisher instance with restarted PDHCG on the GPU."""
    from .driver import SolveConfig, run_solve

    return run_solve(inst, config or SolveConfig(), algo="pdhcg")


def solve_fisher_pdhg(inst, config=None):
    """Solve a Fisher instance with restarted lifted PDHG on the GPU
    (market_eq/pdhg.py:169-173)."""
    from .driver import SolveConfig, run_solve

    return run_solve(inst, config or SolveConfig(), algo="pdhg")
