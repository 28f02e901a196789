"""Restarted PDHCG entry point (market_eq/pdhcg.py:204-208)."""


def solve_fisher_pdhcg(inst, config=None):
    """Solve a Fisher instance with restarted PDHCG on the GPU."""
    from .driver import SolveConfig, run_solve

    return run_solve(inst, config or SolveConfig(), algo="pdhcg")
