"""Lifted PDHG (algo="pdhg") on the device against the reference's own solves
(tests/golden/pdhg_*.npz, produced by oracle/gen_golden.py from the
reference and reproduced bit for bit by the oracle)."""

import numpy as np
import pytest

from conftest import golden, golden_names
from _helpers import instance_from, rel_max

pytestmark = pytest.mark.gpu


def _cfg(g):
    from paper_2506_06258_b200 import SolveConfig

    return SolveConfig(tol=float(g["tol"]), max_iters=int(g["max_iters"]),
                       restart=str(g["restart"]), restart_k=int(g["restart_k"]),
                       step_mode=str(g["step_mode"]))


@pytest.mark.parametrize("name", golden_names("pdhg_"))
def test_lifted_pdhg_matches_reference(name):
    import paper_2506_06258_b200 as mq

    g = golden(name)
    inst = instance_from(g)
    rep = mq.run_solve(inst, _cfg(g), "pdhg")
    assert rep.solver == "pdhg" and rep.subproblem_passes is None
    assert rep.status == str(g["status"])
    assert rep.inner_iterations == int(g["iters"])
    assert rep.restarts == int(g["restarts"])
    assert rel_max(rep.prices, g["prices"]) <= 1e-6
    assert np.allclose(rep.allocation, g["allocation"], rtol=1e-6, atol=1e-9)
    assert np.allclose(rep.utility_values, g["utility_values"], rtol=1e-6)
    assert np.allclose(rep.dual_values, g["dual_values"], rtol=1e-6)
    obj = float(g["objective"])
    if np.isfinite(obj):
        assert abs(rep.objective - obj) <= 1e-8 * abs(obj)
    else:
        assert not np.isfinite(rep.objective)
    hist = np.asarray(rep.residual_history)
    assert np.array_equal(hist[:, 0], g["history"][:, 0])
    assert np.allclose(hist[:, 1], g["history"][:, 1], rtol=1e-6)


def test_lifted_pdhg_is_deterministic():
    import paper_2506_06258_b200 as mq

    g = golden("pdhg_g200.npz")
    inst = instance_from(g)
    a = mq.run_solve(inst, _cfg(g), "pdhg")
    b = mq.run_solve(inst, _cfg(g), "pdhg")
    assert np.array_equal(a.prices, b.prices) and np.array_equal(a.allocation, b.allocation)


def test_lifted_and_compact_prices_agree():
    """SPEC acceptance 4: the two solvers' equilibrium prices agree
    within 1e-3 on the same market."""
    import paper_2506_06258_b200 as mq

    g = golden("pdhg_medium.npz")
    inst = instance_from(g)
    cfg = mq.SolveConfig(tol=1e-6)
    a = mq.run_solve(inst, cfg, "pdhg")
    b = mq.run_solve(inst, cfg, "pdhcg")
    assert rel_max(a.prices, b.prices) <= 1e-3
