"""Theory diagnostics on the device (kkt.py:88-168) against the reference's
own values on random states (tests/golden/theory.npz)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _inst(g, tag):
    from paper_2506_06258_b200 import FisherInstance, SparseMatrix

    n, m = (int(v) for v in g[f"{tag}_nm"])
    return FisherInstance(SparseMatrix(n, m, g[f"{tag}_indptr"], g[f"{tag}_col"], g[f"{tag}_u"]),
                          g[f"{tag}_w"])


CASES = [f"{t}{k}" for t in "ab" for k in range(3)]


@pytest.mark.parametrize("case", CASES)
def test_scaled_kkt_residual_matches_reference(case):
    import paper_2506_06258_b200 as mq

    g = golden("theory.npz")
    inst = _inst(g, case[0])
    xi = float(g[f"{case}_xi"])
    v = mq.scaled_kkt_residual(inst, g[f"{case}_x"], g[f"{case}_t"], g[f"{case}_p"],
                               g[f"{case}_y"], xi)
    assert abs(v - float(g[f"{case}_skkt"])) <= 1e-12 * float(g[f"{case}_skkt"])
    vc = mq.scaled_kkt_residual_compact(inst, g[f"{case}_x"], g[f"{case}_p"], xi)
    assert abs(vc - float(g[f"{case}_skkt_c"])) <= 1e-12 * float(g[f"{case}_skkt_c"])


@pytest.mark.parametrize("case", CASES)
def test_smoothed_gap_matches_reference(case):
    """The reference solves each row's prox by k-section to 1e-12; the device
    solves it exactly, so the gaps agree to ~1e-10 relative."""
    import paper_2506_06258_b200 as mq

    g = golden("theory.npz")
    inst = _inst(g, case[0])
    xi = float(g[f"{case}_xi"])
    v = mq.smoothed_gap(inst, (g[f"{case}_x"], g[f"{case}_p"]),
                        (g[f"{case}_xc"], g[f"{case}_pc"]), xi=xi)
    ref = float(g[f"{case}_gap"])
    assert abs(v - ref) <= 1e-9 * abs(ref)


def test_diagnostics_reject_nonpositive_xi():
    import paper_2506_06258_b200 as mq

    g = golden("theory.npz")
    inst = _inst(g, "a")
    with pytest.raises(ValueError):
        mq.scaled_kkt_residual(inst, g["a0_x"], g["a0_t"], g["a0_p"], g["a0_y"], 0.0)
    with pytest.raises(ValueError):
        mq.smoothed_gap(inst, (g["a0_x"], g["a0_p"]), (g["a0_xc"], g["a0_pc"]), xi=-1.0)


def test_property_suite_passes():
    """theory.py's battery (market_eq/theory.py:215-302) on the device paths:
    boundedness, averaged distance, smoothed-gap nonnegativity, grid
    agreement, cross-solver prices, relabeling symmetry, exchange decay."""
    from paper_2506_06258_b200.theory import run_property_suite

    rep = run_property_suite(seed=0)
    names = {c["name"] for c in rep["checks"]}
    assert names >= {"iterate-boundedness", "averaged-distance", "smoothed-gap-nonnegative",
                     "cross-solver-prices", "relabeling-symmetry",
                     "smoothed-gap-grid-agreement", "exchange-geometric-decay"}
    for c in rep["checks"]:
        print(c)
    assert rep["all_passed"], [c for c in rep["checks"] if not c["passed"]]
    ran = [c for c in rep["checks"] if not c["skipped"]]
    assert len(ran) >= 15
