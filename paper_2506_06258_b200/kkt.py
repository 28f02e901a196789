"""Termination metric and objective (market_eq/kkt.py:29-87, 126-131).

    r_primal = ||colsum(x) - 1||_inf / (1 + max(||colsum(x)||_inf, 1))
    r_dual   = max_j (max_i u_ij y_i - p_j)_+ / (1 + max(||y||_inf, max_j (p_j - max_i u_ij y_i)_+))
    r_gap    = max_ij x_ij (p_j - u_ij y_i)_+ / (1 + max(||x||_inf, max_ij (p_j - u_ij y_i)_+))

with t = u.x per buyer and y = w / t (the compact state's lifted variables, for
which the reference's row-gap and |w/t - y| terms are identically zero).
The maxima are computed on the device (engine.PdhcgEngine residual kernels)
against the ORIGINAL (un-normalized) utilities, as the reference does.
"""

from dataclasses import dataclass


@dataclass
class Residuals:
    r_primal: float
    r_dual: float
    r_gap: float
    rel_kkt: float

    def as_dict(self):
        return {"r_primal": self.r_primal, "r_dual": self.r_dual,
                "r_gap": self.r_gap, "rel_kkt": self.rel_kkt}


def _engine_for(inst, x, p=None):
    import numpy as np

    from .device import DeviceMarket
    from .engine import PdhcgEngine

    dm = DeviceMarket.from_instance(inst)
    eng = PdhcgEngine(dm)
    pp = np.zeros(dm.m) if p is None else np.asarray(p, dtype=np.float64)
    eng.load_state(np.asarray(x, dtype=np.float64), pp)
    return eng


def residuals_compact(inst, x, p):
    """Relative KKT residuals of a compact state (x, p) on `inst`.
    Raises ValueError if some buyer has zero utility (kkt.py:83-86)."""
    return _engine_for(inst, x, p).residuals_pair()[0]


def eg_objective(inst, x):
    """-sum_i w_i log(u_i . x_i); +inf if some buyer has zero utility."""
    return _engine_for(inst, x).final_payload()["objective"]
