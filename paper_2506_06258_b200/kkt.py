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


# ------------------------------------------------------------ theory diagnostics
def _dev(a, dm, dtype=None):
    import numpy as np
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dm.device)


def scaled_kkt_residual(inst, x, t, p, y, xi=1.0):
    """Euclidean norm of the stacked scaled KKT residual (kkt.py:88-111):
    t_i y_i - w_i, x_ij - [x_ij - (p_j - u_ij y_i)/xi]_+, [p_j - u_ij y_i]_-,
    colsum(x) - 1 and t_i - u_i.x_i, computed on the device."""
    import math

    import torch

    from . import _native as nat
    from .device import DeviceMarket
    from .engine import _cur_stream

    if xi <= 0:
        raise ValueError("xi must be positive")
    dm = DeviceMarket.from_instance(inst)
    xd, td, pd, yd = (_dev(a, dm) for a in (x, t, p, y))
    out = torch.zeros(4, dtype=torch.float64, device=dm.device)
    scratch = torch.zeros(int(dm.lib.mq_scratch_doubles()), dtype=torch.float64,
                          device=dm.device)
    nat.check(dm.lib.mq_scaled_kkt_rows(dm.struct, nat.ptr(xd), nat.ptr(td), nat.ptr(pd),
                                        nat.ptr(yd), float(xi), nat.ptr(out), nat.ptr(scratch),
                                        _cur_stream()), "mq_scaled_kkt_rows")
    cs = torch.zeros(dm.m, dtype=torch.float64, device=dm.device)
    nat.check(dm.lib.mq_colsum(dm.struct, nat.ptr(xd), nat.ptr(cs), _cur_stream()), "mq_colsum")
    bud, comp, viol, link = (float(v) for v in out.cpu().numpy())
    col = float(((cs - 1.0) ** 2).sum().item())
    return float(math.sqrt(bud + comp + viol + col + link))  # kkt.py:106-111 order


def scaled_kkt_residual_compact(inst, x, p, xi=1.0):
    """Scaled KKT residual of a compact state via t = u.x, y = w/t
    (kkt.py:114-121)."""
    import numpy as np

    ux = inst.utilities.row_sums(inst.utilities.values * np.asarray(x, dtype=np.float64))
    if np.any(ux <= 0):
        raise ValueError("compact state has a zero-utility buyer")
    return scaled_kkt_residual(inst, x, ux, p, inst.budgets / ux, xi)


def smoothed_gap(inst, z, center, xi=1.0, sections=32, subtol=1e-12):
    """Smoothed duality gap of z = (x, p) centered at (x_c, p_c)
    (kkt.py:134-168).  The price maximization is the exact quadratic; the
    allocation minimization is the exact per-buyer prox with step 1/xi, on the
    device (the reference's k-section with `sections`/`subtol` finds the same
    root to its tolerance; both arguments are accepted for compatibility)."""
    import math

    import numpy as np
    import torch

    from . import _native as nat
    from .device import DeviceMarket
    from .engine import _cur_stream

    if xi <= 0:
        raise ValueError("xi must be positive")
    x, p = (np.asarray(a, dtype=np.float64) for a in z)
    x_c, p_c = (np.asarray(a, dtype=np.float64) for a in center)
    f_x = eg_objective(inst, x)
    if not np.isfinite(f_x):
        return math.inf
    dm = DeviceMarket.from_instance(inst)
    xd, pd, xcd = (_dev(a, dm) for a in (x, p, x_c))
    cs = torch.zeros(dm.m, dtype=torch.float64, device=dm.device)
    nat.check(dm.lib.mq_colsum(dm.struct, nat.ptr(xd), nat.ptr(cs), _cur_stream()), "mq_colsum")
    r = cs.cpu().numpy() - 1.0
    best_price_part = f_x + float(np.dot(p_c, r)) + float(np.dot(r, r)) / (2.0 * xi)
    cbuf = torch.zeros(max(1, dm.nnz), dtype=torch.float64, device=dm.device)
    out = torch.zeros(1, dtype=torch.float64, device=dm.device)
    faults = torch.zeros(1, dtype=torch.int64, device=dm.device)
    scratch = torch.zeros(int(dm.lib.mq_scratch_doubles()), dtype=torch.float64,
                          device=dm.device)
    nat.check(dm.lib.mq_smoothed_gap_rows(dm.struct, nat.ptr(xcd), nat.ptr(pd), float(xi),
                                          nat.ptr(cbuf), nat.ptr(out), nat.ptr(scratch),
                                          nat.ptr(faults), _cur_stream()), "mq_smoothed_gap_rows")
    if int(faults.item()):
        from .errors import SubproblemError

        raise SubproblemError("smoothed gap: a row prox did not settle")
    return best_price_part + float(np.sum(p)) - float(out.item())


def residuals_lifted(inst, x, t, p, y):
    """Relative KKT residuals of a lifted state (x, t, p, y) on `inst`
    (kkt.py:29-76), on the device.  Raises ValueError unless every t > 0."""
    import numpy as np
    import torch

    from . import _native as nat
    from .device import DeviceMarket
    from .engine import _cur_stream
    from .lifted import LiftedEngine

    dm = DeviceMarket.from_instance(inst)
    xd, td, pd, yd = (_dev(a, dm) for a in (x, t, p, y))
    ones = torch.ones(dm.n, dtype=torch.float64, device=dm.device)  # (t, y) given as-is
    out = torch.zeros(16, dtype=torch.float64, device=dm.device)
    colbest = torch.zeros(dm.m, dtype=torch.float64, device=dm.device)
    scratch = torch.zeros(int(dm.lib.mq_scratch_doubles()), dtype=torch.float64,
                          device=dm.device)
    nat.check(dm.lib.mq_pdhg_resid_rows(dm.struct, nat.ptr(ones), nat.ptr(xd), nat.ptr(td),
                                        nat.ptr(yd), nat.ptr(pd), 0, nat.ptr(colbest),
                                        nat.ptr(out[0:10]), nat.ptr(scratch), _cur_stream()),
              "mq_pdhg_resid_rows")
    cs = torch.zeros(dm.m, dtype=torch.float64, device=dm.device)
    nat.check(dm.lib.mq_colsum(dm.struct, nat.ptr(xd), nat.ptr(cs), _cur_stream()), "mq_colsum")
    nat.check(dm.lib.mq_resid_cols(dm.m, nat.ptr(cs), nat.ptr(pd), nat.ptr(colbest),
                                   nat.ptr(out[10:16]), nat.ptr(scratch), _cur_stream()),
              "mq_resid_cols")
    return LiftedEngine._assemble(out.cpu().numpy())
