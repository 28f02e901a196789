"""The fast path's sparse-iterate machinery on the device:
flags, exact dense x, running sums, fixed-point column sums, fault path."""

import numpy as np
import pytest

from conftest import golden
from _helpers import instance_from

pytestmark = pytest.mark.gpu


def _engine(inst, **kw):
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine

    return PdhcgEngine(DeviceMarket.from_instance(inst), **kw)


def _session(name):
    inst = instance_from(golden(name))
    eng = _engine(inst)
    eng.initial_state()
    eng.set_steps(0.05, 0.05)
    return inst, eng


@pytest.mark.parametrize("name", ["solve_medium.npz", "solve_g200_tol0.npz"])
def test_flags_match_the_iterate_and_x_stays_exact(name):
    import torch

    _, eng = _session(name)
    for _ in range(3):
        eng.run_chunk(40)
    torch.cuda.synchronize()
    x = eng.x.cpu().numpy()
    flags = eng.xflag[:eng.dm.nnz].cpu().numpy()
    assert np.all(x >= 0.0)
    assert np.array_equal(flags.astype(bool), x > 0.0)
    assert 0 < flags.sum() < len(flags)          # sparse, not empty


def test_running_sum_is_the_running_average():
    import torch

    _, eng = _session("solve_medium.npz")
    eng.run_chunk(40)
    xs = [eng.x.cpu().numpy().copy()]
    for _ in range(6):  # 1-iteration chunks: the average is re-materialized each time
        eng.run_chunk(1)
        xs.append(eng.x.cpu().numpy().copy())
    torch.cuda.synchronize()
    assert eng.navg == 46
    xbar = eng.xbar.cpu().numpy()
    xsum = eng.xsum.cpu().numpy()
    assert np.allclose(xbar, xsum / eng.navg, rtol=1e-15, atol=0.0)
    # the last 6 iterates enter the average with weight 1/46 each
    tail = (xsum - np.sum(xs[1:], axis=0))
    assert np.all(tail >= -1e-12)


def test_fixed_point_column_sums_match_fp64():
    import torch

    _, eng = _session("solve_g200_tol0.npz")
    eng.run_chunk(40)
    ref = torch.zeros_like(eng.cs)
    eng.colsum(eng.x, ref)
    torch.cuda.synchronize()
    cs, r = eng.cs.cpu().numpy(), ref.cpu().numpy()
    assert np.max(np.abs(cs - r)) <= 1e-11 * max(1.0, np.max(np.abs(r)))
    assert not np.any(eng.bucket.view(torch.int64).cpu().numpy())  # zeroed after use


def test_fixed_point_range_overflow_is_its_own_error():
    from paper_2506_06258_b200.errors import FixedPointRangeError

    _, eng = _session("solve_medium.npz")
    eng.dm.struct.cs_xmax = 1e-12  # every nonzero x is now out of range
    with pytest.raises(FixedPointRangeError, match="cs_xmax"):
        eng.run_chunk(1)


def test_restart_resets_the_running_sum():
    import torch

    _, eng = _session("solve_medium.npz")
    eng.run_chunk(40)
    eng.restart()
    torch.cuda.synchronize()
    assert eng.navg == 0 and not np.any(eng.xsum.cpu().numpy())
    assert np.all(eng.xflag[:eng.dm.nnz].cpu().numpy() == 1)
    eng.run_chunk(40)
    assert np.allclose(eng.xbar.cpu().numpy(), eng.xsum.cpu().numpy() / 40, rtol=1e-15)


def test_fused_residual_pair_is_bitwise_the_two_passes():
    """mq_resid_rows_pair (one sweep for the last and the averaged iterate)
    against the two separate mq_resid_rows passes, mid-solve on a generated
    market with medium and long rows (the latter a CTA each in both):
    identical residuals and column maxima.  The
    fused sweep runs before x̄ is formed (it reads xsum / navg), the separate
    passes after: the lazy average is bit for bit the formed one."""
    import torch

    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.generate import generate_rows

    d = generate_rows(30_000, 3_000, seed=6, powerlaw=2.0, mean_degree=40.0)
    eng = PdhcgEngine(DeviceMarket(d["row_ptr"], d["col"], d["u"], d["w"], d["m"]))
    eng.initial_state()
    eng.set_steps(0.05, 0.05)
    for _ in range(3):
        eng.run_chunk(40)
    assert eng._xbar_stale
    fused = eng.residuals_pair()
    assert eng._xbar_stale
    out_f, cb_f = eng.out.clone(), eng.colbest.clone()
    eng._rows(eng.x, eng.p, 0, 0)
    eng._cols(eng.cs, eng.p, 0)
    eng._rows(eng.xbar, eng.pbar, 0, 1)
    eng._cols(eng.csbar, eng.pbar, 1)
    torch.cuda.synchronize()
    v = eng.out.cpu().numpy()
    sep = (eng._assemble(v[0:16]), eng._assemble(v[16:32]))
    assert fused == sep
    assert torch.equal(out_f, eng.out) and torch.equal(cb_f, eng.colbest)
