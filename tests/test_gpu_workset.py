"""Screened row solves (working sets) against the unscreened
fused kernel: the certificate only skips entries the prox keeps at zero, so
both paths give the same active sets and the same iterate up to the rounding
of the row sums (different lane groupings), and the same solve."""

import numpy as np
import pytest

from conftest import golden
from _helpers import instance_from

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _pair(gen_kw, steps=(0.05, 0.05)):
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.generate import generate_rows

    d = generate_rows(**gen_kw)
    engs = []
    for ws in (True, False):
        dm = DeviceMarket(d["row_ptr"], d["col"], d["u"], d["w"], d["m"])
        e = PdhcgEngine(dm, working_set=ws)
        e.initial_state()
        e.set_steps(*steps)
        engs.append(e)
    assert engs[0].working_set and not engs[1].working_set
    return engs


@pytest.mark.parametrize("gen_kw", [
    dict(n=40_000, m=4_000, q=0.025, seed=5),                       # ~100 entries per row
    dict(n=60_000, m=8_000, powerlaw=2.0, mean_degree=40.0, seed=2),  # short, medium, long rows
])
def test_screened_iterate_equals_unscreened(gen_kw):
    import torch

    ws, full = _pair(gen_kw)
    for chunk in (1, 1, 8, 40, 40, 40):
        ws.run_chunk(chunk)
        full.run_chunk(chunk)
        torch.cuda.synchronize()
        xa, xb = ws.x.cpu().numpy(), full.x.cpu().numpy()
        pa, pb = ws.p.cpu().numpy(), full.p.cpu().numpy()
        assert np.array_equal(xa > 0, xb > 0)                  # identical active sets
        assert np.max(np.abs(xa - xb)) <= 1e-12 * max(1.0, np.max(np.abs(xb)))
        assert np.max(np.abs(pa - pb)) <= 1e-12 * np.max(np.abs(pb))
        assert np.array_equal(ws.xflag[:ws.dm.nnz].cpu().numpy().astype(bool), xa > 0)
    # after the first iterations nearly every tile row is solved over its
    # working set (rows listed for a full solve in the last iteration)
    n_full = int(ws.blk_done[3].item())
    tile_rows = int((ws.ws_init == -1).sum().item())
    assert n_full <= 0.05 * tile_rows, (n_full, tile_rows)
    h = ws.ws_len.cpu().numpy()
    assert np.all(h[ws.ws_init.cpu().numpy() == -3] == -3)


def test_restart_and_load_invalidate_the_working_sets():
    import torch

    ws, _ = _pair(dict(n=20_000, m=2_000, q=0.05, seed=7))
    ws.run_chunk(40)
    assert int((ws.ws_len >= 0).sum().item()) > 0
    ws.restart()
    torch.cuda.synchronize()
    assert torch.equal(ws.ws_len, ws.ws_init)
    ws.run_chunk(40)
    ws.load_state(ws.x.clone(), ws.p.clone())
    assert torch.equal(ws.ws_len, ws.ws_init)


def test_working_set_slots_mirror_the_iterate():
    """Each slot holds (u, x, column, position) of its entry; the nonzero
    entries of a row with a working set are all in its slots."""
    import torch

    from paper_2506_06258_b200 import _native as nat

    ws, _ = _pair(dict(n=20_000, m=2_000, q=0.05, seed=8))
    ws.run_chunk(40)
    ws.run_chunk(3)
    torch.cuda.synchronize()
    K = nat.WS_SLOTS
    h = ws.ws_len.cpu().numpy()
    rp = ws.dm.row_ptr.cpu().numpy()
    u, x, col = ws.dm.u.cpu().numpy(), ws.x.cpu().numpy(), ws.dm.col.cpu().numpy()

    def slots(t):  # [n/32, K, 32] -> [n, K]
        a = t.cpu().numpy().reshape(-1, K, 32)
        return a.transpose(0, 2, 1).reshape(-1, K)

    su, sx, sc, sp = slots(ws.ws_u), slots(ws.ws_x), slots(ws.ws_col), slots(ws.ws_pos)
    rows = np.nonzero(h >= 0)[0]
    assert len(rows) > 0.9 * len(h)
    for i in rows[:: max(1, len(rows) // 500)]:
        k = h[i]
        pos = sp[i, :k].astype(np.int64)
        assert np.all(np.diff(pos) > 0)
        g = rp[i] + pos
        assert np.array_equal(sc[i, :k], col[g])
        assert np.array_equal(su[i, :k], u[g]) and np.array_equal(sx[i, :k], x[g])
        nz = np.nonzero(x[rp[i]:rp[i + 1]] > 0)[0]
        assert set(nz.tolist()) <= set(pos.tolist())


@pytest.mark.parametrize("name", ["solve_spec1000.npz", "solve_g200_tol0.npz",
                                  "solve_medium.npz"])
def test_solves_identical_with_and_without_working_sets(name):
    import paper_2506_06258_b200 as mq

    g = golden(name)
    inst = instance_from(g) if "indptr" in g.files else None
    if inst is None:
        inst = mq.generate_fisher(mq.GeneratorConfig(n=1000, m=400, sparsity_u=0.2, seed=0))
    cfg = dict(tol=float(g["tol"]), subproblem_tol=float(g["subtol"]))
    a = mq.run_solve(inst, mq.SolveConfig(**cfg, working_set=True), "pdhcg")
    b = mq.run_solve(inst, mq.SolveConfig(**cfg, working_set=False), "pdhcg")
    assert a.inner_iterations == b.inner_iterations == int(g["iters"])
    assert a.restarts == b.restarts == int(g["restarts"])
    assert np.max(np.abs(a.prices - b.prices) / np.abs(b.prices)) <= 1e-9


def _check_pools(eng, rows, hdr, pu, px, pc, pp, C):
    """Every valid pool mirrors (u, x, column, position) of its row in
    ascending position and holds each nonzero entry."""
    rp = eng.dm.row_ptr.cpu().numpy()
    u, x, col = eng.dm.u.cpu().numpy(), eng.x.cpu().numpy(), eng.dm.col.cpu().numpy()
    pu, px, pc, pp = (t.cpu().numpy() for t in (pu, px, pc, pp))
    for r, i in enumerate(rows):
        h = hdr[r, 0]
        if h < 0:
            continue
        pos = pp[r * C: r * C + h].astype(np.int64)
        assert np.all(np.diff(pos) > 0)
        g = rp[i] + pos
        assert np.array_equal(pc[r * C: r * C + h], col[g])
        assert np.array_equal(pu[r * C: r * C + h], u[g])
        assert np.array_equal(px[r * C: r * C + h], x[g])
        nz = np.nonzero(x[rp[i]:rp[i + 1]] > 0)[0]
        assert set(nz.tolist()) <= set(pos.tolist())


def test_long_rows_solve_over_working_set_pools():
    """Rows longer than 1024 entries (CTA per row) keep their working sets in
    pools: after the first iterations most long rows have one, the pool
    entries mirror (u, x, column, position) of the row, ascending, and hold
    every nonzero entry."""
    import torch

    from paper_2506_06258_b200 import _native as nat

    ws, _ = _pair(dict(n=60_000, m=8_000, powerlaw=2.0, mean_degree=40.0, seed=2))
    assert ws.pool and ws.dm.long_rows.numel() > 10
    ws.run_chunk(40)
    ws.run_chunk(3)
    torch.cuda.synchronize()
    hdr = ws.pl_hdr.cpu().numpy()
    assert (hdr[:, 0] >= 0).mean() > 0.8
    _check_pools(ws, ws.dm.long_rows.cpu().numpy(), hdr, ws.pl_u, ws.pl_x, ws.pl_col,
                 ws.pl_pos, nat.LONG_CAP)


def test_medium_rows_solve_over_working_set_pools():
    """Rows of 257-1024 entries (warp per row) keep their working sets in
    pools of MED_CAP entries, with the same invariants as the long rows'."""
    import torch

    from paper_2506_06258_b200 import _native as nat

    assert nat.lib().mq_med_cap() == nat.MED_CAP
    ws, _ = _pair(dict(n=60_000, m=8_000, powerlaw=2.0, mean_degree=40.0, seed=2))
    nml = int(ws.dm.struct.nmed_long)
    assert ws.mpool and nml > 100
    ws.run_chunk(40)
    ws.run_chunk(3)
    torch.cuda.synchronize()
    hdr = ws.pm_hdr.cpu().numpy()
    # rows whose certificate failed may be backing off (no pool for a few
    # iterations, ws_lvl countdown > 0)
    lv = ws.ws_lvl[ws.dm.med_rows[:nml].to(torch.int64)].cpu().numpy()
    assert hdr.shape[0] == nml and (hdr[:, 0] >= 0).mean() > 0.6
    assert np.all((hdr[:, 0] >= 0) | (hdr[:, 0] == -1) | (hdr[:, 0] == -2))
    assert np.all(hdr[lv & 31 > 0, 0] == -1)  # a row backing off has no pool
    _check_pools(ws, ws.dm.med_rows[:nml].cpu().numpy(), hdr, ws.pm_u, ws.pm_x, ws.pm_col,
                 ws.pm_pos, nat.MED_CAP)


def test_working_set_levels_move_with_failures_and_rebuilds():
    """Per-row width levels (mq_state.ws_lvl): every row starts at level 0; a
    failed certificate widens its row's set by one level (some rows climb
    over a few chunks of moving prices), levels stay in 0..3, and a rebuild
    of every set (after the host writes the iterate) narrows each row by one
    level.  The iterates are the unscreened ones (the tests above)."""
    import torch

    ws, _ = _pair(dict(n=40_000, m=4_000, q=0.025, seed=5), steps=(0.2, 0.2))
    assert int(ws.ws_lvl.max()) == 0
    for _ in range(6):
        ws.run_chunk(40)
    lv = ws.ws_lvl[:ws.dm.n].to(torch.int64)
    assert int(lv.max()) <= 3 and int((lv > 0).sum()) > 0
    before = lv.clone()
    ws.restart()  # host writes x, p: every working set is rebuilt next iteration
    ws.run_chunk(1)
    after = ws.ws_lvl[:ws.dm.n].to(torch.int64)
    # the rebuild iteration (the tile kernel) narrows every tile row one
    # level; rows it does not rebuild (over 128 entries) keep theirs
    assert bool((after <= before).all())
    assert bool((after >= (before - 1).clamp(min=0)).all())
    assert int((after < before).sum()) > 0
