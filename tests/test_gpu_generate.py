"""Device generator and the large-config plumbing on a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def test_shards_equal_slices_of_the_full_market():
    """Row r's content does not depend on who generates it (multi-GPU)."""
    from paper_2506_06258_b200.generate import generate_rows

    full = generate_rows(20_000, 3_000, seed=3, q=0.01)
    part = generate_rows(20_000, 3_000, seed=3, q=0.01, row0=7_000, nrows=5_000)
    rp = full["row_ptr"].cpu().numpy()
    a, b = rp[7_000], rp[12_000]
    assert np.array_equal(part["row_ptr"].cpu().numpy(), rp[7_000:12_001] - a)
    assert np.array_equal(part["col"].cpu().numpy(), full["col"].cpu().numpy()[a:b])
    assert np.array_equal(part["u"].cpu().numpy(), full["u"].cpu().numpy()[a:b])
    assert np.array_equal(part["w"].cpu().numpy(), full["w"].cpu().numpy()[7_000:12_000])


def test_generated_market_is_valid_and_sane():
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.generate import generate_rows

    d = generate_rows(50_000, 5_000, seed=1, q=0.01)
    rp, col = d["row_ptr"].cpu().numpy(), d["col"].cpu().numpy()
    u, w = d["u"].cpu().numpy(), d["w"].cpu().numpy()
    inst = mq.FisherInstance(mq.SparseMatrix(50_000, 5_000, rp, col.astype(np.int64), u), w)
    assert mq.validate(inst) == []          # constructor checked sortedness / positivity
    deg = np.diff(rp)
    assert abs(deg.mean() - 50.0) < 1.0 and deg.min() >= 1
    assert 0.0 < u.min() and u.max() <= 1.0 and 0.0 < w.min()


def test_powerlaw_degrees_are_heavy_tailed():
    from paper_2506_06258_b200.generate import generate_rows

    d = generate_rows(200_000, 50_000, seed=0, powerlaw=2.0, mean_degree=100.0)
    deg = np.diff(d["row_ptr"].cpu().numpy())
    assert 85 < deg.mean() < 115
    assert deg.max() > 10_000 and np.median(deg) < 40


def test_power_law_market_solves_like_the_oracle(oracle):
    """Long rows (CTA-per-row kernel) and the long-row column sums: a skewed
    market against the oracle's k-section at subtol 0, several iterations."""
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.generate import generate_rows

    d = generate_rows(3_000, 2_500, seed=2, powerlaw=2.0, mean_degree=60.0)
    rp, col = d["row_ptr"].cpu().numpy(), d["col"].cpu().numpy()
    u, w = d["u"].cpu().numpy(), d["w"].cpu().numpy()
    counts = np.bincount(col, minlength=2_500)
    if np.any(counts == 0):
        pytest.skip("empty column in this draw")
    assert np.diff(rp).max() > 1024       # exercises the long-row path
    dm = DeviceMarket(rp, col, u, w, 2_500)
    eng = PdhcgEngine(dm)
    eng.initial_state(w_sum=float(w.sum()))
    eng.set_steps(0.05, 0.05)
    x0 = eng.x.cpu().numpy().copy()
    p0 = eng.p.cpu().numpy().copy()
    eng.run_chunk(5)
    mk = oracle.Market(3_000, 2_500, rp, col, u, w)
    nm, _ = oracle.normalize(mk)
    tperm, tind = oracle.transpose_schedule(nm)
    x, xp, p, xb, pb = x0.copy(), x0.copy(), p0.copy(), x0.copy(), p0.copy()
    oracle.pdhcg_chunk(nm.indptr, nm.col, nm.val, tperm, tind, nm.w, x, xp, p, xb, pb, 0, 0.05,
                       0.05, 32, 0.0, 5, np.empty(nm.nnz), np.zeros(5, dtype=np.int64))
    assert np.max(np.abs(eng.x.cpu().numpy() - x)) <= 1e-10 * max(1.0, np.abs(x).max())
    assert np.max(np.abs(eng.p.cpu().numpy() - p)) <= 1e-11 * max(1.0, np.abs(p).max())
    assert np.max(np.abs(eng.xbar.cpu().numpy() - xb)) <= 1e-10 * max(1.0, np.abs(xb).max())


@pytest.mark.parametrize("seed", [0, 1])
def test_every_row_class_matches_the_oracle(oracle, seed):
    """Register rows (<= 128 entries), medium rows (warp per row), long rows
    held in shared memory and long rows past the shared-memory cap (c in the
    x slots), interleaved in one market, against the oracle's k-section at
    subtol 0 over several iterations."""
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine

    rng = np.random.default_rng(seed)
    m = 12_000
    lens = np.concatenate([rng.integers(1, 101, 300), rng.integers(129, 1025, 60),
                           rng.integers(1025, 5001, 20),
                           [1_535, 1_536, 1_537, 3_071, 3_072, 3_073, 5_119, 5_120, 5_121, 6_000, 10_239, 10_240,
                            10_241, 11_500, m]])
    rng.shuffle(lens)
    n = lens.size
    rows = [np.sort(rng.choice(m, size=int(k), replace=False)) for k in lens]
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum(lens)
    col = np.concatenate(rows).astype(np.int32)
    u = rng.random(col.size)
    u[u == 0.0] = 0.5
    w = rng.random(n) + 0.01
    dm = DeviceMarket(rp, col, u, w, m)
    reg_row = int(dm.lib.mq_reg_row())
    assert dm.long_rows.numel() == 35
    assert dm.med_rows.numel() == int(np.sum((lens > reg_row) & (lens <= 1024)))
    eng = PdhcgEngine(dm)
    eng.initial_state(w_sum=float(w.sum()))
    eng.set_steps(0.05, 0.05)
    x0 = eng.x.cpu().numpy().copy()
    p0 = eng.p.cpu().numpy().copy()
    eng.run_chunk(6)
    mk = oracle.Market(n, m, rp, col, u, w)
    nm, _ = oracle.normalize(mk)
    tperm, tind = oracle.transpose_schedule(nm)
    x, xp, p, xb, pb = x0.copy(), x0.copy(), p0.copy(), x0.copy(), p0.copy()
    oracle.pdhcg_chunk(nm.indptr, nm.col, nm.val, tperm, tind, nm.w, x, xp, p, xb, pb, 0, 0.05,
                       0.05, 32, 0.0, 6, np.empty(nm.nnz), np.zeros(6, dtype=np.int64))
    assert np.max(np.abs(eng.x.cpu().numpy() - x)) <= 1e-10 * max(1.0, np.abs(x).max())
    assert np.max(np.abs(eng.p.cpu().numpy() - p)) <= 1e-11 * max(1.0, np.abs(p).max())
    assert np.max(np.abs(eng.xbar.cpu().numpy() - xb)) <= 1e-10 * max(1.0, np.abs(xb).max())


@pytest.mark.parametrize("name,row0,nrows", [("c2", 0, None), ("c3", 0, 300_000),
                                             ("c3", 700_000, 300_000),
                                             ("c4", 4_000_000, 400_000), ("c5", 0, None)])
def test_host_regeneration_is_byte_identical(name, row0, nrows):
    """oracle/market_gen.c rebuilds the device market byte for byte (the CPU
    reference arm of bench.py builds its instance with it)."""
    from oracle import gen as hg
    from paper_2506_06258_b200.generate import generate_config

    d = generate_config(name, seed=0, row0=row0, nrows=nrows)
    h = hg.generate_config(name, seed=0, row0=row0, nrows=nrows)
    for k in ("row_ptr", "col", "u", "w"):
        a = d[k].cpu().numpy()
        assert a.dtype == h[k].dtype and np.array_equal(a, h[k]), (name, k)
