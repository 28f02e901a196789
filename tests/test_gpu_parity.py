"""Parity of the CUDA path against the reference (golden fixtures produced by
running it, oracle/gen_golden.py) and against the CPU oracle, on a B200."""

import os

import numpy as np
import pytest

from conftest import golden, golden_names
from _helpers import device_ksection_chunk, instance_from, oracle_market, rel_max

pytestmark = pytest.mark.gpu

CHUNKS = golden_names("chunk_")
SOLVES = [n for n in golden_names("solve_")]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2506_06258_b200 import _build

    _build.build()


# ------------------------------------------------------------ faithful chunk

@pytest.mark.parametrize("name", CHUNKS)
def test_ksection_chunk_bit_exact_vs_reference(name):
    """mq_pdhcg_chunk == kernels.pdhcg_chunk bit for bit (x, x_prev, p,
    averages, pass counts, navg, faults)."""
    g = golden(name)
    out = device_ksection_chunk(g)
    for k in ("x", "x_prev", "p", "xbar", "pbar"):
        assert np.array_equal(out[k], g[f"out_{k}"]), f"{name}: {k} differs"
    assert np.array_equal(out["passes"], g["passes"])
    assert out["navg"] == int(g["navg_out"])
    assert out["faults"] == int(g["faults"])


def test_ksection_chunk_deterministic():
    g = golden("chunk_powerlaw400.npz")
    a = device_ksection_chunk(g)
    b = device_ksection_chunk(g)
    for k in ("x", "p", "xbar"):
        assert np.array_equal(a[k], b[k])


# ------------------------------------------------------------ fast chunk

def _engine(inst, **kw):
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine

    return PdhcgEngine(DeviceMarket.from_instance(inst), **kw)


@pytest.mark.parametrize("name", CHUNKS)
@pytest.mark.parametrize("graphs", [True, False])
def test_exact_chunk_matches_oracle(name, graphs, oracle):
    """Fast path (exact active-set prox, 2cs-cs_prev price step) vs the
    oracle's k-section at subtol=0 from the same mid-run state."""
    g = golden(name)
    inst = instance_from(g)   # golden u is already normalized (row max 1)
    eng = _engine(inst, use_graphs=graphs)
    iters = int(g["iters"])
    eng.load_full_state(g["in_x"], g["in_x_prev"], g["in_p"], g["in_xbar"], g["in_pbar"],
                        int(g["navg_in"]))
    eng.set_steps(float(g["tau"]), float(g["sigma"]))
    eng.run_chunk(iters)
    st = {k: g[f"in_{k}"].copy() for k in ("x", "x_prev", "p", "xbar", "pbar")}
    passes = np.zeros(iters, dtype=np.int64)
    oracle.pdhcg_chunk(g["indptr"], g["col"], g["u"], g["tperm"], g["tindptr"], g["w"],
                       st["x"], st["x_prev"], st["p"], st["xbar"], st["pbar"],
                       int(g["navg_in"]), float(g["tau"]), float(g["sigma"]), 32, 0.0, iters,
                       np.empty(len(g["u"])), passes)
    x = eng.x.cpu().numpy()
    scale = max(1.0, float(np.max(np.abs(st["x"]))))
    assert np.max(np.abs(x - st["x"])) <= 1e-10 * scale
    assert np.max(np.abs(eng.p.cpu().numpy() - st["p"])) <= 1e-11 * max(1.0, np.max(np.abs(st["p"])))
    assert np.max(np.abs(eng.xbar.cpu().numpy() - st["xbar"])) <= 1e-10 * scale
    assert np.max(np.abs(eng.pbar.cpu().numpy() - st["pbar"])) <= 1e-11 * max(1.0, np.max(np.abs(st["pbar"])))
    assert eng.navg == int(g["navg_in"]) + iters


# ------------------------------------------------------------ full solves

def _cfg_from(g, **kw):
    from paper_2506_06258_b200 import SolveConfig

    extra = {}
    if "restart" in g.files:
        extra = dict(restart=str(g["restart"]), restart_k=int(g["restart_k"]),
                     step_mode=str(g["step_mode"]), max_iters=int(g["max_iters"]))
    return SolveConfig(tol=float(g["tol"]), subproblem_tol=float(g["subtol"]),
                       sections=int(g["sections"]), **extra, **kw)


SMALL_SOLVES = [n for n in SOLVES if "n" in np.load(os.path.join(os.path.dirname(__file__), "golden", n)).files]


@pytest.mark.parametrize("name", SMALL_SOLVES)
@pytest.mark.parametrize("solver", ["ksection", "exact"])
def test_solve_matches_reference(name, solver):
    """run_solve on the B200 vs the reference's run_solve (golden): status,
    prices (1e-6 rel), objective (1e-8 rel); iteration counts side by side."""
    import paper_2506_06258_b200 as mq

    g = golden(name)
    inst = instance_from(g)
    rep = mq.run_solve(inst, _cfg_from(g, row_solver=solver), "pdhcg")
    ref_iters = int(g["iters"])
    print(f"{name} [{solver}]: iters {rep.inner_iterations} (ref {ref_iters}), restarts "
          f"{rep.restarts} (ref {int(g['restarts'])}), price rel {rel_max(rep.prices, g['prices']):.2e}")
    assert rep.status == str(g["status"])
    assert rep.instance_fingerprint == str(g["fingerprint"])
    assert rel_max(rep.prices, g["prices"]) <= 1e-6
    assert abs(rep.objective - float(g["objective"])) <= 1e-8 * abs(float(g["objective"]))
    # both row solvers take the reference's decisions: the exact prox differs
    # from the reference's bracket midpoint by <= the bracket width (1e-10)
    assert rep.inner_iterations == ref_iters
    assert rep.restarts == int(g["restarts"])


@pytest.mark.parametrize("name", ["solve_spec1000.npz", "solve_c1.npz"])
@pytest.mark.parametrize("solver", ["ksection", "exact"])
def test_big_solve_matches_reference(name, solver):
    """SPEC acceptance instance and BASELINE config 1 (dense 1000x500)."""
    import paper_2506_06258_b200 as mq

    g = golden(name)
    if name == "solve_c1.npz":
        U = np.random.default_rng(0).random((1000, 500))
        U[U == 0.0] = 0.5
        inst = mq.FisherInstance(mq.SparseMatrix.from_dense(U), np.ones(1000))
    else:
        inst = mq.generate_fisher(mq.GeneratorConfig(n=1000, m=400, sparsity_u=0.2, seed=0))
    assert mq.instance_fingerprint(inst) == str(g["fingerprint"])
    rep = mq.run_solve(inst, _cfg_from(g, row_solver=solver), "pdhcg")
    print(f"{name} [{solver}]: iters {rep.inner_iterations} (ref {int(g['iters'])}), restarts "
          f"{rep.restarts} (ref {int(g['restarts'])}), price rel {rel_max(rep.prices, g['prices']):.2e}, "
          f"obj {rep.objective!r} (ref {float(g['objective'])!r}), "
          f"{rep.device_stats['iters_per_second']:.0f} it/s")
    assert rep.status == "optimal"
    assert rel_max(rep.prices, g["prices"]) <= 1e-6
    assert abs(rep.objective - float(g["objective"])) <= 1e-8 * abs(float(g["objective"]))
    assert rep.inner_iterations == int(g["iters"])
    assert rep.restarts == int(g["restarts"])


def test_solve_deterministic(small_random_fisher):
    import paper_2506_06258_b200 as mq

    a = mq.run_solve(small_random_fisher, mq.SolveConfig(tol=1e-7), "pdhcg")
    b = mq.run_solve(small_random_fisher, mq.SolveConfig(tol=1e-7), "pdhcg")
    assert np.array_equal(a.prices, b.prices) and np.array_equal(a.allocation, b.allocation)
    assert a.residual_history == b.residual_history


# ------------------------------------------------------------ residuals

def test_residuals_match_reference():
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine

    g = golden("resid.npz")
    inst = instance_from(g)
    eng = PdhcgEngine(DeviceMarket.from_instance(inst))
    for x, p, r, obj in zip(g["x"], g["p"], g["r"], g["objective"]):
        eng.load_state(x, p)
        got = eng.residuals_pair()[0]
        assert np.allclose([got.r_primal, got.r_dual, got.r_gap, got.rel_kkt], r, rtol=1e-12,
                           atol=0)
        assert abs(eng.final_payload()["objective"] - obj) <= 1e-12 * abs(obj)
    # public API
    res = mq.residuals_compact(inst, g["x"][0], g["p"][0])
    assert abs(res.rel_kkt - g["r"][0][3]) <= 1e-12 * g["r"][0][3]


def test_zero_utility_state_raises(tiny_fisher):
    import paper_2506_06258_b200 as mq

    x = np.array([0.0, 0.0, 1.0, 0.0, 0.5, 0.5])
    with pytest.raises(ValueError, match="buyer 0 has zero utility"):
        mq.residuals_compact(tiny_fisher, x, np.ones(2))


# ------------------------------------------------------------ known answers

def test_analytic_single_good():
    import paper_2506_06258_b200 as mq

    w = np.array([0.3, 1.2, 0.5, 2.0])
    u = mq.SparseMatrix.from_triplets(4, 1, np.arange(4), np.zeros(4, dtype=np.int64),
                                      np.array([1.0, 0.5, 2.0, 0.7]))
    rep = mq.run_solve(mq.FisherInstance(u, w), mq.SolveConfig(tol=1e-9), "pdhcg")
    assert abs(rep.prices[0] - w.sum()) <= 1e-6 * w.sum()
    assert np.allclose(rep.allocation, w / w.sum(), atol=1e-6)


def test_analytic_uniform_utility():
    import paper_2506_06258_b200 as mq

    w = np.array([0.4, 0.7, 0.9, 1.5])
    inst = mq.FisherInstance(mq.SparseMatrix.from_dense(np.full((4, 3), 2.5)), w)
    rep = mq.run_solve(inst, mq.SolveConfig(tol=1e-9), "pdhcg")
    assert np.allclose(rep.prices, w.sum() / 3, rtol=1e-6)
    assert rep.final_residuals.rel_kkt <= 1e-9


def test_analytic_single_buyer():
    import paper_2506_06258_b200 as mq

    uu = np.array([0.2, 0.9, 0.4])
    inst = mq.FisherInstance(mq.SparseMatrix.from_dense(uu[None, :]), np.array([1.7]))
    rep = mq.run_solve(inst, mq.SolveConfig(tol=1e-9), "pdhcg")
    assert np.allclose(rep.prices, 1.7 * uu / uu.sum(), rtol=1e-6)
    assert np.allclose(rep.allocation, 1.0, atol=1e-6)


# ------------------------------------------------------------ exchange

@pytest.mark.parametrize("name", ["exchange.npz", "exchange_converged.npz"])
@pytest.mark.parametrize("solver", ["exact", "ksection"])
def test_exchange_matches_reference(name, solver):
    """solve_exchange (exchange.py:104-156) against the reference's own trace:
    the usual inner-failure case and a case the reference's loop converges
    on (outer count, every budget gap, final prices and budgets)."""
    import paper_2506_06258_b200 as mq

    g = golden(name)
    U = mq.SparseMatrix(int(g["n"]), int(g["m"]), g["u_indptr"], g["u_col"], g["u"])
    E = mq.SparseMatrix(int(g["n"]), int(g["m"]), g["e_indptr"], g["e_col"], g["e"])
    tr = mq.solve_exchange(mq.ExchangeInstance(U, E), outer_tol=1e-6,
                           inner_config=mq.SolveConfig(row_solver=solver))
    print(f"{name} [{solver}]: {tr.status} outer={tr.outer_iterations} (ref {str(g['status'])} "
          f"{int(g['outer'])}), inner {[r.inner_iterations for r in tr.inner_reports]} "
          f"(ref {list(g['inner_iters'])})")
    assert tr.status == str(g["status"])
    assert tr.outer_iterations == int(g["outer"])
    assert [r.inner_iterations for r in tr.inner_reports] == list(g["inner_iters"])
    assert np.allclose(tr.budget_gaps, g["gaps"], rtol=1e-5, atol=1e-12)
    if tr.status == "converged":
        assert rel_max(tr.final_prices, g["final_prices"]) <= 1e-6
        assert np.allclose(tr.budgets_history[-1], g["final_budgets"], rtol=1e-6, atol=1e-12)


# ------------------------------------------------------------ C2 lockstep

def test_c2_first_chunk_bit_exact():
    """BASELINE config 2 (100k x 10k, 1%): the first 40 iterations of the
    faithful chunk reproduce the reference's prices and allocation hash."""
    import hashlib

    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine

    g = golden("c2_lockstep.npz")
    inst = mq.generate_fisher(mq.GeneratorConfig(n=100_000, m=10_000, sparsity_u=0.01, seed=0))
    assert mq.instance_fingerprint(inst) == str(g["fingerprint"])
    for tag, subtol in (("default", 1e-10), ("tol0", 0.0)):
        eng = PdhcgEngine(DeviceMarket.from_instance(inst), row_solver="ksection",
                          subproblem_tol=subtol)
        eng.initial_state(w_sum=float(np.sum(inst.budgets)))
        eng.set_steps(float(g["tau"]), float(g["tau"]))
        passes = eng.run_chunk(40)
        assert np.array_equal(eng.p.cpu().numpy(), g[f"{tag}_p"])
        assert list(passes) == list(g[f"{tag}_passes"])
        assert hashlib.sha256(eng.x.cpu().numpy().tobytes()).hexdigest() == str(g[f"{tag}_x_sha"])
