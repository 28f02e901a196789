"""The CPU oracle is pinned to the reference: every golden vector the
reference produced (oracle/gen_golden.py) must be reproduced bit for bit."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_names
from _helpers import instance_from, oracle_market


@pytest.mark.parametrize("name", golden_names("chunk_"))
def test_oracle_chunk_bit_exact(name, oracle):
    g = golden(name)
    st = {k: g[f"in_{k}"].copy() for k in ("x", "x_prev", "p", "xbar", "pbar")}
    passes = np.zeros(int(g["iters"]), dtype=np.int64)
    navg, faults = oracle.pdhcg_chunk(g["indptr"], g["col"], g["u"], g["tperm"], g["tindptr"],
                                      g["w"], st["x"], st["x_prev"], st["p"], st["xbar"],
                                      st["pbar"], int(g["navg_in"]), float(g["tau"]),
                                      float(g["sigma"]), int(g["sections"]), float(g["subtol"]),
                                      int(g["iters"]), np.empty(len(g["u"])), passes)
    for k in st:
        assert np.array_equal(st[k], g[f"out_{k}"]), k
    assert np.array_equal(passes, g["passes"])
    assert navg == int(g["navg_out"]) and faults == int(g["faults"])


def test_oracle_chunk_thread_invariant(oracle):
    g = golden("chunk_powerlaw400.npz")
    outs = []
    for threads in (1, 3, 8):
        oracle.set_threads(threads)
        st = {k: g[f"in_{k}"].copy() for k in ("x", "x_prev", "p", "xbar", "pbar")}
        oracle.pdhcg_chunk(g["indptr"], g["col"], g["u"], g["tperm"], g["tindptr"], g["w"],
                           st["x"], st["x_prev"], st["p"], st["xbar"], st["pbar"],
                           int(g["navg_in"]), float(g["tau"]), float(g["sigma"]), 32, 1e-10,
                           int(g["iters"]), np.empty(len(g["u"])),
                           np.zeros(int(g["iters"]), dtype=np.int64))
        outs.append(st)
    oracle.set_threads(os.cpu_count() or 1)
    for st in outs[1:]:
        for k in st:
            assert np.array_equal(st[k], outs[0][k])


def test_oracle_row_root_bit_exact(oracle):
    g = golden("rowroot.npz")
    ptr = g["ptr"]
    for r in range(len(ptr) - 1):
        u = g["u"][ptr[r]:ptr[r + 1]]
        c = g["c"][ptr[r]:ptr[r + 1]]
        tw, s0, sec, tol = g["meta"][r]
        s, npass = oracle.row_root(u, c, tw, s0, int(sec), tol)
        assert s == g["s"][r] and npass == g["passes"][r], r


def test_spec_sqrt2_row(oracle):
    # u=[1,1], w=1, tau=1, p=[1,1], x^k=[1,1] -> s = sqrt(2)
    s, _ = oracle.row_root(np.ones(2), np.zeros(2), 1.0, 2.0, 32, 1e-12)
    assert abs(s - np.sqrt(2.0)) < 1e-11


def _oracle_solve_kwargs(g):
    kw = dict(tol=float(g["tol"]), sections=int(g["sections"]), subtol=float(g["subtol"]))
    if "restart" in g.files:
        kw.update(restart=str(g["restart"]), restart_k=int(g["restart_k"]),
                  step_mode=str(g["step_mode"]), max_iters=int(g["max_iters"]))
    return kw


SMALL = [n for n in golden_names("solve_") if "n" in np.load(os.path.join(GOLDEN, n)).files]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_solve_bit_exact(name, oracle):
    g = golden(name)
    inst = instance_from(g)
    o = oracle.solve(oracle_market(inst), **_oracle_solve_kwargs(g))
    assert o["status"] == str(g["status"])
    assert o["inner_iterations"] == int(g["iters"]) and o["restarts"] == int(g["restarts"])
    assert np.array_equal(o["prices"], g["prices"])
    assert np.array_equal(o["allocation"], g["allocation"])
    assert np.array_equal(np.asarray(o["residual_history"]), g["history"])
    assert np.array_equal(np.asarray(o["final_residuals"]), g["final"])
    assert np.array_equal(np.asarray(o["subproblem_passes"]), g["passes"])
    assert o["objective"] == float(g["objective"])


@pytest.mark.parametrize("name", golden_names("pdhg_"))
def test_oracle_lifted_pdhg_bit_exact(name, oracle):
    """Lifted PDHG (kernels.py:146-197, driver.py:184-268): the oracle's
    restatement reproduces the reference's solve bit for bit."""
    g = golden(name)
    inst = instance_from(g)
    o = oracle.solve_lifted(oracle_market(inst), tol=float(g["tol"]),
                            max_iters=int(g["max_iters"]), restart=str(g["restart"]),
                            restart_k=int(g["restart_k"]), step_mode=str(g["step_mode"]))
    assert o["status"] == str(g["status"])
    assert o["inner_iterations"] == int(g["iters"]) and o["restarts"] == int(g["restarts"])
    for k in ("prices", "allocation", "utility_values", "dual_values"):
        assert np.array_equal(o[k], g[k]), k
    assert np.array_equal(np.asarray(o["residual_history"]), g["history"])
    assert np.array_equal(np.asarray(o["final_residuals"]), g["final"])
    assert o["objective"] == float(g["objective"])


@pytest.mark.slow
def test_oracle_solve_spec1000(oracle):
    import paper_2506_06258_b200 as mq

    g = golden("solve_spec1000.npz")
    inst = mq.generate_fisher(mq.GeneratorConfig(n=1000, m=400, sparsity_u=0.2, seed=0))
    o = oracle.solve(oracle_market(inst), **_oracle_solve_kwargs(g))
    assert o["inner_iterations"] == int(g["iters"])
    assert np.array_equal(o["prices"], g["prices"])


def test_oracle_residuals_bit_exact(oracle):
    g = golden("resid.npz")
    mk = oracle_market(instance_from(g))
    for x, p, r, obj in zip(g["x"], g["p"], g["r"], g["objective"]):
        assert np.array_equal(np.asarray(oracle.residuals_compact(mk, x, p)), r)
        assert oracle.eg_objective(mk, x) == obj


@pytest.mark.parametrize("name", ["exchange.npz", "exchange_converged.npz"])
def test_oracle_exchange_matches_reference(oracle, name):
    g = golden(name)
    U = oracle.Market(int(g["n"]), int(g["m"]), g["u_indptr"], g["u_col"], g["u"],
                      np.ones(int(g["n"])))
    E = oracle.Market(int(g["n"]), int(g["m"]), g["e_indptr"], g["e_col"], g["e"],
                      np.ones(int(g["n"])))
    o = oracle.solve_exchange(U, E, outer_tol=1e-6)
    assert o["status"] == str(g["status"]) and o["outer_iterations"] == int(g["outer"])
    assert np.array_equal(o["budget_gaps"], g["gaps"])
    assert np.array_equal(o["final_prices"], g["final_prices"])


def test_generator_fingerprints_match_reference():
    """The package's host generator reproduces the reference's instances."""
    import paper_2506_06258_b200 as mq

    fps = json.load(open(os.path.join(GOLDEN, "gen.json")))
    checked = 0
    for key, rec in fps.items():
        parts = key.split(":")
        if parts[0] == "fisher":
            n, m, q, seed = int(parts[1]), int(parts[2]), float(parts[3]), int(parts[4])
            if n * m > 5_000_000:
                continue
            inst = mq.generate_fisher(mq.GeneratorConfig(n=n, m=m, sparsity_u=q, seed=seed))
        else:
            n, m, q, qe, seed = (int(parts[1]), int(parts[2]), float(parts[3]),
                                 float(parts[4]), int(parts[5]))
            inst = mq.generate_exchange(mq.GeneratorConfig(n=n, m=m, sparsity_u=q,
                                                           sparsity_e=qe, seed=seed))
        assert mq.instance_fingerprint(inst) == rec["fingerprint"], key
        checked += 1
    assert checked >= 6


def test_generator_math_matches_libm():
    """The bit-specified log / exp of the generator (restated from
    csrc/mq_genmath.cuh) agree with libm to an ulp or two."""
    import math

    from oracle import gen as hg

    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.random(2000), 10.0 ** rng.uniform(-300, 300, 2000)])
    for x in xs:
        assert abs(hg.gm_log(x) - math.log(x)) <= 4e-16 * max(1.0, abs(math.log(x)))
    for y in rng.uniform(-700, 700, 2000):
        assert abs(hg.gm_exp(y) / math.exp(y) - 1.0) <= 4e-16


def test_host_generator_independent_of_threads_and_slicing():
    from oracle import gen as hg

    a = hg.generate_rows(20_000, 3_000, seed=3, q=0.01, threads=1)
    b = hg.generate_rows(20_000, 3_000, seed=3, q=0.01, threads=7)
    for k in ("row_ptr", "col", "u", "w"):
        assert np.array_equal(a[k], b[k])
    part = hg.generate_rows(20_000, 3_000, seed=3, q=0.01, row0=7_000, nrows=5_000)
    rp = a["row_ptr"]
    lo, hi = rp[7_000], rp[12_000]
    assert np.array_equal(part["row_ptr"], rp[7_000:12_001] - lo)
    assert np.array_equal(part["col"], a["col"][lo:hi])
    assert np.array_equal(part["u"], a["u"][lo:hi])
    # valid support: ascending columns, values in (0, 1], ~1% density
    deg = np.diff(rp)
    assert deg.min() >= 1 and abs(deg.mean() - 30.0) < 1.0
    starts = rp[:-1]
    d = np.diff(a["col"].astype(np.int64))
    inner = np.ones(len(d), dtype=bool)
    inner[starts[1:] - 1] = False
    assert (d[inner] > 0).all()
    assert 0.0 < a["u"].min() and a["u"].max() <= 1.0


def test_host_powerlaw_generator_is_heavy_tailed():
    from oracle import gen as hg

    d = hg.generate_rows(200_000, 50_000, seed=0, powerlaw=2.0, mean_degree=100.0)
    deg = np.diff(d["row_ptr"])
    assert 85 < deg.mean() < 115 and deg.max() > 10_000 and np.median(deg) < 40
