"""Generate tests/golden/ by running the REFERENCE itself (build container only).

    NUMBA_CACHE_DIR=/tmp/nbcache python oracle/gen_golden.py [--big]

Imports the unmodified reference package from /root/reference/pkg/src (it
cannot travel to the GPU box, so its outputs are frozen here as fixtures) and
records, for each case, the reference's own outputs.  It also re-runs the
oracle restatement (oracle/solve.py + oracle/pdhcg_oracle.c) on the same
inputs and refuses to write a fixture unless the two agree bit for bit.

Fixtures (all float64 stored exactly):
  chunk_*.npz    state -> kernels.pdhcg_chunk(iters) -> state   (kernel vectors)
  rowroot.npz    rows  -> kernels._row_root                      (row-solver vectors)
  solve_*.npz    instance -> run_solve(...) report               (full solves)
  pdhg_*.npz     instance -> run_solve(..., "pdhg") report       (lifted PDHG solves)
  theory.npz     random states -> kkt.scaled_kkt_residual(_compact), kkt.smoothed_gap
  fileio/        instance files written by fileio.save + malformed files with the
                 reference reader's errors (errors.json)
  resid.npz      random states -> kkt.residuals_compact           (residual formulas)
  exchange.npz   generate_exchange -> solve_exchange trace       (Arrow-Debreu)
  gen.json       generator fingerprints (instance_fingerprint)   (generator parity)
  c2_lockstep.npz  C2 (100k x 10k, 1%) first 40 iterations: prices, checksums
"""

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import market_eq as me  # noqa: E402
from market_eq import kernels as rk  # noqa: E402

from oracle import solve as orc  # noqa: E402


def to_mk(inst, w=None):
    u = inst.utilities
    return orc.Market(u.n_rows, u.n_cols, u.row_offsets, u.col_indices, u.values,
                      inst.budgets if w is None else w)


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.1f} kB)")


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


# ------------------------------------------------------------------ chunks

def chunk_case(name, inst, seed, iters, sections=32, subtol=1e-10, zero_rows=0,
               tau=None, sigma=None):
    """Perturbed state -> reference pdhcg_chunk -> outputs."""
    rng = np.random.default_rng(seed)
    norm, _ = me.normalize(inst)
    u = norm.utilities
    tperm, tindptr = u.transpose_schedule()
    x = rng.random(u.nnz) * 2.0 / np.maximum(1, u.column_counts()[u.col_indices])
    if zero_rows:
        for i in rng.choice(u.n_rows, size=zero_rows, replace=False):
            x[u.row_offsets[i]:u.row_offsets[i + 1]] = 0.0
    x_prev = x * (1.0 + 0.1 * rng.standard_normal(u.nnz))
    x_prev = np.maximum(x_prev, 0.0)
    p = float(np.sum(norm.budgets)) / u.n_cols * (0.5 + rng.random(u.n_cols))
    xbar = x * (0.9 + 0.2 * rng.random(u.nnz))
    pbar = p * (0.9 + 0.2 * rng.random(u.n_cols))
    navg = int(rng.integers(0, 30))
    L = np.sqrt(np.max(u.column_counts()))
    tau = 0.9 / L if tau is None else tau
    sigma = 0.9 / L if sigma is None else sigma
    state_in = dict(x=x.copy(), x_prev=x_prev.copy(), p=p.copy(), xbar=xbar.copy(),
                    pbar=pbar.copy())
    ref = {k: v.copy() for k, v in state_in.items()}
    pass_ref = np.zeros(iters, dtype=np.int64)
    navg_ref, faults_ref = rk.pdhcg_chunk(
        u.row_offsets, u.col_indices, u.values, tperm, tindptr, norm.budgets,
        ref["x"], ref["x_prev"], ref["p"], ref["xbar"], ref["pbar"], navg,
        tau, sigma, sections, subtol, iters, np.empty(u.nnz), pass_ref)
    mine = {k: v.copy() for k, v in state_in.items()}
    pass_o = np.zeros(iters, dtype=np.int64)
    navg_o, faults_o = orc.pdhcg_chunk(
        u.row_offsets, u.col_indices, u.values, tperm, tindptr, norm.budgets,
        mine["x"], mine["x_prev"], mine["p"], mine["xbar"], mine["pbar"], navg,
        tau, sigma, sections, subtol, iters, np.empty(u.nnz), pass_o)
    for k in ref:
        assert same(ref[k], mine[k]), (name, k)
    assert same(pass_ref, pass_o) and navg_ref == navg_o and faults_ref == faults_o, name
    save(f"chunk_{name}.npz",
         n=u.n_rows, m=u.n_cols, indptr=u.row_offsets, col=u.col_indices, u=u.values,
         tperm=tperm, tindptr=tindptr, w=norm.budgets,
         **{f"in_{k}": v for k, v in state_in.items()},
         **{f"out_{k}": v for k, v in ref.items()},
         navg_in=navg, navg_out=navg_ref, faults=faults_ref, passes=pass_ref,
         tau=tau, sigma=sigma, sections=sections, subtol=subtol, iters=iters)


def chunk_cases():
    tiny = me.FisherInstance(me.SparseMatrix.from_dense([[.8, .3], [.2, .9], [.5, .5]]),
                             np.array([.4, .7, .9]))
    chunk_case("tiny", tiny, 0, 5)
    g = me.generate_fisher(me.GeneratorConfig(n=300, m=100, sparsity_u=0.05, seed=7))
    chunk_case("g300", g, 1, 3)
    chunk_case("g300_zero_rows", g, 2, 2, zero_rows=20)
    chunk_case("g300_tol0", g, 3, 2, subtol=0.0)
    chunk_case("g300_bisect", g, 4, 2, sections=2)
    chunk_case("g300_sec7", g, 5, 2, sections=7, subtol=1e-12)
    # tiny budgets: the C2 failure mode (roots ~1e-6, absolute bracket tol)
    u = g.utilities
    w = np.random.default_rng(9).random(u.n_rows) * 1e-5
    chunk_case("g300_tinyw", me.FisherInstance(u, w), 6, 2)
    chunk_case("g300_tinyw_tol0", me.FisherInstance(u, w), 6, 2, subtol=0.0)
    # long rows (dense) and a power-law-ish row profile
    rng = np.random.default_rng(11)
    dense = rng.random((40, 700))
    dense[dense < 0.05] = 0.0
    chunk_case("dense40x700", me.FisherInstance(me.SparseMatrix.from_dense(dense),
                                                np.ones(40)), 7, 2)
    deg = np.minimum(1 + (rng.pareto(1.2, 400) * 3).astype(int), 250)
    rows, cols = [], []
    for i, d in enumerate(deg):
        c = np.sort(rng.choice(250, size=d, replace=False))
        rows.append(np.full(d, i)), cols.append(c)
    rows, cols = np.concatenate(rows), np.concatenate(cols)
    missing = np.setdiff1d(np.arange(250), cols)
    rows = np.concatenate([rows, rng.integers(0, 400, len(missing))])
    cols = np.concatenate([cols, missing])
    key = np.unique(rows * 1000 + cols)
    rows, cols = key // 1000, key % 1000
    pl = me.SparseMatrix.from_triplets(400, 250, rows, cols, rng.random(len(rows)) + 1e-3)
    chunk_case("powerlaw400", me.FisherInstance(pl, rng.random(400) + 1e-3), 8, 3)


# ---------------------------------------------------------------- row roots

def rowroot_cases():
    rng = np.random.default_rng(21)
    rows = []
    # SPEC:298 example: u=[1,1], w=1, tau=1, p=[1,1], x^k=[1,1] -> s = sqrt(2)
    rows.append((np.array([1.0, 1.0]), np.array([0.0, 0.0]), 1.0, 2.0, 32, 1e-10))
    # single good exact hit: c=0, u=1, tw=1 -> s=1 immediately
    rows.append((np.array([1.0]), np.array([0.0]), 1.0, 1.0, 32, 1e-10))
    for k in range(300):
        ln = int(rng.integers(1, 200))
        u = rng.random(ln) + 1e-6
        c = rng.standard_normal(ln) * 10.0 ** rng.uniform(-6, 0)
        tw = 10.0 ** rng.uniform(-9, 0)
        s0 = 0.0 if k % 7 == 0 else float(np.dot(u, np.maximum(c, 0)) * rng.uniform(0.5, 2))
        sections = [32, 2, 3, 16, 33][k % 5]
        tol = [1e-10, 0.0, 1e-12, 1e-8][k % 4]
        rows.append((u, c, tw, s0, sections, tol))
    ptr = np.cumsum([0] + [len(r[0]) for r in rows])
    U = np.concatenate([r[0] for r in rows])
    C = np.concatenate([r[1] for r in rows])
    meta = np.array([[r[2], r[3], r[4], r[5]] for r in rows])
    s_out, p_out = [], []
    for (u, c, tw, s0, sec, tol) in rows:
        s, npass = rk._row_root(0, len(u), u, c, tw, s0, sec, tol)
        so, po = orc.row_root(u, c, tw, s0, sec, tol)
        assert s == so and npass == po, (s, so, npass, po)
        s_out.append(s), p_out.append(npass)
    save("rowroot.npz", ptr=ptr, u=U, c=C, meta=meta, s=np.array(s_out),
         passes=np.array(p_out, dtype=np.int64))


# ------------------------------------------------------------------- solves

def report_arrays(rep, with_alloc=True):
    d = dict(status=rep.status, iters=rep.inner_iterations, restarts=rep.restarts,
             prices=rep.prices, utility_values=rep.utility_values,
             dual_values=rep.dual_values,
             passes=np.asarray(rep.subproblem_passes or [], dtype=np.int64),
             history=np.asarray(rep.residual_history, dtype=np.float64),
             final=np.array([rep.final_residuals.r_primal, rep.final_residuals.r_dual,
                             rep.final_residuals.r_gap, rep.final_residuals.rel_kkt]),
             fingerprint=rep.instance_fingerprint)
    if with_alloc:
        d["allocation"] = rep.allocation
    return d


def solve_case(name, inst, cfg, store_instance, with_alloc=True):
    t = time.time()
    rep = me.run_solve(inst, cfg, "pdhcg")
    t_ref = time.time() - t
    t = time.time()
    o = orc.solve(to_mk(inst), tol=cfg.tol, max_iters=cfg.max_iters,
                  sections=cfg.sections, subtol=cfg.subproblem_tol,
                  check_every=cfg.check_every, restart=cfg.restart,
                  restart_k=cfg.restart_k, step_mode=cfg.step_mode, adapt_eta=cfg.adapt_eta)
    t_orc = time.time() - t
    assert rep.inner_iterations == o["inner_iterations"] and rep.restarts == o["restarts"], name
    assert same(rep.prices, o["prices"]) and same(rep.allocation, o["allocation"]), name
    assert list(rep.residual_history) == o["residual_history"], name
    obj = me.kkt.eg_objective(inst, rep.allocation)
    assert obj == o["objective"], name
    extra = {}
    if store_instance:
        u = inst.utilities
        extra = dict(n=u.n_rows, m=u.n_cols, indptr=u.row_offsets, col=u.col_indices,
                     u=u.values, w=inst.budgets)
    save(f"solve_{name}.npz", **report_arrays(rep, with_alloc), objective=obj,
         tol=cfg.tol, subtol=cfg.subproblem_tol, sections=cfg.sections,
         restart=cfg.restart, restart_k=cfg.restart_k, step_mode=cfg.step_mode,
         max_iters=cfg.max_iters, ref_seconds=t_ref, **extra)
    print(f"  {name}: {rep.status} iters={rep.inner_iterations} restarts={rep.restarts} "
          f"obj={obj!r} ref {t_ref:.1f}s oracle {t_orc:.1f}s")
    return rep


def pdhg_case(name, inst, cfg):
    """Lifted PDHG (algo="pdhg", driver.py:184-268): the reference's report,
    written only if oracle.solve_lifted reproduces it bit for bit."""
    t = time.time()
    rep = me.run_solve(inst, cfg, "pdhg")
    t_ref = time.time() - t
    o = orc.solve_lifted(to_mk(inst), tol=cfg.tol, max_iters=cfg.max_iters,
                         check_every=cfg.check_every, restart=cfg.restart,
                         restart_k=cfg.restart_k, step_mode=cfg.step_mode,
                         adapt_eta=cfg.adapt_eta)
    assert rep.inner_iterations == o["inner_iterations"] and rep.restarts == o["restarts"], name
    assert same(rep.prices, o["prices"]) and same(rep.allocation, o["allocation"]), name
    assert same(rep.utility_values, o["utility_values"]), name
    assert same(rep.dual_values, o["dual_values"]), name
    assert list(rep.residual_history) == o["residual_history"], name
    obj = me.kkt.eg_objective(inst, rep.allocation)
    assert obj == o["objective"], name
    u = inst.utilities
    d = report_arrays(rep, True)
    d.pop("passes")
    save(f"pdhg_{name}.npz", **d, objective=obj, tol=cfg.tol, restart=cfg.restart,
         restart_k=cfg.restart_k, step_mode=cfg.step_mode, max_iters=cfg.max_iters,
         ref_seconds=t_ref, n=u.n_rows, m=u.n_cols, indptr=u.row_offsets, col=u.col_indices,
         u=u.values, w=inst.budgets)
    print(f"  pdhg {name}: {rep.status} iters={rep.inner_iterations} restarts={rep.restarts} "
          f"obj={obj!r} ref {t_ref:.1f}s")


def pdhg_cases():
    tiny = me.FisherInstance(me.SparseMatrix.from_dense([[.8, .3], [.2, .9], [.5, .5]]),
                             np.array([.4, .7, .9]))
    pdhg_case("tiny", tiny, me.SolveConfig(tol=1e-7, max_iters=100_000))
    pdhg_case("small", me.generate_fisher(me.GeneratorConfig(n=12, m=6, sparsity_u=0.5, seed=3)),
              me.SolveConfig(tol=1e-6))
    pdhg_case("medium", me.generate_fisher(me.GeneratorConfig(n=60, m=25, sparsity_u=0.3, seed=11)),
              me.SolveConfig(tol=1e-5))
    g = me.generate_fisher(me.GeneratorConfig(n=200, m=80, sparsity_u=0.2, seed=1))
    pdhg_case("g200", g, me.SolveConfig(tol=1e-4))
    g = me.generate_fisher(me.GeneratorConfig(n=80, m=30, sparsity_u=0.3, seed=5))
    pdhg_case("g80_fixed", g, me.SolveConfig(tol=1e-5, restart="fixed", restart_k=120))
    pdhg_case("g80_theory", g, me.SolveConfig(tol=1e-3, step_mode="theory", max_iters=6000))


def theory_case():
    """kkt.py:88-168 diagnostics on random states of two generated markets."""
    out = {}
    rng = np.random.default_rng(7)
    for tag, cfg in (("a", me.GeneratorConfig(n=60, m=25, sparsity_u=0.3, seed=11)),
                     ("b", me.GeneratorConfig(n=200, m=80, sparsity_u=0.2, seed=1))):
        inst = me.generate_fisher(cfg)
        u = inst.utilities
        out[f"{tag}_indptr"], out[f"{tag}_col"] = u.row_offsets, u.col_indices
        out[f"{tag}_u"], out[f"{tag}_w"] = u.values, inst.budgets
        out[f"{tag}_nm"] = np.array([u.n_rows, u.n_cols])
        for k in range(3):
            x = rng.random(u.nnz) * 0.1
            t = rng.random(u.n_rows) + 0.1
            p = rng.random(u.n_cols) + 0.05
            y = rng.random(u.n_rows) * 2.0 - 0.2
            xc = rng.random(u.nnz) * 0.1
            pc = rng.random(u.n_cols) + 0.05
            xi = [0.5, 1.0, 3.0][k]
            out[f"{tag}{k}_x"], out[f"{tag}{k}_t"], out[f"{tag}{k}_p"] = x, t, p
            out[f"{tag}{k}_y"], out[f"{tag}{k}_xc"], out[f"{tag}{k}_pc"] = y, xc, pc
            out[f"{tag}{k}_xi"] = np.float64(xi)
            out[f"{tag}{k}_skkt"] = np.float64(me.kkt.scaled_kkt_residual(inst, x, t, p, y, xi))
            out[f"{tag}{k}_skkt_c"] = np.float64(me.kkt.scaled_kkt_residual_compact(inst, x, p, xi))
            out[f"{tag}{k}_gap"] = np.float64(me.kkt.smoothed_gap(inst, (x, p), (xc, pc), xi=xi))
            print(f"  theory {tag}{k}: skkt={out[f'{tag}{k}_skkt']!r} gap={out[f'{tag}{k}_gap']!r}")
    save("theory.npz", **out)


FILEIO_BAD = {
    "bad_header.mtx": "%%MatrixMarket matrix array real general\n2 2 1\n1 1 0.5\n",
    "bad_size.mtx": "%%MatrixMarket matrix coordinate real general\n2 2\n1 1 0.5\n",
    "bad_index.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0.5\n3 1 0.5\n",
    "bad_neg.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0.5\n2 1 -0.5\n",
    "bad_count.mtx": "%%MatrixMarket matrix coordinate real general\n% c\n2 2 3\n1 1 0.5\n2 2 0.5\n",
    "bad_malformed.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0.5\n2 x 0.5\n",
    "bad_float_index.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 0.5\n2.0 1 0.5\n",
    "bad_many.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 0.5\n2 2 0.5\n",
    "bad_cols.csv": "2,2,2\n0,0,0.5\n1,0\n",
    "bad_hdr.csv": "2,2\n0,0,0.5\n",
    "bad_idx.csv": "2,2,2\n0,0,0.5\n0,2,0.5\n",
    "ok_comments.mtx": ("%%MatrixMarket matrix coordinate real general\n% hi\n2 2 2\n1 1 0.5\n"
                        "% mid\n\n2 2 0.25\n"),
}


def fileio_case():
    """Files the reference's fileio.save writes, and its reader's verdicts on
    malformed files (message, line)."""
    from market_eq import fileio as rf

    out = os.path.join(OUT, "fileio")
    os.makedirs(out, exist_ok=True)
    inst = me.generate_fisher(me.GeneratorConfig(n=30, m=12, sparsity_u=0.3, seed=4))
    ex = me.generate_exchange(me.GeneratorConfig(n=10, m=8, sparsity_u=0.4, seed=2))
    rf.save(inst, os.path.join(out, "fisher"), "mtx")
    rf.save(inst, os.path.join(out, "fisher"), "csv")
    rf.save(ex, os.path.join(out, "exch"), "mtx")
    msgs = {}
    for name, text in FILEIO_BAD.items():
        path = os.path.join(out, name)
        with open(path, "w") as fh:
            fh.write(text)
        reader = rf.read_matrix_market if name.endswith(".mtx") else rf.read_csv_triplets
        try:
            M = reader(path)
            msgs[name] = {"ok": True, "values": M.values.tolist(), "col": M.col_indices.tolist(),
                          "rows": M.row_offsets.tolist()}
        except Exception as e:  # noqa: BLE001 - record the reference's verdict
            msgs[name] = {"ok": False, "type": type(e).__name__, "line": getattr(e, "line", None),
                          "msg": str(e).replace(out + "/", "")}
    with open(os.path.join(out, "errors.json"), "w") as fh:
        json.dump(msgs, fh, indent=1)
    print(f"  fileio: {len(msgs)} reader cases")


def c1_instance():
    """BASELINE config 1: dense 1000x500, U~U(0,1) (default_rng(0)), w=1."""
    U = np.random.default_rng(0).random((1000, 500))
    U[U == 0.0] = 0.5
    return me.FisherInstance(me.SparseMatrix.from_dense(U), np.ones(1000))


def solve_cases(big):
    tiny = me.FisherInstance(me.SparseMatrix.from_dense([[.8, .3], [.2, .9], [.5, .5]]),
                             np.array([.4, .7, .9]))
    solve_case("tiny", tiny, me.SolveConfig(tol=1e-8, max_iters=100_000), True)
    norm_tiny, _ = me.normalize(tiny)
    solve_case("tiny_norm", norm_tiny, me.SolveConfig(tol=1e-9, max_iters=100_000), True)
    solve_case("small", me.generate_fisher(me.GeneratorConfig(n=12, m=6, sparsity_u=0.5, seed=3)),
               me.SolveConfig(tol=1e-6), True)
    solve_case("medium", me.generate_fisher(me.GeneratorConfig(n=60, m=25, sparsity_u=0.3, seed=11)),
               me.SolveConfig(tol=1e-6), True)
    solve_case("g200_tol0", me.generate_fisher(me.GeneratorConfig(n=200, m=80, sparsity_u=0.2, seed=1)),
               me.SolveConfig(tol=1e-5, subproblem_tol=0.0), True)
    # theory steps and fixed restarts exercise the other controller branches
    g = me.generate_fisher(me.GeneratorConfig(n=80, m=30, sparsity_u=0.3, seed=5))
    solve_case("g80_fixed", g, me.SolveConfig(tol=1e-5, restart="fixed", restart_k=120), True)
    solve_case("g80_theory", g, me.SolveConfig(tol=1e-4, step_mode="theory", max_iters=4000), True)


def big_solve_cases():
    # SPEC acceptance instance: 1000 x 400, q=0.2, seed 0
    spec = me.generate_fisher(me.GeneratorConfig(n=1000, m=400, sparsity_u=0.2, seed=0))
    solve_case("spec1000", spec, me.SolveConfig(tol=1e-4), False, with_alloc=True)
    solve_case("c1", c1_instance(), me.SolveConfig(tol=1e-4), False, with_alloc=False)


# ---------------------------------------------------------------- residuals

def resid_cases():
    inst = me.generate_fisher(me.GeneratorConfig(n=50, m=20, sparsity_u=0.3, seed=13))
    rng = np.random.default_rng(5)
    u = inst.utilities
    X, P, R = [], [], []
    for _ in range(20):
        x = rng.random(u.nnz) * rng.choice([1e-3, 1.0, 10.0])
        p = rng.random(u.n_cols) * rng.choice([0.01, 1.0])
        r = me.residuals_compact(inst, x, p)
        assert orc.residuals_compact(to_mk(inst), x, p) == (r.r_primal, r.r_dual, r.r_gap, r.rel_kkt)
        X.append(x), P.append(p), R.append([r.r_primal, r.r_dual, r.r_gap, r.rel_kkt])
    save("resid.npz", n=u.n_rows, m=u.n_cols, indptr=u.row_offsets, col=u.col_indices,
         u=u.values, w=inst.budgets, x=np.array(X), p=np.array(P), r=np.array(R),
         objective=np.array([me.kkt.eg_objective(inst, x) for x in X]))


# ----------------------------------------------------------------- exchange

def exchange_case(name="exchange.npz", n=40, m=30, qu=0.3, qe=0.5, seed=2):
    """The reference's fixed-point loop on a generated exchange instance.
    exchange.npz: inner-failure (the reference's usual outcome);
    exchange_converged.npz: an instance on which it converges
    (tools/ad_search.py: 1 of 108 generated instances)."""
    ex = me.generate_exchange(me.GeneratorConfig(n=n, m=m, sparsity_u=qu,
                                                 sparsity_e=qe, seed=seed))
    t = time.time()
    tr = me.solve_exchange(ex, outer_tol=1e-6)
    t_ref = time.time() - t
    U = ex.utilities
    E = ex.endowments
    mkU = orc.Market(U.n_rows, U.n_cols, U.row_offsets, U.col_indices, U.values,
                     np.ones(U.n_rows))
    mkE = orc.Market(E.n_rows, E.n_cols, E.row_offsets, E.col_indices, E.values,
                     np.ones(E.n_rows))
    o = orc.solve_exchange(mkU, mkE, outer_tol=1e-6)
    assert o["status"] == tr.status and o["outer_iterations"] == tr.outer_iterations
    assert same(o["budget_gaps"], tr.budget_gaps) and same(o["final_prices"], tr.final_prices)
    save(name, n=U.n_rows, m=U.n_cols,
         u_indptr=U.row_offsets, u_col=U.col_indices, u=U.values,
         e_indptr=E.row_offsets, e_col=E.col_indices, e=E.values,
         status=tr.status, outer=tr.outer_iterations, gaps=np.array(tr.budget_gaps),
         final_budgets=tr.final_budgets, final_prices=tr.final_prices,
         inner_iters=np.array([r.inner_iterations for r in tr.inner_reports]),
         ref_seconds=t_ref)
    print(f"  {name}: {tr.status} outer={tr.outer_iterations} ref {t_ref:.1f}s")


# --------------------------------------------------------------- generators

def gen_fingerprints(big):
    out = {}
    cfgs = [(12, 6, 0.5, 0.5, 3), (60, 25, 0.3, 0.5, 11), (300, 100, 0.05, 0.5, 7),
            (1000, 400, 0.2, 0.5, 0), (500, 2000, 0.001, 0.5, 4), (3, 50, 0.01, 0.01, 8)]
    if big:
        cfgs.append((100_000, 10_000, 0.01, 0.5, 0))
    for (n, m, q, qe, seed) in cfgs:
        cfg = me.GeneratorConfig(n=n, m=m, sparsity_u=q, sparsity_e=qe, seed=seed)
        f = me.generate_fisher(cfg)
        key = f"fisher:{n}:{m}:{q}:{seed}"
        out[key] = {"fingerprint": me.instance_fingerprint(f), "nnz": f.utilities.nnz}
        if n * m <= 2_000_000:
            e = me.generate_exchange(cfg)
            out[f"exchange:{n}:{m}:{q}:{qe}:{seed}"] = {
                "fingerprint": me.instance_fingerprint(e), "nnz_u": e.utilities.nnz,
                "nnz_e": e.endowments.nnz}
        print("  ", key, out[key])
    path = os.path.join(OUT, "gen.json")
    old = {}
    if os.path.exists(path):
        old = json.load(open(path))
    old.update(out)
    json.dump(old, open(path, "w"), indent=1, sort_keys=True)


# -------------------------------------------------------------- C2 lockstep

def c2_lockstep():
    """First 40 iterations of BASELINE config 2 through the reference kernel."""
    t = time.time()
    inst = me.generate_fisher(me.GeneratorConfig(n=100_000, m=10_000, sparsity_u=0.01, seed=0))
    print(f"  C2 generated in {time.time() - t:.1f}s, nnz={inst.utilities.nnz}")
    norm, _ = me.normalize(inst)
    u = norm.utilities
    tperm, tindptr = u.transpose_schedule()
    from market_eq.pdhcg import initial_compact_state
    st = initial_compact_state(norm)
    out = {}
    for subtol in (1e-10, 0.0):
        x, p = st.x.copy(), st.p.copy()
        x_prev, xbar, pbar = x.copy(), x.copy(), p.copy()
        L = orc.selector_op_norm(to_mk(norm), tperm.astype(np.int64))
        tau = sigma = 0.9 / L
        passes = np.zeros(40, dtype=np.int64)
        t = time.time()
        navg, faults = rk.pdhcg_chunk(u.row_offsets, u.col_indices, u.values, tperm, tindptr,
                                      norm.budgets, x, x_prev, p, xbar, pbar, 0, tau, sigma,
                                      32, subtol, 40, np.empty(u.nnz), passes)
        print(f"  C2 40 its subtol={subtol}: {time.time() - t:.1f}s faults={faults}")
        tag = "tol0" if subtol == 0.0 else "default"
        out[f"{tag}_p"] = p
        out[f"{tag}_pbar"] = pbar
        out[f"{tag}_passes"] = passes
        out[f"{tag}_x_sum"] = np.array([x.sum(), (x * x).sum(), xbar.sum()])
        out[f"{tag}_x_sample"] = x[:: 997]
        out[f"{tag}_x_sha"] = hashlib.sha256(x.tobytes()).hexdigest()
        out[f"{tag}_xbar_sha"] = hashlib.sha256(xbar.tobytes()).hexdigest()
        out[f"{tag}_ux"] = inst.utilities.row_sums(inst.utilities.values * x)
    out["tau"] = tau
    out["fingerprint"] = me.instance_fingerprint(inst)
    save("c2_lockstep.npz", **out)


def c2_solve():
    """BASELINE config 2 solved to 1e-4 by the reference at subproblem_tol=0
    (the default 1e-10 bracket crashes at iteration 41).
    ~2.5 h on 8 cores; the allocation (1e7 entries) is kept as a checksum, a
    strided sample and the per-buyer utilities."""
    t = time.time()
    inst = me.generate_fisher(me.GeneratorConfig(n=100_000, m=10_000, sparsity_u=0.01, seed=0))
    print(f"  C2 generated in {time.time() - t:.1f}s, nnz={inst.utilities.nnz}", flush=True)
    import logging
    logging.basicConfig(level=logging.INFO)
    cfg = me.SolveConfig(tol=1e-4, subproblem_tol=0.0)
    t = time.time()
    rep = me.run_solve(inst, cfg, "pdhcg")
    t_ref = time.time() - t
    obj = me.kkt.eg_objective(inst, rep.allocation)
    d = report_arrays(rep, with_alloc=False)
    d["allocation_sha"] = hashlib.sha256(rep.allocation.tobytes()).hexdigest()
    d["allocation_sample"] = rep.allocation[::997]
    d["allocation_sum"] = np.array([rep.allocation.sum(), (rep.allocation ** 2).sum()])
    save("solve_c2_tol0.npz", **d, objective=obj, tol=cfg.tol, subtol=cfg.subproblem_tol,
         sections=cfg.sections, max_iters=cfg.max_iters, ref_seconds=t_ref,
         threads=os.cpu_count())
    print(f"  C2 tol0: {rep.status} iters={rep.inner_iterations} restarts={rep.restarts} "
          f"obj={obj!r} ref {t_ref:.1f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also C1, SPEC-1000 and C2 cases")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    orc.set_threads(os.cpu_count())
    steps = {"chunk": chunk_cases, "rowroot": rowroot_cases, "solve": lambda: solve_cases(a.big),
             "pdhg": pdhg_cases, "theory": theory_case, "fileio": fileio_case,
             "bigsolve": big_solve_cases,
             "resid": resid_cases, "exchange": exchange_case,
             "gen": lambda: gen_fingerprints(a.big), "c2": c2_lockstep, "c2solve": c2_solve,
             "exchange_conv": lambda: exchange_case("exchange_converged.npz", 10, 6, 0.3, 1.0,
                                                    2)}
    for k, fn in steps.items():
        if a.only and k not in a.only.split(","):
            continue
        if k in ("c2", "bigsolve", "c2solve") and not a.big:
            continue
        print(f"[{k}]")
        fn()


if __name__ == "__main__":
    main()
