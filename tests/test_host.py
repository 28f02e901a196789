"""Host-side logic (no GPU): data model, controller, norm, report, C ABI."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def test_native_library_exports_every_header_symbol():
    """libmarket_eq_b200.so loads (no device needed) and exports exactly what
    include/market_eq_b200.h declares."""
    from paper_2506_06258_b200 import _build, _native

    _build.build()
    lib = _native.load_library()
    header = open(os.path.join(ROOT, "include", "market_eq_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(mq_\w+)\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_native.EXPORTED)
    for name in declared:
        assert hasattr(lib, name)
    assert lib.mq_abi_version() == 1
    assert lib.mq_scratch_doubles() > 0


def test_no_device_raises_loudly(monkeypatch):
    import torch

    from paper_2506_06258_b200 import _native

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    with pytest.raises(_native.NativeUnavailable):
        _native.lib()


def test_sparse_matrix_contract():
    from paper_2506_06258_b200 import SparseMatrix, StructureError

    m = SparseMatrix.from_triplets(2, 3, [1, 0, 0], [2, 2, 0], [3.0, 2.0, 1.0])
    assert m.row_offsets.tolist() == [0, 2, 3]
    assert m.col_indices.tolist() == [0, 2, 2]
    assert not m.values.flags.writeable
    with pytest.raises(StructureError):
        SparseMatrix(1, 2, [0, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(StructureError):
        SparseMatrix(1, 2, [0, 1], [0], [0.0])
    with pytest.raises(StructureError):
        SparseMatrix.from_triplets(1, 1, [0, 0], [0, 0], [1.0, 2.0])
    tperm, tind = m.transpose_schedule()
    assert tperm.tolist() == [0, 1, 2] and tind.tolist() == [0, 1, 1, 3]
    assert np.allclose(m.apply(np.ones(3)), [3.0, 3.0])
    assert np.allclose(m.apply_transpose(np.ones(2)), [1.0, 0.0, 5.0])


def test_validate_and_normalize():
    from paper_2506_06258_b200 import (FisherInstance, GeneratorConfig, SparseMatrix,
                                       generate_fisher, normalize, validate)

    u = SparseMatrix.from_triplets(2, 2, [0, 1], [0, 0], [1.0, 2.0])
    assert any("good 1 unvalued" in v for v in validate(FisherInstance(u, np.ones(2))))
    inst = FisherInstance(SparseMatrix.from_dense([[2.0, 4.0]]), np.array([1.0]))
    out, scales = normalize(inst)
    assert out.utilities.values.tolist() == [0.5, 1.0] and scales.tolist() == [4.0]
    g = generate_fisher(GeneratorConfig(n=6, m=4, sparsity_u=0.7, seed=5))
    once, _ = normalize(g)
    twice, s2 = normalize(once)
    assert np.array_equal(once.utilities.values, twice.utilities.values) and np.all(s2 == 1.0)


def test_selector_norm_matches_reference_construction(oracle):
    """O(m) column-count power iteration == the reference's nnz-sized
    selector power iteration (driver.py:117-121) to ~1e-15."""
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.sparse import selector_norm_from_counts

    for cfg in [(60, 25, 0.3, 11), (300, 100, 0.05, 7), (200, 80, 0.2, 1)]:
        inst = mq.generate_fisher(mq.GeneratorConfig(n=cfg[0], m=cfg[1], sparsity_u=cfg[2],
                                                     seed=cfg[3]))
        u = inst.utilities
        mk = oracle.Market(u.n_rows, u.n_cols, u.row_offsets, u.col_indices, u.values,
                           inst.budgets)
        tperm, _ = oracle.transpose_schedule(mk)
        ref = oracle.selector_op_norm(mk, tperm)
        mine = selector_norm_from_counts(u.column_counts())
        assert abs(mine - ref) <= 1e-14 * ref


def test_controller_matches_oracle(oracle):
    from paper_2506_06258_b200 import RestartParams, StepController, should_restart, update_weights

    rng = np.random.default_rng(3)
    ctrl = StepController(eta_initial=0.9 / 7.0, omega_initial=1.3, eta_max=0.95 / 7.0,
                          omega_lower=1.3 / 16, omega_upper=1.3 * 16)
    ref = oracle.Steps(0.9 / 7.0, 1.3, 0.95 / 7.0, 1.3 / 16, 1.3 * 16)
    for _ in range(50):
        pm, dm, eta = rng.random(3) * 10 ** rng.uniform(-3, 3, 3)
        update_weights(ctrl, pm, dm, eta)
        ref.update(pm, dm, eta)
        assert (ctrl.tau, ctrl.sigma) == (ref.tau, ref.sigma)
    p = RestartParams()
    for now, last, prev, inner, tot in rng.random((100, 5)) * [1, 1, 1, 100, 400]:
        assert should_restart(now, last, prev, inner, tot, p) == oracle.should_restart(
            now, last, prev, inner, tot)


def test_solve_config_validation():
    from paper_2506_06258_b200 import SolveConfig

    with pytest.raises(ValueError):
        SolveConfig(tol=0)
    with pytest.raises(ValueError):
        SolveConfig(restart="fixed")
    with pytest.raises(ValueError):
        SolveConfig(row_solver="newton")
    assert SolveConfig().as_dict()["row_solver"] == "exact"


def test_report_json_round_trip(tmp_path):
    from paper_2506_06258_b200 import Residuals, SolveReport

    rep = SolveReport(solver="pdhcg", status="optimal", inner_iterations=40, restarts=1,
                      wall_time_seconds=0.5, final_residuals=Residuals(1e-5, 2e-5, 3e-6, 2e-5),
                      residual_history=[(40, 2e-5)], prices=np.array([0.1, 1 / 3]),
                      allocation=np.array([np.pi, 1e-300]), utility_values=np.array([1.0]),
                      dual_values=np.array([2.0]), subproblem_passes=[3, 4])
    path = tmp_path / "r.json"
    rep.to_json(str(path))
    back = SolveReport.from_json(str(path))
    assert np.array_equal(back.prices, rep.prices)
    assert np.array_equal(back.allocation, rep.allocation)
    assert back.final_residuals == rep.final_residuals


def test_oracle_not_imported_by_package():
    """The shipped package never imports the test oracle."""
    pkg = os.path.join(ROOT, "paper_2506_06258_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", text, re.M), f


def test_abi_marshaling_without_device():
    """Every entry point accepts its ctypes argument list; without a GPU the
    CUDA runtime error comes back as a negative code (never a crash)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present: exercised by the gpu tests")
    from paper_2506_06258_b200 import _native as nat

    lib = nat.load_library()
    mk, st = nat.MqMarket(), nat.MqState()
    n64 = ctypes.c_int64(0)
    calls = {
        "mq_dual_step": (mk, st, 0, None),
        "mq_primal_step": (mk, st, 0, None, None),
        "mq_colsum_step": (mk, st, 0, 1, None),
        "mq_colsum_finalize": (mk, st, 0, None),
        "mq_chunk_end": (st, 1, None),
        "mq_fast_chunk": (mk, st, 1, None),
        "mq_colsum": (mk, None, None, None),
        "mq_resid_rows": (mk, None, None, 0, None, None, None, None, None, None),
        "mq_resid_cols": (0, None, None, None, None, None, None),
        "mq_restart_moves": (mk, None, None, None, None, None, None, None, None, None),
        "mq_spmv": (0, None, None, None, None, None, None),
        "mq_normalize_rows": (0, None, None, None, None, None),
        "mq_gen_degrees": (0, 1, 10, 0, 0.5, 2.0, 1.0, 1, None, None),
        "mq_gen_fill": (0, 1, 10, 0, 0.5, 2.0, 1.0, 1, None, None, None, None, None),
        "mq_pdhcg_chunk": (0, 0, None, None, None, None, None, None, None, None, None, None,
                           None, 0, 0.1, 0.1, 32, 1e-10, 1, None, None, ctypes.byref(n64), None),
    }
    for name, args in calls.items():
        rc = getattr(lib, name)(*args)
        assert rc != 0, name
        assert lib.mq_last_error()
