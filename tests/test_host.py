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
    assert lib.mq_abi_version() == 12
    # the ctypes mirrors have the C layout
    assert lib.mq_market_bytes() == ctypes.sizeof(_native.MqMarket)
    assert lib.mq_state_bytes() == ctypes.sizeof(_native.MqState)
    assert lib.mq_med_cap() == _native.MED_CAP and lib.mq_long_cap() == _native.LONG_CAP
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
        "mq_resid_rows": (mk, None, None, 0, None, None, None, None, None, None, None),
        "mq_resid_cols": (0, None, None, None, None, None, None),
        "mq_restart_moves": (mk, None, None, None, None, None, None, None, None, None),
        "mq_spmv": (0, None, None, None, None, None, None),
        "mq_normalize_rows": (0, None, None, None, None, None),
        "mq_gen_degrees": (0, 1, 10, 0, 0.5, 2.0, 1.0, 1, None, None),
        "mq_tile_entries": (),
        "mq_reg_row": (),
        "mq_colsum_mode": (),
        "mq_fixed_colsum": (),
        "mq_x_sparse": (),
        "mq_avg_materialize": (mk, st, None),
        "mq_gen_fill": (0, 1, 10, 0, 0.5, 2.0, 1.0, 1, None, None, None, None, None),
        "mq_pdhcg_chunk": (0, 0, None, None, None, None, None, None, None, None, None, None,
                           None, 0, 0.1, 0.1, 32, 1e-10, 1, None, None, ctypes.byref(n64), None),
    }
    for name, args in calls.items():
        rc = getattr(lib, name)(*args)
        if name == "mq_colsum_mode":
            assert rc in (0, 1, 2, 3, 4, 5)
            continue
        if name in ("mq_fixed_colsum", "mq_x_sparse"):
            assert rc >= 0
            continue
        assert rc != 0, name
        if name in ("mq_tile_entries", "mq_reg_row"):
            continue
        assert lib.mq_last_error()


def _random_csr(rng, n, m, lens):
    rows = [np.sort(rng.choice(m, size=min(int(l), m), replace=False)) for l in lens]
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[1:] = np.cumsum([len(r) for r in rows])
    col = np.concatenate(rows) if rows else np.zeros(0, dtype=np.int64)
    return rp, col


def test_primal_tiles_cover_rows_once():
    """Tiles are contiguous runs of short rows with <= 2048 entries; long
    rows are listed separately; every row appears exactly once."""
    import torch

    from paper_2506_06258_b200.device import build_tiles

    rng = np.random.default_rng(0)
    for lens in (rng.poisson(100, 3000), np.minimum(1 + rng.pareto(1.1, 3000) * 20, 5000),
                 np.full(40, 700), np.array([0, 3, 2000, 0, 5, 1500, 7]),
                 np.ones(5000, dtype=np.int64), rng.integers(1, 4, 3000)):
        lens = np.asarray(lens, dtype=np.int64)
        rp = np.zeros(len(lens) + 1, dtype=np.int64)
        rp[1:] = np.cumsum(lens)
        tiles, long_rows = build_tiles(torch.from_numpy(rp), 2048, 1024)
        tiles = tiles.numpy()
        seen = np.zeros(len(lens), dtype=int)
        for r0, r1 in tiles:
            assert r1 > r0
            assert rp[r1] - rp[r0] <= 2048 and r1 - r0 <= 256
            assert np.all(lens[r0:r1] <= 1024)
            seen[r0:r1] += 1
        seen[long_rows.numpy()] += 1
        assert np.all(seen == 1)
        assert set(long_rows.tolist()) == set(np.flatnonzero(lens > 1024).tolist())


def test_tiles_are_greedy_and_medium_rows_listed():
    """Each tile ends only where the next row would overflow it (entries or
    rows) or is long; medium rows are the tile rows above the register
    capacity, longest first."""
    import torch

    from paper_2506_06258_b200.device import build_tiles, medium_rows

    rng = np.random.default_rng(3)
    lens = np.concatenate([rng.poisson(30, 4000), rng.integers(129, 1025, 300),
                           rng.integers(1025, 3000, 40)]).astype(np.int64)
    rng.shuffle(lens)
    rp = np.zeros(len(lens) + 1, dtype=np.int64)
    rp[1:] = np.cumsum(lens)
    rpt = torch.from_numpy(rp)
    tiles, long_rows = build_tiles(rpt, 2560, 1024, 256)
    tiles = tiles.numpy()
    for r0, r1 in tiles:
        assert rp[r1] - rp[r0] <= 2560 and r1 - r0 <= 256
        if r1 < len(lens) and lens[r1] <= 1024:
            assert rp[r1 + 1] - rp[r0] > 2560 or r1 + 1 - r0 > 256
    med = medium_rows(rpt, long_rows, 128).numpy()
    want = np.flatnonzero((lens > 128) & (lens <= 1024))
    assert sorted(med.tolist()) == want.tolist()
    assert np.all(np.diff(lens[med]) <= 0)


def test_blocked_schedule_preserves_column_order():
    """Walking a good block by block visits every entry of the good once, in
    ascending row order (long rows included where they lie): the reference's
    column_sums order."""
    import torch

    from paper_2506_06258_b200.device import build_blocked_schedule, build_tiles

    rng = np.random.default_rng(1)
    n, m = 700, 60
    lens = rng.poisson(8, n) + 1
    lens[[0, 5, 300, 301, 650]] = [35, 59, 45, 50, 40]   # long rows (threshold 30 below)
    rp, col = _random_csr(rng, n, m, lens)
    rpt = torch.from_numpy(rp)
    tiles, long_rows = build_tiles(rpt, 64, 30, 16)
    bperm, bptr, nblk, tpb = build_blocked_schedule(
        rpt, torch.from_numpy(col.astype(np.int32)), m, tiles, long_rows, prim_grid=3,
        tiles_per_cta=2)
    bperm, bptr = bperm.numpy(), bptr.numpy()
    assert tpb == 6 and nblk == -(-tiles.shape[0] // 6)
    assert np.array_equal(np.sort(bperm), np.arange(len(col)))
    for j in range(m):
        walk = np.concatenate([bperm[bptr[b * m + j]:bptr[b * m + j + 1]]
                               for b in range(nblk + 1)])
        assert np.array_equal(walk, np.flatnonzero(col == j))
        assert bptr[nblk * m + j] == bptr[nblk * m + j + 1]   # the last block is empty


def test_fixed_point_scale_cannot_overflow():
    """The fixed-point column sums: cs_xmax * cs_scale * (entries of the
    fullest good) <= 2^62, so no u64 accumulator can overflow; the scale is a
    power of two between 2^24 and 2^48 (resolution <= 6e-8)."""
    import math

    from paper_2506_06258_b200.device import fixed_point_scale

    for c in [0, 1, 7, 500, 1000, 10_000, 123_457, 10**6, 10**8, 2**31]:
        scale, xmax = fixed_point_scale(c)
        k = math.log2(scale)
        assert k == int(k) and 24 <= k <= 48
        assert xmax * scale * max(1, c) <= 2.0 ** 62 * (1 + 1e-12)
        if c <= 10**6:
            assert xmax >= 1024


def test_library_is_verified_by_source_digest(tmp_path):
    """build() trusts a prebuilt library only if the digest stored beside it
    matches the sources, header, compiler and flags it would be built from."""
    import shutil

    from paper_2506_06258_b200 import _build

    d = _build.source_digest()
    assert d == _build.source_digest() and d != _build.source_digest(("-DMQ_WS_GAMMA=1.1",))
    lib = tmp_path / "lib.so"
    shutil.copy(_build.LIB, lib) if os.path.exists(_build.LIB) else lib.write_bytes(b"x")
    assert not _build.up_to_date(str(lib))              # no digest beside it
    (tmp_path / "lib.so.sha256").write_text(d + "\n")
    assert _build.up_to_date(str(lib))
    (tmp_path / "lib.so.sha256").write_text("0" * 64 + "\n")
    assert not _build.up_to_date(str(lib))              # stale or foreign build
