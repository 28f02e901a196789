"""Row-sharded PDHCG over 2 ranks (gloo, CPU): the engine's N-GPU
orchestration — partial column sums all-reduced every iteration, replicated
prices, distributed residual / restart reductions — reproduces the 1-rank
solve, which matches the reference's golden solve.

The per-rank device operations are the CPU stand-in of tests/_cpu_ops.py; on
the GPU box the same engine code drives the CUDA kernels and NCCL."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden
from _helpers import instance_from, rel_max


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shard_bounds(row_ptr, world):
    """Contiguous row ranges balanced by entries (what bench.py uses)."""
    total = row_ptr[-1]
    cuts = [0] + [int(np.searchsorted(row_ptr, total * r // world, side="right")) for r in
                  range(1, world)] + [len(row_ptr) - 1]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def _cfg(g):
    from paper_2506_06258_b200 import SolveConfig

    extra = {}
    if "restart" in g.files:
        extra = dict(restart=str(g["restart"]), restart_k=int(g["restart_k"]),
                     step_mode=str(g["step_mode"]), max_iters=int(g["max_iters"]))
    return SolveConfig(tol=float(g["tol"]), **extra)


def _solve(inst, cfg, row0, nrows, group):
    from _cpu_ops import CpuMarket, cpu_session
    from paper_2506_06258_b200.driver import solve_on_device

    dm = CpuMarket(inst, row0, nrows)
    sess = cpu_session(dm, group)
    return solve_on_device(sess, cfg, w_sum=float(np.sum(inst.budgets)))


def _worker(rank, world, port, name, out_dir):
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = golden(name)
    inst = instance_from(g)
    lo, hi = shard_bounds(inst.utilities.row_offsets, world)[rank]
    rep = _solve(inst, _cfg(g), lo, hi - lo, dist.group.WORLD)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), prices=rep.prices,
             allocation=rep.allocation, iters=rep.inner_iterations, restarts=rep.restarts,
             objective_part=rep.objective, lo=lo, hi=hi,
             history=np.asarray(rep.residual_history))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["solve_g80_fixed.npz", "solve_medium.npz"])
def test_two_rank_solve_matches_single_rank_and_reference(name, tmp_path):
    g = golden(name)
    inst = instance_from(g)
    one = _solve(inst, _cfg(g), 0, None, None)
    assert one.inner_iterations == int(g["iters"]) and one.restarts == int(g["restarts"])
    assert rel_max(one.prices, g["prices"]) <= 1e-6

    mp.start_processes(_worker, args=(2, _free_port(), name, str(tmp_path)), nprocs=2,
                       start_method="spawn")
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    assert r[0]["lo"] == 0 and r[1]["hi"] == inst.n_buyers and r[0]["hi"] == r[1]["lo"]
    for k in range(2):
        assert int(r[k]["iters"]) == one.inner_iterations
        assert int(r[k]["restarts"]) == one.restarts
        assert rel_max(r[k]["prices"], one.prices) <= 1e-10
        assert np.allclose(r[k]["history"], np.asarray(one.residual_history), rtol=1e-8)
    alloc = np.concatenate([r[0]["allocation"], r[1]["allocation"]])
    assert np.allclose(alloc, one.allocation, rtol=1e-9, atol=1e-13)
    # the objective is reported from the all-reduced row sums
    assert abs(float(r[0]["objective_part"]) - one.objective) <= 1e-10 * abs(one.objective)


def test_shard_bounds_balance_entries():
    rp = np.concatenate([[0], np.cumsum(np.random.default_rng(0).poisson(50, 1000))])
    b = shard_bounds(rp, 4)
    sizes = [rp[h] - rp[l] for l, h in b]
    assert b[0][0] == 0 and b[-1][1] == 1000
    assert max(sizes) - min(sizes) <= 2 * 50 * 3


# ---------------------------------------------------------------- GPU ranks
def _gpu_worker(rank, world, port, name, out_dir):
    """One rank of the sharded device path: its rows' DeviceMarket on cuda:0,
    the engine's per-iteration all-reduce of the fixed-point column sums and
    the check-time reductions over gloo (the kernels of the two ranks never
    wait on each other; only the host-driven collectives couple them)."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.driver import DeviceSession, solve_on_device

    g = golden(name)
    inst = instance_from(g)
    u = inst.utilities
    lo, hi = shard_bounds(u.row_offsets, world)[rank]
    rp = u.row_offsets[lo:hi + 1] - u.row_offsets[lo]
    e0, e1 = int(u.row_offsets[lo]), int(u.row_offsets[hi])
    dm = DeviceMarket(rp, u.col_indices[e0:e1], u.values[e0:e1], inst.budgets[lo:hi],
                      u.n_cols, row_begin=lo)
    cfg = _cfg(g)
    sess = DeviceSession(None, cfg, group=dist.group.WORLD, dm=dm)
    rep = solve_on_device(sess, cfg, w_sum=float(np.sum(inst.budgets)))
    np.savez(os.path.join(out_dir, f"grank{rank}.npz"), prices=rep.prices,
             allocation=rep.allocation, iters=rep.inner_iterations, restarts=rep.restarts,
             lo=lo, hi=hi)
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["solve_medium.npz", "solve_g200_tol0.npz"])
def test_two_rank_device_solve_matches_single_rank(name, tmp_path):
    import paper_2506_06258_b200 as mq

    g = golden(name)
    inst = instance_from(g)
    one = mq.run_solve(inst, _cfg(g), "pdhcg")
    mp.start_processes(_gpu_worker, args=(2, _free_port(), name, str(tmp_path)), nprocs=2,
                       start_method="spawn")
    r = [np.load(tmp_path / f"grank{k}.npz") for k in range(2)]
    for k in range(2):
        assert int(r[k]["iters"]) == one.inner_iterations == int(g["iters"])
        assert int(r[k]["restarts"]) == one.restarts == int(g["restarts"])
        assert rel_max(r[k]["prices"], one.prices) <= 1e-9
    alloc = np.concatenate([r[0]["allocation"], r[1]["allocation"]])
    assert np.allclose(alloc, one.allocation, rtol=1e-8, atol=1e-12)


def _api_worker(rank, world, port, name, out_dir, mode):
    """One rank calling the public run_solve with SolveConfig(group=...):
    mode "full" passes the whole instance (the solver takes its rows and
    gathers the allocation), "shard" passes this rank's FisherShard."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2506_06258_b200 as mq
    from paper_2506_06258_b200.driver import split_rows

    g = golden(name)
    inst = instance_from(g)
    cfg = _cfg(g).with_overrides(group=dist.group.WORLD)
    if mode == "shard":
        u = inst.utilities
        cuts = split_rows(u.row_offsets, world)
        lo, hi = cuts[rank], cuts[rank + 1]
        e0, e1 = int(u.row_offsets[lo]), int(u.row_offsets[hi])
        sm = mq.SparseMatrix(hi - lo, u.n_cols, u.row_offsets[lo:hi + 1] - e0,
                             u.col_indices[e0:e1], u.values[e0:e1])
        inst = mq.FisherShard(sm, inst.budgets[lo:hi], lo, u.n_rows)
    rep = mq.run_solve(inst, cfg, "pdhcg")
    np.savez(os.path.join(out_dir, f"api{rank}.npz"), prices=rep.prices,
             allocation=rep.allocation, t=rep.utility_values, iters=rep.inner_iterations,
             restarts=rep.restarts, objective=rep.objective, fp=rep.instance_fingerprint)
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["full", "shard"])
def test_run_solve_with_a_group_matches_single_rank(mode, tmp_path):
    import paper_2506_06258_b200 as mq

    name = "solve_g200_tol0.npz"
    g = golden(name)
    inst = instance_from(g)
    one = mq.run_solve(inst, _cfg(g), "pdhcg")
    mp.start_processes(_api_worker, args=(2, _free_port(), name, str(tmp_path), mode), nprocs=2,
                       start_method="spawn")
    r = [np.load(tmp_path / f"api{k}.npz") for k in range(2)]
    for k in range(2):
        assert int(r[k]["iters"]) == one.inner_iterations == int(g["iters"])
        assert int(r[k]["restarts"]) == one.restarts == int(g["restarts"])
        assert rel_max(r[k]["prices"], one.prices) <= 1e-9
        assert abs(float(r[k]["objective"]) / one.objective - 1.0) <= 1e-8
    if mode == "full":  # every rank reports the whole market
        for k in range(2):
            assert np.allclose(r[k]["allocation"], one.allocation, rtol=1e-8, atol=1e-12)
            assert np.allclose(r[k]["t"], one.utility_values, rtol=1e-9)
            assert str(r[k]["fp"]) == one.instance_fingerprint
    else:
        alloc = np.concatenate([r[0]["allocation"], r[1]["allocation"]])
        assert np.allclose(alloc, one.allocation, rtol=1e-8, atol=1e-12)


def _nccl_capture_worker(rank, world, port, name, out_dir):
    """A 1-rank NCCL group with the N-rank step forced: the chunk graph
    captures the NCCL all-reduce of the fixed-point column sums together with
    the kernels (what N GPUs replay every chunk)."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    sys.path.insert(0, os.path.dirname(os.path.dirname(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.engine import PdhcgEngine

    g = golden(name)
    inst = instance_from(g)
    out = {}
    for tag, force in (("forced", True), ("plain", False)):
        dm = DeviceMarket.from_instance(inst)
        eng = PdhcgEngine(dm, group=dist.group.WORLD, force_collectives=force)
        eng.initial_state()
        eng.set_steps(0.05, 0.05)
        for _ in range(3):
            eng.run_chunk(40)
        torch.cuda.synchronize()
        out[tag + "_p"] = eng.p.cpu().numpy()
        out[tag + "_x"] = eng.x.cpu().numpy()
        out[tag + "_graphs"] = np.array([eng.use_graphs, len(eng._graphs) > 0, eng.distributed])
    np.savez(os.path.join(out_dir, "nccl.npz"), **out)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_nccl_collectives_are_captured_in_the_chunk_graph(tmp_path):
    mp.start_processes(_nccl_capture_worker,
                       args=(1, _free_port(), "solve_g200_tol0.npz", str(tmp_path)), nprocs=1,
                       start_method="spawn")
    r = np.load(tmp_path / "nccl.npz")
    assert list(r["forced_graphs"]) == [1, 1, 1]   # captured with the collectives
    assert list(r["plain_graphs"]) == [1, 1, 0]
    # integer all-reduce of one rank is the identity: bitwise the same iterate
    assert np.array_equal(r["forced_p"], r["plain_p"])
    assert np.array_equal(r["forced_x"], r["plain_x"])
