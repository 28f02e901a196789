#!/usr/bin/env python
"""PDHCG throughput on BASELINE config 4 (10M buyers x 100k goods, ~1e9 nnz).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl b200|reference]

One "step" is one PDHCG iteration over the whole market (price step, exact
per-buyer prox fused with the running average, deterministic column sums),
replayed from CUDA graphs of `check_every` iterations.  `value` = iterations/s
of the whole job with the market resident in HBM (device clock, max over
ranks); the per-kernel CUDA events give the primal kernel's achieved HBM
bandwidth (`roofline`).  `e2e` is a full solve to 1e-4 relative KKT through
the public API (run_solve on a host instance: upload, setup, every residual
check, download) — the time-to-tolerance of BASELINE.json — and
`cpu_baseline` the reference algorithm (the C oracle port of
kernels.pdhcg_chunk) on a bounded row sample of the same market on this
host's cores.  N>1: buyer rows are sharded contiguously (nnz-balanced), the
m-length column sums are NCCL-all-reduced every iteration (strong scaling).
"""

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PDHCG iter/s + time to 1e-4 rel. KKT; achieved HBM GB/s vs peak; 1/2/4/8 GPUs"
CONFIG_TEXT = {
    "c1": "dense 1000 x 500 linear Fisher market",
    "c2": "sparse 100k x 10k, 1% density, random budgets",
    "c3": "power-law 1M x 50k, nnz~1e8",
    "c4": "sparse 10M buyers x 100k goods, nnz~1e9",
    "c5": "100k x 100k, 1% density (Arrow-Debreu inner market)",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workload

def shard_rows(name, rank, world, seed):
    """Rows of this rank (contiguous, balanced by nnz) generated on device."""
    import torch

    from paper_2506_06258_b200 import _native as nat
    from paper_2506_06258_b200.generate import CONFIGS, generate_rows, powerlaw_dmin

    c = CONFIGS[name]
    n, m = c["n"], c["m"]
    if world == 1:
        return generate_rows(n, m, seed=seed, q=c.get("q"), powerlaw=c.get("powerlaw"),
                             mean_degree=c.get("mean_degree"))
    # degree pass over all rows (cheap) -> nnz-balanced split points
    lib = nat.lib()
    pl = c.get("powerlaw")
    q_mode, q, alpha, dmin = ((1, 0.0, float(pl), powerlaw_dmin(m, pl, c["mean_degree"]))
                              if pl else (0, float(c["q"]), 2.0, 1.0))
    deg = torch.empty(n, dtype=torch.int64, device="cuda")
    nat.check(lib.mq_gen_degrees(0, n, m, q_mode, q, alpha, dmin, seed, nat.ptr(deg),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
              "mq_gen_degrees")
    cum = torch.cumsum(deg, 0)
    total = int(cum[-1].item())
    targets = torch.tensor([total * r // world for r in range(1, world)], device="cuda")
    cuts = [0] + torch.searchsorted(cum, targets).add_(1).tolist() + [n]
    del deg, cum
    lo, hi = cuts[rank], cuts[rank + 1]
    return generate_rows(n, m, seed=seed, q=c.get("q"), powerlaw=pl,
                         mean_degree=c.get("mean_degree"), row0=lo, nrows=hi - lo)


def make_session(shard, group):
    import torch

    from paper_2506_06258_b200.adaptive import StepController
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.driver import OMEGA_BOUND_FACTOR
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.sparse import selector_norm_from_counts

    dm = DeviceMarket(shard["row_ptr"], shard["col"], shard["u"], shard["w"], shard["m"],
                      row_begin=shard["row0"])
    eng = PdhcgEngine(dm, group=group)
    w_sum = eng._allreduce(dm.w.sum().reshape(1)).item()
    eng.initial_state(w_sum=w_sum)
    L = selector_norm_from_counts(eng._global_counts().cpu().numpy())
    pr, du = eng.omega_norms()
    omega0 = max(1.0, du / pr) if (pr > 1e-8 and du > 1e-8) else 1.0
    ctrl = StepController(eta_initial=0.9 / L, omega_initial=omega0, eta_max=0.95 / L,
                          omega_lower=omega0 / OMEGA_BOUND_FACTOR,
                          omega_upper=omega0 * OMEGA_BOUND_FACTOR)
    eng.set_steps(ctrl.tau, ctrl.sigma)
    torch.cuda.synchronize()
    return dm, eng


def run_iters(eng, iters, chunk=40):
    done = 0
    passes = 0
    while done < iters:
        c = min(chunk, iters - done)
        passes += sum(eng.run_chunk(c))
        done += c
    return passes


def kernel_breakdown(eng, iters):
    """Per-kernel device time inside real iterations (eager launches, CUDA
    events on the launching stream)."""
    import torch

    from paper_2506_06258_b200 import _native as nat

    lib, mk, st = eng.ops.lib, eng.dm.struct, eng.state
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(iters)]
    eng.pass_buf.zero_()
    eng.faults.zero_()
    for it in range(iters):
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        e = ev[it]
        e[0].record()
        nat.check(lib.mq_dual_step(mk, st, it, s), "dual")
        e[1].record()
        nat.check(lib.mq_primal_step(mk, st, it, None, s), "primal")
        e[2].record()
        nat.check(lib.mq_colsum_step(mk, st, it, 1, s), "colsum")
        if eng.world > 1:
            eng._allreduce(eng.cs)
            nat.check(lib.mq_colsum_finalize(mk, st, it, s), "finalize")
        e[3].record()
    cur = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    nat.check(lib.mq_chunk_end(st, iters, cur), "chunk_end")
    if eng.sparse:
        nat.check(lib.mq_avg_materialize(mk, st, cur), "avg_materialize")
    torch.cuda.synchronize()
    eng.navg += iters
    t = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])]
                  for e in ev])
    passes = int(eng.pass_buf[:iters].sum().item())
    return t.mean(axis=0), passes


# random 8-byte gathers from an L2-resident 800 KB vector, 148 SMs, 164 KB of
# shared memory per SM (the fused kernel's carveout): profiles/micro_gather_l1.txt
GATHER_PEAK = 2.66e11


def traffic_from_profile(name, config):
    """ncu DRAM bytes per launch of `name` on `config` (profiles/ncu_traffic.json,
    written by tools/ncu_summary.py from the round's full capture), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh).get(name, {})
        return d.get("dram_bytes_per_launch") if d.get("config", "c4") == config else None
    except Exception:
        return None


# ------------------------------------------------------------------ CPU side

def host_sample(shard, target_nnz):
    """First rows of the market with ~target_nnz entries, as host arrays."""
    rp = shard["row_ptr"]
    rows = int(np.searchsorted(rp.cpu().numpy(), target_nnz, side="right")) - 1
    rows = max(1, min(rows, rp.numel() - 1))
    nnz = int(rp[rows].item())
    return (rp[:rows + 1].cpu().numpy(), shard["col"][:nnz].cpu().numpy().astype(np.int64),
            shard["u"][:nnz].cpu().numpy(), shard["w"][:rows].cpu().numpy())


def cpu_iteration_rate(sample, m, nnz_full, tau, sigma, iters, threads):
    """Oracle (C restatement of kernels.pdhcg_chunk) on the sample; returns
    (full-market iterations/s extrapolated by nnz, seconds per sample iteration)."""
    from oracle import solve as orc

    rp, col, u, w = sample
    orc.set_threads(threads)
    mk = orc.Market(len(rp) - 1, m, rp, col, u, w)
    nm, _ = orc.normalize(mk)
    tperm, tind = orc.transpose_schedule(nm)
    counts = np.bincount(nm.col, minlength=m).astype(np.float64)
    x = 1.0 / np.maximum(counts, 1.0)[nm.col]
    p = np.full(m, float(np.sum(w)) / m)
    xp, xb, pb = x.copy(), x.copy(), p.copy()
    cbuf = np.empty(nm.nnz)
    col32, tp32 = nm.col.astype(np.int32), tperm.astype(np.int32)
    passes = np.zeros(1, dtype=np.int64)
    orc.pdhcg_chunk(nm.indptr, col32, nm.val, tp32, tind, nm.w, x, xp, p, xb, pb, 0, tau, sigma,
                    32, 1e-10, 1, cbuf, passes)  # warm-up
    t0 = time.perf_counter()
    passes = np.zeros(iters, dtype=np.int64)
    orc.pdhcg_chunk(nm.indptr, col32, nm.val, tp32, tind, nm.w, x, xp, p, xb, pb, 1, tau, sigma,
                    32, 1e-10, iters, cbuf, passes)
    dt = (time.perf_counter() - t0) / iters
    return (nm.nnz / nnz_full) / dt, dt, nm.nnz, len(rp) - 1


def calibrated_sample_nnz(shard, m, nnz_full, tau, sigma, threads, seconds_per_iter):
    probe = host_sample(shard, 1_000_000)
    _, dt, nnz_probe, _ = cpu_iteration_rate(probe, m, nnz_full, tau, sigma, 1, threads)
    return int(min(nnz_full, max(200_000, nnz_probe * seconds_per_iter / max(dt, 1e-6))))


# ------------------------------------------------------------------ main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIG_TEXT))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-max-iters", type=int, default=2000)
    ap.add_argument("--breakdown-iters", type=int, default=20)
    a = ap.parse_args()
    a.warmup = max(a.warmup, 3)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the N-rank path on a 1-GPU box: every rank on cuda:0,
    # gloo collectives (numbers meaningless; never used for measurements)
    shared = os.environ.get("MQ_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    if a.impl == "reference":
        return reference_arm(a, rank, world)

    from paper_2506_06258_b200 import _build

    _build.build()
    hbm_peak, peak_kind = peaks()
    t_setup = time.perf_counter()
    shard = shard_rows(a.config, rank, world, a.seed)
    dm, eng = make_session(shard, group)
    setup_s = time.perf_counter() - t_setup
    n_full, m = shard["n"], shard["m"]
    nnz_local = dm.nnz
    nnz_full = int(eng._allreduce(torch.tensor([nnz_local], dtype=torch.int64,
                                               device="cuda")).item())

    run_iters(eng, a.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        passes = run_iters(eng, a.steps)
        e1.record()
        torch.cuda.synchronize()
    t_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    eng._allreduce(t_ms, "max")
    t_ms = float(t_ms.item())
    if world > 1:
        dist.barrier()
    value = a.steps / (t_ms / 1e3)
    # kernels launched in the timed region: dual + non-empty primal bins + colsum
    # per iteration, chunk_end (+ the running-average materialization) per chunk
    # (+ finalize on N>1)
    primal_kernels = (int(dm.tiles.shape[0] > 0) + int(dm.long_rows.numel() > 0)
                      + int(dm.med_rows.numel() > 0))
    per_it = 2 + primal_kernels + (1 if world > 1 else 0)
    launches = a.steps * per_it + -(-a.steps // 40) * (1 + int(eng.sparse))

    # per-kernel breakdown and the primal kernel's roofline
    kt, kpass = kernel_breakdown(eng, a.breakdown_iters)
    n_local = dm.n
    # algorithmic bytes of one iteration's nnz sweep in the dense formulation
    # (prox + averages 44 B/nnz, column sums 12 B/nnz, + rows and
    # goods).  The default kernel skips the ~99 % zero entries of x (sparse
    # iterate), so its DRAM traffic is far lower (`dram_*`);
    # its binding resource is the random L2 gather of p[col], one 32-byte
    # sector per entry (`gather_*`, peak = tools/micro/gather_l1.cu)
    primal_bytes = 56 * nnz_local + 20 * n_local + 8 * m
    achieved = primal_bytes / (kt[1] / 1e3) / 1e9
    traffic = traffic_from_profile("primal", a.config)
    gathers_per_s = nnz_local / (kt[1] / 1e3)
    iter_bytes = 56 * nnz_full + 16 * n_full + 48 * m      # SURVEY §8(d) B_iter
    iter_gbs = iter_bytes / (t_ms / 1e3 / a.steps) / 1e9 / world

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "iter/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(t_ms / a.steps, 4),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config {a.config[1]}: {CONFIG_TEXT[a.config]}",
                   "n_buyers": n_full, "m_goods": m, "nnz": nnz_full, "seed": a.seed,
                   "row_solver": "exact", "parallelism": f"row-shard x{world}",
                   "l2": f"inputs larger than L2 ({iter_bytes / 1e9:.1f} GB algorithmic "
                         "traffic per iteration vs 126 MB L2)"},
        "roofline": {"bound": "hbm",
                     "kernel": "primal step: primal_fused_kernel (exact prox + averages + "
                               "column sums) + medium / long row kernels where present",
                     "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4),
                     "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": primal_bytes,
                     "note": "achieved = SURVEY 8(d) algorithmic bytes (dense formulation) / "
                             "kernel time; the sparse-iterate kernel does not move the zero "
                             "entries of x, see dram_* for its own traffic and gather_* for "
                             "the resource that binds it",
                     "dram_achieved": (round(traffic / (kt[1] / 1e3) / 1e9, 1)
                                       if traffic else None),
                     "dram_frac": (round(traffic / (kt[1] / 1e3) / 1e9 / hbm_peak, 4)
                                   if traffic else None),
                     "gather_achieved": round(gathers_per_s / 1e9, 1),
                     "gather_peak": GATHER_PEAK / 1e9, "gather_unit": "G random 8-byte L2 "
                     "gathers/s", "gather_frac": round(gathers_per_s / GATHER_PEAK, 4)},
        "iteration_roofline": {"bytes_per_iteration": iter_bytes,
                               "achieved_gbs_per_gpu": round(iter_gbs, 1),
                               "frac": round(iter_gbs / hbm_peak, 4)},
        "kernels_ms": {"dual": round(kt[0], 4), "primal": round(kt[1], 4),
                       "colsum": round(kt[2], 4)},
        "sweeps_per_row_per_iter": round(passes / a.steps / n_full, 3),
        "gpu_launches": launches, "setup_seconds": round(setup_s, 2),
    }
    with torch.cuda.device(local):
        out["clocks"] = clk.summary()
    del eng, dm
    torch.cuda.empty_cache()

    out["e2e"] = None
    if world == 1 and not a.no_e2e:
        out["e2e"] = e2e_solve(shard, a.e2e_max_iters)
        out["ttt_seconds"] = out["e2e"]["ttt_seconds"]
    if rank == 0 and world == 1 and not a.no_cpu:
        out["cpu_baseline"] = cpu_baseline(shard, m, nnz_full)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_solve(shard, max_iters):
    """Full solve to 1e-4 through the public API from host buffers."""
    import torch

    import paper_2506_06258_b200 as mq

    rp = shard["row_ptr"].cpu().numpy()
    col = shard["col"].cpu().numpy().astype(np.int64)
    u = shard["u"].cpu().numpy()
    w = shard["w"].cpu().numpy()
    inst = mq.FisherInstance(mq.SparseMatrix(shard["n"], shard["m"], rp, col, u), w)
    del col, u
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = mq.run_solve(inst, mq.SolveConfig(tol=1e-4, max_iters=max_iters), "pdhcg")
    wall = time.perf_counter() - t0
    nnz, n, m = inst.utilities.nnz, inst.n_buyers, inst.n_goods
    h2d = 8 * (n + 1) + 4 * nnz + 8 * nnz + 8 * n
    d2h = 8 * m + 8 * nnz + 8 * n + 8 * n
    its = rep.inner_iterations
    return {"value": round(its / wall, 3), "unit": "iter/s",
            "h2d_bytes_per_step": h2d // max(its, 1), "d2h_bytes_per_step": d2h // max(its, 1),
            "ttt_seconds": round(wall, 3), "iterations": its, "restarts": rep.restarts,
            "status": rep.status, "rel_kkt": rep.final_residuals.rel_kkt,
            "objective": rep.objective,
            "device_iters_per_second": round(rep.device_stats["iters_per_second"], 3),
            "note": "one run_solve(tol=1e-4) on a host FisherInstance; per-step bytes = "
                    "instance upload + result download amortized over the iterations"}


def cpu_baseline(shard, m, nnz_full, seconds_per_iter=4.0, iters=3):
    threads = os.cpu_count() or 1
    tau = sigma = 0.9 / np.sqrt(float(nnz_full) / m)  # representative step sizes
    target = calibrated_sample_nnz(shard, m, nnz_full, tau, sigma, threads, seconds_per_iter)
    sample = host_sample(shard, target)
    rate, dt, nnz_s, rows = cpu_iteration_rate(sample, m, nnz_full, tau, sigma, iters, threads)
    return {"value": round(rate, 6), "unit": "iter/s", "cores": threads, "kind": "port",
            "sample": f"first {rows} buyers ({nnz_s} nnz, {100.0 * nnz_s / nnz_full:.2f}% of "
                      f"the market) x {iters} iterations of the C oracle "
                      f"(kernels.pdhcg_chunk restatement, k-section 32, subtol 1e-10); "
                      f"{dt:.3f} s/iteration on the sample, extrapolated linearly in nnz",
            "seconds_per_sample_iteration": round(dt, 4)}


def reference_arm(a, rank, world):
    """The reference algorithm (C oracle port) on the host cores, rank 0 only."""
    import torch.distributed as dist

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    import torch

    from paper_2506_06258_b200 import _build

    _build.build()
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    shard = shard_rows(a.config, 0, 1, a.seed)
    n, m = shard["n"], shard["m"]
    nnz_full = int(shard["row_ptr"][-1].item())
    threads = os.cpu_count() or 1
    tau = sigma = 0.9 / np.sqrt(float(nnz_full) / m)
    # size one step so that warmup + steps fit in ~2 minutes
    per_step = max(0.05, 120.0 / (a.steps + a.warmup))
    target = calibrated_sample_nnz(shard, m, nnz_full, tau, sigma, threads, per_step)
    sample = host_sample(shard, target)
    del shard
    torch.cuda.empty_cache()
    cpu_iteration_rate(sample, m, nnz_full, tau, sigma, a.warmup, threads)
    rate, dt, nnz_s, rows = cpu_iteration_rate(sample, m, nnz_full, tau, sigma, a.steps, threads)
    out = {
        "metric": METRIC, "value": round(rate, 6), "unit": "iter/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(1e3 / rate, 3),
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"BASELINE config {a.config[1]}: {CONFIG_TEXT[a.config]}",
                   "n_buyers": n, "m_goods": m, "nnz": nnz_full, "seed": a.seed,
                   "row_solver": "ksection"},
        "cpu_baseline": {"value": round(rate, 6), "unit": "iter/s", "cores": threads,
                         "kind": "port",
                         "sample": f"each step = one iteration of the C oracle "
                                   f"(kernels.pdhcg_chunk restatement) over the first {rows} "
                                   f"buyers ({nnz_s} nnz), extrapolated linearly in nnz to "
                                   f"the full market"},
        "e2e": {"value": round(rate, 6), "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
