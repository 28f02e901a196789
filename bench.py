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
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML
    polling thread (every ~0.5 ms, so even a 20 ms region gets dozens of
    samples); nvidia-smi -lms 200 if NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []  # (t, sm_mhz, reason bits) from NVML
        self.nvml = None
        self.stop = threading.Event()

    def _handle(self):
        import pynvml
        import torch

        pynvml.nvmlInit()
        try:  # the CUDA device's own GPU, whatever CUDA_VISIBLE_DEVICES maps
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(
                uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, nv, h):
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((time.perf_counter(), float(sm), int(rs)))
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        try:
            nv, h = self._handle()
            self.nvml = (nv, h, float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))
            self.t = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.t.start()
            while not self.samples and self.t.is_alive():  # polling before the region starts
                time.sleep(0.0002)
            self.t0 = time.perf_counter()
            return self
        except Exception:
            self.nvml = None
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
        if self.nvml is not None:
            self.t1 = time.perf_counter()
            self.stop.set()
            self.t.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nvml is not None:
            nv, _, mx = self.nvml
            inside = [x for x in self.samples if self.t0 <= x[0] <= self.t1]
            if not inside and self.samples:  # region shorter than a poll: the nearest ones
                inside = sorted(self.samples, key=lambda x: min(abs(x[0] - self.t0),
                                                                abs(x[0] - self.t1)))[:2]
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted({k for _, _, r in inside for k, b in bits.items() if r & b})
            if not inside:
                return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0,
                        "source": "nvml"}
            return {"sm_mhz": statistics.median(x[1] for x in inside), "sm_max_mhz": mx,
                    "reasons": reasons, "samples": len(inside), "source": "nvml"}
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvidia-smi"}


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


def warm_graphs(eng, iters, chunk=40):
    """Capture (not run) the chunk graphs run_iters(eng, iters) will replay,
    so no capture falls inside a timed region."""
    if not getattr(eng, "use_graphs", False):
        return
    for c in {min(chunk, iters)} | ({iters % chunk} if iters > chunk and iters % chunk else set()):
        if (c, False) not in eng._graphs:
            try:
                eng._capture(c, False)
            except Exception:  # capture unsupported here: run_chunk falls back itself
                return


def run_iters(eng, iters, chunk=40):
    done = 0
    passes = 0
    while done < iters:
        c = min(chunk, iters - done)
        passes += sum(eng.run_chunk(c))
        done += c
    return passes


def kernel_breakdown(eng, iters):
    """Per-kernel device time inside real iterations, launched exactly as the
    engine's chunk does it (eager; CUDA events on the launching stream), and
    the working-set counts of those iterations."""
    import torch

    ops = eng.ops
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(iters)]
    full_rows = torch.zeros(1, dtype=torch.int64, device=eng.dm.device)
    eng.pass_buf.zero_()
    eng.faults.zero_()
    for it in range(iters):
        e = ev[it]
        e[0].record()
        ops.dual(it)
        e[1].record()
        ops.primal(it)
        e[2].record()
        if eng.world > 1:  # the engine's N-rank step: integer all-reduce, then convert
            eng._allreduce(eng.bucket.view(torch.int64)[:eng.dm.m])
        ops.colsum_rest(it, True)
        e[3].record()
        if eng.working_set:
            full_rows += eng.blk_done[3]
    ops.chunk_end(iters)
    torch.cuda.synchronize()
    eng.navg += iters
    t = np.array([[e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), e[2].elapsed_time(e[3])]
                  for e in ev])
    counts = {"passes": int(eng.pass_buf[:iters].sum().item())}
    if eng.working_set:
        h = eng.ws_len
        counts.update(full_rows=float(full_rows.item()) / iters,
                      ws_entries=int(h.clamp(min=0).sum().item()),
                      ws_rows=int((h >= 0).sum().item()),
                      tile_rows=int((eng.ws_init == -1).sum().item()),
                      nonzero=int(eng.xflag[:eng.dm.nnz].sum().item()))
    return t.mean(axis=0), counts


def screened_bytes(dm, c):
    """Algorithmic bytes of one screened iteration: what the
    working-set algorithm must touch once — per tile row its working-set
    length (4 B) and, with a working set, budget, warm start r/w, certificate
    and row offset (56 B); per working-set entry its slot (24 B) and price
    (8 B); per nonzero entry its x write, running-sum r/w and column-sum add
    (32 B); rows solved in full and the medium / long rows read u, col, flag
    and price (21 B per entry, 64 B per row); per good 48 B."""
    rp = dm.row_ptr
    lens = (rp[1:] - rp[:-1])
    big = lens > 128
    big_entries = int(lens[big].sum().item())
    big_rows = int(big.sum().item())
    full_entries = c["full_rows"] * (dm.nnz - big_entries) / max(1, c["tile_rows"])
    return (4 * c["tile_rows"] + 56 * c["ws_rows"] + 32 * c["ws_entries"] + 32 * c["nonzero"]
            + 21 * (big_entries + full_entries) + 64 * (big_rows + c["full_rows"]) + 48 * dm.m)


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

REF_BUDGET_S = 300.0  # the reference arm's timed steps (whole-market iterations)

def host_copy(shard):
    """Host arrays of this rank's shard (the e2e input and the CPU legs)."""
    from paper_2506_06258_b200.engine import to_host

    return {"row_ptr": shard["row_ptr"].cpu().numpy(), "col": to_host(shard["col"]),
            "u": to_host(shard["u"]), "w": shard["w"].cpu().numpy(), "n": shard["n"],
            "m": shard["m"], "row0": shard["row0"]}


def cpu_chunk_run(host, threads):
    """The reference's compact iterate on the FULL market on the host cores:
    oracle.solve.ChunkRun = _CompactRun's setup (normalize, transpose
    schedule, x = 1/colcount, p = sum(w)/m, L, omega_0 -> the first restart
    window's tau/sigma) around the C restatement of kernels.pdhcg_chunk
    (k-section 32, subproblem_tol 1e-10: the reference defaults)."""
    from oracle import solve as orc

    orc.set_threads(threads)
    t0 = time.perf_counter()
    run = orc.ChunkRun(host["row_ptr"], host["col"], host["u"], host["w"], host["m"])
    return run, time.perf_counter() - t0


def cpu_baseline(host, iters=1):
    """Reported CPU baseline: `iters` iterations of the reference algorithm
    over the whole market from its initial state (no sample, no
    extrapolation)."""
    threads = os.cpu_count() or 1
    run, setup = cpu_chunk_run(host, threads)
    t0 = time.perf_counter()
    passes = run.step(iters)
    dt = (time.perf_counter() - t0) / iters
    nnz = int(host["row_ptr"][-1])
    return {"value": round(1.0 / dt, 6), "unit": "iter/s", "cores": threads, "kind": "port",
            "sample": f"{iters} iteration(s) of the whole market (n={host['n']}, m={host['m']}, "
                      f"nnz={nnz}) from the initial state, C oracle = restated "
                      f"kernels.pdhcg_chunk (k-section 32, subtol 1e-10), tau=sigma="
                      f"{run.tau:.6g} (the solver's first restart window), {threads} threads; "
                      f"{passes.sum() / max(1, host['n']) / iters:.2f} k-section passes per "
                      f"row per iteration",
            "seconds_per_iteration": round(dt, 4), "setup_seconds": round(setup, 2)}


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
    ap.add_argument("--e2e-max-iters", type=int, default=100_000)
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
    if a.impl == "reference":  # host cores only: no device, gloo for the barrier
        if world > 1:
            dist.init_process_group("gloo")
        return reference_arm(a, rank, world)
    if shared:
        local = 0
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            # NCCL's INFO lines show the communicator (ranks, NVLink/NVLS paths)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD

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
    warm_graphs(eng, a.steps)
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
    # our kernels launched in the timed region, per iteration: dual, the
    # screened solve + full-solve list (or the tile kernel), medium / long
    # row kernels where present, column sums; per chunk: chunk_end and the
    # running-average materialization
    primal_kernels = ((2 if eng.working_set else int(dm.tiles.shape[0] > 0))
                      + int(dm.long_rows.numel() > 0) + int(dm.med_rows.numel() > 0))
    launches = a.steps * (2 + primal_kernels) + -(-a.steps // 40) * (1 + int(eng.sparse))

    # per-kernel breakdown (CUDA events, the engine's own launch sequence)
    kt, counts = kernel_breakdown(eng, a.breakdown_iters)
    t_primal = kt[1] / 1e3
    iter_bytes = 56 * nnz_full + 16 * n_full + 48 * m      # SURVEY §8(d) B_iter (dense)
    if eng.working_set:
        alg = screened_bytes(dm, counts)
        rkernel = ("primal step: ws_kernel (screened exact prox over the working sets, "
                   "averages, column sums) + ws_full_kernel (listed rows) + medium / long row "
                   "kernels where present")
        model = ("algorithmic bytes of the screened iteration (DESIGN.md §7): 4 B per tile "
                 "row, 56 B per row with a working set, 32 B per working-set entry, 32 B per "
                 "nonzero entry, 21 B per entry of rows solved in full (+64 B per row), 48 B "
                 "per good; counts measured on the breakdown iterations")
    else:
        alg = 56 * dm.nnz + 20 * dm.n + 8 * m
        rkernel = "primal step: primal_fused_kernel + medium / long row kernels"
        model = "SURVEY 8(d) dense-formulation bytes"
    achieved = alg / t_primal / 1e9
    traffic = traffic_from_profile("primal", a.config)
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "iter/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(t_ms / a.steps, 4),
        "higher_is_better": True, "scaling": "strong",  # one fixed market at every N
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config {a.config[1]}: {CONFIG_TEXT[a.config]}",
                   "n_buyers": n_full, "m_goods": m, "nnz": nnz_full, "seed": a.seed,
                   "row_solver": "exact", "working_set": bool(eng.working_set),
                   "parallelism": f"row-shard x{world}",
                   "l2": "inputs larger than L2 (8 GB of utilities per GPU vs 126 MB L2)"},
        "roofline": {"bound": "hbm", "kernel": rkernel,
                     "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                     "peak_kind": peak_kind, "algorithmic_bytes_per_launch": int(alg),
                     "model": model,
                     "dram_achieved": (round(traffic / t_primal / 1e9, 1) if traffic else None),
                     "dram_frac": (round(traffic / t_primal / 1e9 / hbm_peak, 4)
                                   if traffic else None)},
        "dense_equivalent": {"bytes_per_iteration": iter_bytes,
                             "gbs_per_gpu": round(iter_bytes / (t_ms / 1e3 / a.steps) / 1e9
                                                  / world, 1),
                             "note": "SURVEY 8(d) dense-formulation bytes / iteration time: "
                                     "an equivalent throughput, not bandwidth (the screened "
                                     "iteration does not move the entries it certifies)"},
        "kernels_ms": {"dual": round(kt[0], 4), "primal": round(kt[1], 4),
                       "colsum": round(kt[2], 4)},
        "working_set": counts, "sweeps_per_row_per_iter": round(passes / a.steps / n_full, 3),
        "gpu_launches": launches, "setup_seconds": round(setup_s, 2),
    }
    with torch.cuda.device(local):
        out["clocks"] = clk.summary()
    del eng, dm
    torch.cuda.empty_cache()

    host = None
    if not (a.no_e2e and a.no_cpu):
        host = host_copy(shard)
    del shard
    torch.cuda.empty_cache()
    out["e2e"] = None
    if not a.no_e2e:
        out["e2e"] = e2e_solve(host, a.e2e_max_iters, group=group if world > 1 else None)
        out["ttt_seconds"] = out["e2e"]["ttt_seconds"]
    if rank == 0 and world == 1 and not a.no_cpu:
        out["cpu_baseline"] = cpu_baseline(host)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def e2e_solve(host, max_iters, group=None):
    """Time to 1e-4 relative KKT through the public API: run_solve on a host
    FisherInstance (upload, device setup, every residual check, the final
    download), timed by the host clock around the call, plus the solve
    loop alone as the reference's wall_time_seconds measures it
    (driver.py:319,359)."""
    import torch

    import paper_2506_06258_b200 as mq

    n, m = host["n"], host["m"]
    sm = mq.SparseMatrix(host["row_ptr"].shape[0] - 1, m, host["row_ptr"], host["col"],
                         host["u"])
    if group is None:
        inst = mq.FisherInstance(sm, host["w"])
    else:  # this rank's rows: the public multi-GPU input
        inst = mq.FisherShard(sm, host["w"], host["row0"], n)
    cfg = mq.SolveConfig(tol=1e-4, max_iters=max_iters, group=group)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = mq.run_solve(inst, cfg, "pdhcg")
    wall = time.perf_counter() - t0
    nnz, nl = inst.utilities.nnz, inst.n_buyers
    # copies made by the call: row offsets, columns (int64), values, budgets
    # up; prices, allocation, utility values and budgets back (+ 32 doubles
    # of residual scalars per check)
    h2d = 8 * (nl + 1) + 8 * nnz + 8 * nnz + 8 * nl
    checks = len(rep.residual_history)
    d2h = 8 * m + 8 * nnz + 8 * nl + 8 * nl + 8 * 32 * (checks + 2)
    its = rep.inner_iterations
    return {"value": round(its / wall, 3), "unit": "iter/s",
            "h2d_bytes_per_step": h2d // max(its, 1), "d2h_bytes_per_step": d2h // max(its, 1),
            "ttt_seconds": round(wall, 3), "solve_loop_seconds": round(rep.wall_time_seconds, 3),
            "iterations": its, "restarts": rep.restarts, "status": rep.status,
            "rel_kkt": rep.final_residuals.rel_kkt, "objective": rep.objective,
            "checks": checks,
            "device_iters_per_second": round(rep.device_stats["iters_per_second"], 3),
            "note": "one run_solve(tol=1e-4) on a host FisherInstance, max_iters = "
                    f"{max_iters} (the reference default); value = iterations / wall time "
                    "of the call; per-step bytes = upload + download amortized"}


def reference_arm(a, rank, world):
    """--impl reference: the reference algorithm (oracle port of
    kernels.pdhcg_chunk around _CompactRun's setup) on the host cores, on
    the same market (regenerated on the host byte for byte by
    oracle/market_gen.c; the product's CUDA library is never loaded), every
    step one iteration of the whole market.  Rank 0 only."""
    import torch.distributed as dist

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    from oracle import gen as hg

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    host = hg.generate_config(a.config, seed=a.seed, threads=threads)
    gen_s = time.perf_counter() - t0
    n, m = host["n"], host["m"]
    nnz = int(host["row_ptr"][-1])
    run, setup_s = cpu_chunk_run(host, threads)
    del host
    # every step is one whole-market iteration; the run stays within
    # REF_BUDGET_S: at most 2 warm-up iterations (a C kernel needs no JIT
    # warm-up) and K timed ones unless K of them would exceed the budget
    warm = max(1, min(a.warmup, 2))
    tw = time.perf_counter()
    for _ in range(warm):
        run.step(1)
    t_it = (time.perf_counter() - tw) / warm
    steps = int(max(3, min(a.steps, REF_BUDGET_S // max(t_it, 1e-9))))
    times, passes = [], 0
    for _ in range(steps):
        t1 = time.perf_counter()
        passes += int(run.step(1).sum())
        times.append(time.perf_counter() - t1)
    total = sum(times)
    rate = steps / total
    out = {
        "metric": METRIC, "value": round(rate, 6), "unit": "iter/s", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": round(1e3 * total / steps, 3),
        "steps_requested": a.steps, "warmup_requested": a.warmup,
        "higher_is_better": True, "scaling": "strong",  # one fixed market at every N
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"BASELINE config {a.config[1]}: {CONFIG_TEXT[a.config]}",
                   "n_buyers": n, "m_goods": m, "nnz": nnz, "seed": a.seed,
                   "row_solver": "ksection (sections 32, subproblem_tol 1e-10)",
                   "tau": run.tau, "sigma": run.sigma},
        "cpu_baseline": {"value": round(rate, 6), "unit": "iter/s", "cores": threads,
                         "kind": "port",
                         "sample": f"the whole market every step: iterations {warm + 1}.."
                                   f"{warm + steps} from the initial state of the C "
                                   "oracle (restated kernels.pdhcg_chunk, bit-identical to the "
                                   "reference's numba kernel), tau/sigma of the solver's first "
                                   "restart window"},
        "e2e": {"value": round(rate, 6), "unit": "iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "passes_per_row_per_iteration": round(passes / steps / n, 3),
        "generate_seconds": round(gen_s, 2), "setup_seconds": round(setup_s, 2),
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
