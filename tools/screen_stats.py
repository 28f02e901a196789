"""Safe-screening statistics of the PDHCG row solve (design experiment).

    python tools/screen_stats.py [c4|c3|c2] [K1,K2,...]

For each K: solve K iterations (the real restarted loop), then step the
iterate 41 more iterations one at a time and measure, for several margins
gamma:
  * near fraction: zero entries with p_j s_i / (w_i u_ij) < gamma (they would
    still be gathered every iteration), plus the nonzero entries;
  * certificate pass rate d iterations after a refresh at d=0: per row
    theta_i (1 - D_d / P_i) s_i^(d) >= w_i, theta_i = min over screened
    entries of p_j/u_ij, P_i = min of their p_j, D_d = sum of the per-iteration
    maximum price decrease;
  * the true rate (every screened entry still inactive at iteration d).
"""

import json
import os
import sys
import time
from types import SimpleNamespace

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GAMMAS = [1.02, 1.05, 1.1, 1.2, 1.5, 2.0]
CHUNK = 100_000_000


def row_stats(dm, eng, p, s, gammas):
    """(near fraction per gamma, theta [G, n], P [G, n])"""
    n = dm.n
    rp = dm.row_ptr
    G = len(gammas)
    theta = torch.full((G, n), float("inf"), dtype=torch.float64, device="cuda")
    pmin = torch.full((G, n), float("inf"), dtype=torch.float64, device="cuda")
    near = torch.zeros(G, dtype=torch.float64, device="cuda")
    nz = 0
    r0 = 0
    rpc = rp.cpu()
    while r0 < n:
        r1 = int(torch.searchsorted(rpc, rpc[r0] + CHUNK, right=True).item()) - 1
        r1 = max(r1, r0 + 1)
        r1 = min(r1, n)
        e0, e1 = int(rpc[r0]), int(rpc[r1])
        lens = (rp[r0 + 1:r1 + 1] - rp[r0:r1])
        rows = torch.repeat_interleave(torch.arange(r0, r1, device="cuda"), lens)
        col = dm.col[e0:e1].long()
        u = dm.u[e0:e1]
        x = eng.x[e0:e1]
        pc = p[col]
        t = pc * s[rows] / (dm.w[rows] * u)
        zero = x <= 0
        nz += int((~zero).sum().item())
        for g, gam in enumerate(gammas):
            scr = zero & (t >= gam)
            near[g] += (zero & ~scr).sum()
            lr = rows - r0
            th = torch.where(scr, pc / u, torch.full_like(pc, float("inf")))
            pm = torch.where(scr, pc, torch.full_like(pc, float("inf")))
            theta[g, r0:r1] = theta[g, r0:r1].scatter_reduce(0, lr, th, "amin")
            pmin[g, r0:r1] = pmin[g, r0:r1].scatter_reduce(0, lr, pm, "amin")
        del rows, col, u, x, pc, t, zero
        r0 = r1
    frac = ((near + nz) / dm.nnz).tolist()
    return frac, nz / dm.nnz, theta, pmin


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    Ks = [int(k) for k in (sys.argv[2] if len(sys.argv) > 2 else "400,4000,16000").split(",")]
    from bench import make_session, shard_rows  # noqa: F401
    from paper_2506_06258_b200.device import DeviceMarket
    from paper_2506_06258_b200.driver import SolveConfig, solve_on_device
    from paper_2506_06258_b200.engine import PdhcgEngine
    from paper_2506_06258_b200.sparse import selector_norm_from_counts

    shard = shard_rows(cfg, 0, 1, 0)
    dm = DeviceMarket(shard["row_ptr"], shard["col"], shard["u"], shard["w"], shard["m"])
    del shard
    out = {"config": cfg, "gammas": GAMMAS, "runs": []}
    for K in Ks:
        eng = PdhcgEngine(dm)
        sess = SimpleNamespace(dm=dm, engine=eng,
                               op_norm=selector_norm_from_counts(eng._global_counts().cpu().numpy()))
        eng.final_payload = lambda: {"prices": None, "allocation": None, "utility_values": None,
                                     "dual_values": None, "objective": 0.0}
        t0 = time.time()
        rep = solve_on_device(sess, SolveConfig(tol=1e-9, max_iters=K),
                              w_sum=float(dm.w.sum().item()))
        print(f"K={K}: solved in {time.time() - t0:.1f}s restarts={rep.restarts}", flush=True)
        for _ in range(2):
            eng.run_chunk(1)
        p_ref = eng.p.clone()
        s_ref = eng.srow.clone()
        frac, nzf, theta, pmin = row_stats(dm, eng, p_ref, s_ref, GAMMAS)
        run = {"K": K, "gather_fraction": frac, "nonzero_fraction": nzf, "cert": [],
               "true_cert": []}
        has = torch.isfinite(theta)
        D = 0.0
        p_prev = p_ref
        for d in range(1, 41):
            eng.run_chunk(1)
            p = eng.p
            D += float((p_prev - p).clamp_min(0).max().item())
            p_prev = p.clone()
            s = eng.srow
            lhs = theta * (1.0 - D / pmin) * s[None, :]
            ok = (lhs >= dm.w[None, :]) | ~has
            rate = ok.double().mean(1).tolist()
            run["cert"].append([d, D] + rate)
            if d in (1, 5, 10, 20, 40):
                # true rate: every screened entry (w.r.t. d=0) still inactive
                f2, _, th2, _ = row_stats(dm, eng, p, s, [1.0])
                run["true_cert"].append([d, f2[0]])
                print(f"  d={d} D={D:.3e} cert={['%.4f' % r for r in rate]} "
                      f"active-frac(now)={f2[0]:.4f}", flush=True)
        print(f"  gather fraction by gamma: {['%.4f' % f for f in frac]} (nonzero {nzf:.4f})",
              flush=True)
        out["runs"].append(run)
        del eng, theta, pmin
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"screen_{cfg}.json"), "w") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
