"""Command line (market_eq/cli.py): `python -m paper_2506_06258_b200
{generate,solve,check,bench,exchange} ...` with the reference's commands,
flags, outputs and exit codes: 0 done (solver optimal / check ran / files
written), 1 usage error, 2 solver stopped unsolved, 3 data or I/O failure.
MARKET_EQ_LOG (error | info | debug) sets the stderr log level.
"""

import argparse
import csv
import json
import logging
import math
import os
import sys

from . import fileio
from .driver import SolveConfig, run_solve
from .errors import MarketError
from .exchange import solve_exchange, verify_fixed_point
from .instance import (ExchangeInstance, FisherInstance, GeneratorConfig, generate_exchange,
                       generate_fisher)
from .kkt import residuals_compact, residuals_lifted
from .report import SolveReport, instance_fingerprint

OK, USAGE, UNSOLVED, DATA = 0, 1, 2, 3
log = logging.getLogger("market_eq")


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1, not argparse's 2
        self.print_usage(sys.stderr)
        self.exit(USAGE, f"{self.prog}: error: {message}\n")


def _solver_config(a):
    if a.restart == "adaptive":
        restart, k = "adaptive", 0
    elif a.restart.startswith("fixed:"):
        restart, k = "fixed", int(a.restart.split(":", 1)[1])
    else:
        raise ValueError(f"bad --restart value {a.restart!r}")
    return SolveConfig(tol=a.tol, max_iters=a.max_iters, restart=restart, restart_k=k,
                       sections=a.sections, step_mode=a.step, threads=a.threads,
                       check_every=a.check_every, subproblem_tol=a.subproblem_tol)


def _emit(payload):
    print(json.dumps(payload))


def generate(a):
    g = GeneratorConfig(n=a.n, m=a.m, sparsity_u=a.sparsity_u, sparsity_e=a.sparsity_e,
                        seed=a.seed)
    inst = generate_fisher(g) if a.kind == "fisher" else generate_exchange(g)
    written = fileio.save(inst, a.out, fmt=a.format)
    _emit({"written": written, "fingerprint": instance_fingerprint(inst),
           "nnz_u": inst.utilities.nnz})
    return OK


def solve(a):
    inst = fileio.load(a.instance, fmt=a.format)
    if not isinstance(inst, FisherInstance):
        raise MarketError("solve expects a Fisher instance (with budgets); "
                          "use the exchange command for endowment instances")
    rep = run_solve(inst, _solver_config(a), algo=a.algo)
    path = a.out or f"{a.instance}.report.json"
    rep.to_json(path)
    _emit({"status": rep.status, "inner_iterations": rep.inner_iterations,
           "restarts": rep.restarts, "rel_kkt": rep.final_residuals.rel_kkt,
           "wall_time_seconds": rep.wall_time_seconds, "report": path})
    return OK if rep.status == "optimal" else UNSOLVED


def check(a):
    inst = fileio.load(a.instance, fmt=a.format)
    if isinstance(inst, ExchangeInstance):
        raise MarketError("check expects a Fisher instance")
    rep = SolveReport.from_json(a.solution)
    if rep.solver == "pdhg" and rep.utility_values is not None:
        res = residuals_lifted(inst, rep.allocation, rep.utility_values, rep.prices,
                               rep.dual_values)
    else:
        res = residuals_compact(inst, rep.allocation, rep.prices)
    out = res.as_dict()
    out["matches_report"] = bool(abs(res.rel_kkt - rep.final_residuals.rel_kkt) <= 1e-12)
    text = json.dumps(out, indent=2)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text + "\n")
    print(text)
    return OK


def _geomean(v):
    return math.exp(sum(math.log(max(x, 1e-300)) for x in v) / len(v))


def bench(a):
    with open(a.suite) as fh:
        suite = json.load(fh)
    solvers, seeds = suite.get("solvers", ["pdhcg", "pdhg"]), suite.get("seeds", [0])
    if a.report_dir:
        os.makedirs(a.report_dir, exist_ok=True)
    rows = []
    for c in suite["configs"]:
        for solver in solvers:
            its, secs, ok = [], [], []
            for seed in seeds:
                inst = generate_fisher(GeneratorConfig(n=c["n"], m=c["m"],
                                                       sparsity_u=c["sparsity_u"],
                                                       sparsity_e=c.get("sparsity_e", 0.5),
                                                       seed=seed))
                cfg = SolveConfig(tol=c.get("tol", 1e-4), max_iters=c.get("max_iters", 100_000),
                                  sections=c.get("sections", 32), threads=a.threads)
                rep = run_solve(inst, cfg, algo=solver)
                its.append(rep.inner_iterations)
                secs.append(rep.wall_time_seconds)
                ok.append(rep.status == "optimal")
                if a.report_dir:
                    rep.to_json(os.path.join(
                        a.report_dir, f"n{c['n']}_m{c['m']}_q{c['sparsity_u']}_{solver}_s{seed}.json"))
            rows.append({"n": c["n"], "m": c["m"], "sparsity_u": c["sparsity_u"],
                         "solver": solver, "seeds": len(seeds),
                         "geomean_iterations": _geomean(its),
                         "geomean_time_seconds": _geomean(secs), "all_optimal": all(ok)})
    fields = ["n", "m", "sparsity_u", "solver", "seeds", "geomean_iterations",
              "geomean_time_seconds", "all_optimal"]
    fh = open(a.out, "w", newline="") if a.out else sys.stdout
    try:
        w = csv.DictWriter(fh, fieldnames=fields)
        w.writeheader()
        w.writerows(rows)
    finally:
        if a.out:
            fh.close()
    return OK if all(r["all_optimal"] for r in rows) else UNSOLVED


def exchange(a):
    inst = fileio.load(a.instance, fmt=a.format)
    if not isinstance(inst, ExchangeInstance):
        raise MarketError("exchange expects an instance with endowments")
    cfg = _solver_config(a)
    trace = solve_exchange(inst, outer_tol=a.outer_tol, max_outer=a.max_outer,
                           inner_config=cfg)
    path = a.out or f"{a.instance}.trace.json"
    trace.to_json(path)
    out = {"status": trace.status, "outer_iterations": trace.outer_iterations,
           "final_gap": trace.budget_gaps[-1] if trace.budget_gaps else None, "trace": path}
    if trace.status == "converged" and a.verify:
        gap, _ = verify_fixed_point(inst, trace.final_budgets, inner_tol=a.outer_tol / 100.0,
                                    inner_config=cfg)
        out["verified_fixed_point_gap"] = gap
    if trace.inner_reports:
        rpath = path.replace(".trace.json", ".report.json")
        rpath = rpath if rpath != path else path + ".report.json"
        trace.inner_reports[-1].to_json(rpath)
        out["final_inner_report"] = rpath
    _emit(out)
    return OK if trace.status == "converged" else UNSOLVED


def _solver_flags(p):
    p.add_argument("--algo", choices=("pdhg", "pdhcg"), default="pdhcg")
    p.add_argument("--tol", type=float, default=1e-4)
    p.add_argument("--max-iters", type=int, default=100_000)
    p.add_argument("--restart", default="adaptive", help="'adaptive' or 'fixed:K'")
    p.add_argument("--sections", type=int, default=32)
    p.add_argument("--step", choices=("theory", "adaptive"), default="adaptive")
    p.add_argument("--threads", type=int, default=1)
    p.add_argument("--check-every", type=int, default=40)
    p.add_argument("--subproblem-tol", type=float, default=1e-10)


def build_parser():
    top = _ArgParser(prog="market-eq", description="market equilibrium solvers on a B200")
    sub = top.add_subparsers(dest="command", required=True)
    fmt = dict(choices=fileio.FORMATS, default="mtx")

    p = sub.add_parser("generate", help="write a synthetic instance")
    p.add_argument("--kind", choices=("fisher", "exchange"), default="fisher")
    p.add_argument("--n", type=int, required=True)
    p.add_argument("--m", type=int, required=True)
    p.add_argument("--sparsity-u", type=float, default=0.2)
    p.add_argument("--sparsity-e", type=float, default=0.5)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--format", **fmt)
    p.add_argument("--out", required=True, help="path prefix for the instance files")
    p.set_defaults(func=generate)

    p = sub.add_parser("solve", help="solve a Fisher instance")
    p.add_argument("--instance", required=True, help="instance path prefix")
    p.add_argument("--format", **fmt)
    _solver_flags(p)
    p.add_argument("--out", help="report path (default <instance>.report.json)")
    p.set_defaults(func=solve)

    p = sub.add_parser("check", help="recompute residuals of a solve report")
    p.add_argument("--instance", required=True)
    p.add_argument("--format", **fmt)
    p.add_argument("--solution", required=True, help="solve report JSON")
    p.add_argument("--out")
    p.set_defaults(func=check)

    p = sub.add_parser("bench", help="run a benchmark suite file")
    p.add_argument("--suite", required=True, help="suite JSON file")
    p.add_argument("--out", help="CSV output (default stdout)")
    p.add_argument("--report-dir", help="write per-seed reports here")
    p.add_argument("--threads", type=int, default=1)
    p.set_defaults(func=bench)

    p = sub.add_parser("exchange", help="solve an Arrow-Debreu exchange instance")
    p.add_argument("--instance", required=True)
    p.add_argument("--format", **fmt)
    p.add_argument("--outer-tol", type=float, default=1e-6)
    p.add_argument("--max-outer", type=int, default=100)
    p.add_argument("--verify", action="store_true",
                   help="re-solve tightly and report the true fixed-point gap")
    _solver_flags(p)
    p.add_argument("--out", help="trace path (default <instance>.trace.json)")
    p.set_defaults(func=exchange)
    return top


def main(argv=None):
    level = {"error": logging.ERROR, "info": logging.INFO, "debug": logging.DEBUG}.get(
        os.environ.get("MARKET_EQ_LOG", "error").lower(), logging.ERROR)
    h = logging.StreamHandler(sys.stderr)
    h.setFormatter(logging.Formatter("%(levelname)s %(name)s: %(message)s"))
    log.addHandler(h)
    log.setLevel(level)
    a = build_parser().parse_args(argv)
    try:
        return a.func(a)
    except (MarketError, ValueError, OSError) as exc:
        print(f"market-eq: {exc}", file=sys.stderr)
        return DATA
