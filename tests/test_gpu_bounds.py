"""Memory safety without compute-sanitizer (closed on the GPU pool): the
library rebuilt with -DMQ_DEBUG_BOUNDS (device asserts on every index the
new kernels form — entries, goods, slots, list rows, row lengths) runs the
whole-library workload of tools/sanitize_run.py (tile / screened / full /
medium / long row kernels, rebuilds, k-section drop-in, residuals, restart
moves, lifted PDHG, theory diagnostics, exchange); a failed check traps and
fails the run."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_build_runs_the_workload_clean():
    from paper_2506_06258_b200 import _build

    lib = os.path.join(ROOT, "paper_2506_06258_b200", "libmarket_eq_b200_checked.so")
    _build.build(extra_flags=("-DMQ_DEBUG_BOUNDS",), out=lib)  # cached by source digest
    env = dict(os.environ, MQ_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")],
                       env=env, capture_output=True, text=True, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "sanitize workload ok" in r.stdout
    assert "Assertion" not in r.stderr
