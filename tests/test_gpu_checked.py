"""Memory safety under the checked build (libcfb200_checked.so, -DCF_CHECKED=1).

compute-sanitizer is closed on the GPU pool. The checked build instead asserts, on the
device, every index the passes and the on-chip solvers dereference (idx/val positions,
gathered indices, tile bounds, shared-memory CSR/CSC indices) and places canaries behind
every device buffer, verified when the buffer is released (cf_debug_guard_violations).
Each engine is driven through the C ABI on small instances (tools/sanitize_cases.py) and
its result is checked against the oracle; a trap, a canary hit or a wrong answer fails.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2203_05027_b200", "libcfb200_checked.so")


@pytest.mark.parametrize("case", ["plan", "plan_knobs", "cluster1", "cluster8", "cluster16", "batch", "gen"])
def test_checked_build_case(case):
    if not os.path.exists(CHECKED):
        pytest.fail("libcfb200_checked.so missing: build with __graft_entry__.build()")
    env = dict(os.environ, CF_LIB_PATH=CHECKED)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), case], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert f"case {case}: ok (guard violations: 0)" in out.stdout, out.stdout[-2000:]
