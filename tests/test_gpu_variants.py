"""The checked build (CF_CHECKED=1, libcfb200_checked.so built by __graft_entry__.build():
device bounds asserts + buffer guard canaries) passes the same golden iterate parity as
the product build: run in a subprocess with CF_LIB_PATH pointing at the variant library.
(The round-1 TMA-ring engine variant was removed in round 2 with the tile-ranked JDS
layout; it had measured 1-3 % slower.)"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
from conftest import load_golden, problem_from, init_from, rel_err
from paper_2203_05027_b200 import _lib
assert _lib.LIB_PATH.endswith("libcfb200_checked.so"), _lib.LIB_PATH
from paper_2203_05027_b200.api import build_plan
for case in ("lp_mu1", "socp4_mu5", "mixed_cones", "lp_raw_mu1_warm"):
    g = load_golden("iterates_" + case + ".npz")
    p = problem_from(g)
    mu = float(g["mu"])
    worst = 0.0
    with build_plan(p) as plan:
        plan.set_state(mu, init_from(g))
        done = 0
        for k in g["keep"]:
            plan.iterate(mu, int(k) - done)
            done = int(k)
            st = plan.get_state()
            for key in ("x", "y", "z", "lam", "gamma", "delta"):
                worst = max(worst, rel_err(st[key], g["k%d_%s" % (k, key)]))
    assert worst <= 1e-9, (case, worst)
assert _lib.lib().cf_debug_guard_violations() == 0
print("ok")
"""


def test_checked_build_iterate_parity():
    lib = os.path.join(ROOT, "paper_2203_05027_b200", "libcfb200_checked.so")
    if not os.path.exists(lib):
        pytest.fail("libcfb200_checked.so missing: run __graft_entry__.build()")
    env = dict(os.environ, CF_LIB_PATH=lib)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
