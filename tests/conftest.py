import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

STATE_KEYS = ("x", "y", "z", "lam", "gamma", "delta")
REPORT_FIELDS = ("iter", "prim_res_inf", "prim_res_2", "dual_res_inf", "dual_res_2", "stat_res_inf",
                 "stat_res_2", "ax_inf", "atl_inf", "cone_gap", "pobj", "dobj", "gap")
STATUS = ("running", "solved", "max_iters", "diverged")
ITERATE_CASES = ("lp_mu1", "lp_mu03", "socp4_mu5", "socp4_mu07_warm", "lp_raw_mu1_warm", "mixed_cones")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel_err(got, want):
    """max|got - want| / (1 + max|want|) — the reference's parity metric (pkg/tests/conftest.py:32-37)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    if want.size == 0:
        return 0.0
    return float(np.max(np.abs(got - want)) / (1.0 + np.max(np.abs(want))))


def problem_from(d, prefix=""):
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix

    m, n = int(d[prefix + "m"]), int(d[prefix + "n"])
    a = TripletMatrix(m, n, d[prefix + "rows"], d[prefix + "cols"], d[prefix + "vals"])
    return ProblemInstance(a, d[prefix + "b"], d[prefix + "c"], ConeSpec(d[prefix + "block_sizes"]))


def init_from(d):
    from paper_2203_05027_b200 import SolverState

    if "init_x" not in d.files:
        return None
    return SolverState(**{k: d["init_" + k].copy() for k in STATE_KEYS})


@pytest.fixture(scope="session")
def has_gpu():
    from paper_2203_05027_b200 import _lib

    return _lib.device_count() > 0
