"""Host logic of the drop-in API (CPU): config validation, termination semantics,
error paths that never reach the GPU, and the C-ABI library surface."""

import math
import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import ROOT

from paper_2203_05027_b200 import (ConeSpec, IterationReport, ProblemInstance, SolverConfig, TripletMatrix,
                                   check_termination, solve)
from paper_2203_05027_b200 import _lib
from paper_2203_05027_b200.api import _decide, norms
from paper_2203_05027_b200.engine import config_struct


def test_config_defaults_and_errors():
    cfg = SolverConfig()
    assert (cfg.mu, cfg.max_iters, cfg.check_every, cfg.term_mode) == (1.0, 100_000, 25, "scs")
    assert (cfg.eps_abs, cfg.eps_rel, cfg.eps_prim, cfg.eps_dual, cfg.eps_gap) == (1e-4, 1e-3, 1e-3, 1e-3, 1e-3)
    for kw, msg in ((dict(mu=0.0), "mu must be > 0"), (dict(max_iters=0), "max_iters"),
                    (dict(check_every=0), "check_every"), (dict(term_mode="x"), "term_mode"),
                    (dict(eps_gap=-1.0), "eps_gap must be >= 0"), (dict(term_mode="target"), "target mode")):
        with pytest.raises(ValueError, match=msg):
            SolverConfig(**kw)


def _rep(**kw):
    base = dict(iter=25, prim_res_inf=0.0, prim_res_2=0.0, dual_res_inf=0.0, dual_res_2=0.0, stat_res_inf=0.0,
                stat_res_2=0.0, ax_inf=0.0, atl_inf=0.0, cone_gap=0.0, pobj=0.0, dobj=0.0, gap=0.0)
    base.update(kw)
    return IterationReport(**base)


P = SimpleNamespace(b=np.array([3.0, 4.0]), c=np.array([1.0, 0.0]))


def test_zero_residuals_solved_in_every_mode():
    for cfg in (SolverConfig(), SolverConfig(term_mode="osqp"),
                SolverConfig(term_mode="target", target_prim_res=1e-3, target_gap=1e-3)):
        assert check_termination(_rep(), cfg, P) == "solved"


def test_scs_bound_is_inclusive_and_osqp_strict():
    cfg = SolverConfig()
    bound = cfg.eps_prim * (1.0 + 5.0)  # ||b||_2 = 5
    assert check_termination(_rep(prim_res_2=bound), cfg, P) == "solved"
    assert check_termination(_rep(prim_res_2=math.nextafter(bound, 1.0)), cfg, P) == "running"
    ocfg = SolverConfig(term_mode="osqp")
    ep = ocfg.eps_abs + ocfg.eps_rel * 4.0
    assert check_termination(_rep(prim_res_inf=ep), ocfg, P) == "running"
    assert check_termination(_rep(prim_res_inf=math.nextafter(ep, 0.0)), ocfg, P) == "solved"


def test_stationarity_not_dual_residual_drives_the_test():
    # solver.py:259,263 use stat_res, not dual_res
    cfg = SolverConfig()
    assert check_termination(_rep(dual_res_2=1e6, dual_res_inf=1e6), cfg, P) == "solved"
    assert check_termination(_rep(stat_res_2=1.0), cfg, P) == "running"


def test_diverged_passthrough():
    assert check_termination(_rep(status="diverged"), SolverConfig(), P) == "diverged"


def test_config_struct_bounds_match_python_expressions():
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=2e-4, eps_gap=3e-4)
    b, c = np.array([1.0, -2.0, 2.0]), np.array([0.5, 0.25])
    s = config_struct(cfg, norms(b), norms(c))
    assert s.scs_prim_bound == cfg.eps_prim * (1.0 + math.sqrt(np.dot(b, b)))
    assert s.scs_dual_bound == cfg.eps_dual * (1.0 + math.sqrt(np.dot(c, c)))
    assert (s.b_inf, s.c_inf, s.term_mode, s.max_iters) == (2.0, 0.5, 1, 100_000)


def test_host_detectable_errors_raise_before_the_device():
    a = TripletMatrix(2, 2, [0, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError, match=r"invalid problem: b has length 3 != m=2"):
        solve(ProblemInstance(a, np.zeros(3), np.zeros(2), ConeSpec.orthant(2)))
    with pytest.raises(ValueError, match=r"cone sizes sum 3 != n=2"):
        solve(ProblemInstance(a, np.zeros(2), np.zeros(2), ConeSpec((3,))))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "cfb200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cf_[A-Za-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    names = _header_functions()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, name
    assert lib.cf_abi_version() == 1


def test_plan_create_argument_checks():
    """cf_plan_create rejects bad sizes before touching CUDA: negative sizes, the int32 limit
    of the tile indices (m, n, o < 2^31), NULL arrays and cone sizes that do not sum to n."""
    import ctypes

    L = _lib.lib()
    out = ctypes.c_void_p()
    chk = _lib.CfChecks()
    sizes = (ctypes.c_int64 * 2)(2, 2)
    one = (ctypes.c_int64 * 1)(0)
    val = (ctypes.c_double * 1)(1.0)
    cvec = (ctypes.c_double * 5)(1.0, 1.0, 1.0, 1.0, 1.0)   # c for every n below

    def create(m, n, o, rows, vals, nb, bs):
        return L.cf_plan_create(m, n, o, rows, rows, vals, vals, cvec, nb, bs, 0, None, ctypes.byref(chk),
                                ctypes.byref(out))

    cases = [
        ((-1, 1, 1, one, val, 0, None), "negative size"),
        ((1, 2 ** 31, 1, one, val, 0, None), "< 2\\^31"),
        ((1, 1, 2 ** 31 - 1, one, val, 0, None), "< 2\\^31"),
        ((1, 1, 1, None, val, 0, None), "NULL input array"),
        ((1, 4, 1, one, val, 2, ctypes.cast(sizes, ctypes.c_void_p)), None),   # sums to 4: passes the checks
        ((1, 5, 1, one, val, 2, ctypes.cast(sizes, ctypes.c_void_p)), "cone sizes sum 4 != n=5"),
    ]
    for args, msg in cases:
        rc = create(*args)
        if msg is None:
            assert rc != _lib.CF_EINVAL or "cone" not in _lib.last_error()
            if rc == 0:
                L.cf_plan_destroy(out)
            continue
        assert rc == _lib.CF_EINVAL, (args, rc)
        assert re.search(msg, _lib.last_error()), (msg, _lib.last_error())
        assert not out.value


def test_no_gpu_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    a = TripletMatrix(1, 1, [0], [0], [1.0])
    with pytest.raises(_lib.CfError, match="no CUDA device"):
        solve(ProblemInstance(a, [1.0], [1.0], ConeSpec.orthant(1)))


def test_decide_max_iters_passthrough():
    assert _decide(_rep(status="max_iters"), SolverConfig(), (0.0, 0.0), (0.0, 0.0)) == "max_iters"


def test_benchrun_csv_and_shapes():
    """benchrun mirrors bench.py's CSV layout and shape_for_nnz (bench.py:48-55, 109-119)."""
    import math

    from paper_2203_05027_b200.benchrun import BENCH_COLUMNS, bench_csv, shape_for_nnz

    assert BENCH_COLUMNS[0] == "instance_id" and BENCH_COLUMNS[-1] == "status" and len(BENCH_COLUMNS) == 15
    for nnz, dens, kind in ((20_000, 0.01, "lp"), (1_000, 0.05, "lp"), (40_000_000, 5e-6, "socp4")):
        cells = nnz / dens
        m = max(1, round(math.sqrt(cells / 4.0)))
        n = max(1, round(cells / m))
        if kind == "socp4":
            n = max(4, 4 * round(n / 4))
        assert shape_for_nnz(nnz, dens, kind) == (m, n)
    row = {c: 0 for c in BENCH_COLUMNS}
    row.update({"density": 0.1, "time_ms": 1.5, "status": "solved", "cone_kind": "lp", "term_mode": "scs"})
    text = bench_csv([row])
    assert text.splitlines()[1].split(",")[4] == "0.1" and text.endswith("\n")
