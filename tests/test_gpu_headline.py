"""Parity at the BASELINE sizes (C2: 1e8 nonzeros, C3: 4e7 with 1M K4 cones).

The exact bench instances (cfgen, seed 0 — bit-identical on host and device,
tests/test_gpu_gen.py) are iterated on the GPU and, from the same arrays copied to the
host, by the oracle port (the literal per-nonzero reference iteration, solver.py:168-197,
pinned bit-for-bit to the reference in tests/test_oracle_golden.py). All six state
vectors (y and gamma rebuilt by the export) must agree, and the report too.

Tolerances (north_star: iterates <= 1e-9 relative over the first 100 iterations):
  * state vectors: rel_err = max|got - want| / (1 + max|want|) <= 1e-9
  * report fields: |got - want| / (1 + |want|) <= 1e-9
  * time to 1e-4 (fixtures from the UNMODIFIED reference, tests/golden/make_headline_golden.py):
    the same status, the iteration count within +-check_every (25; measured: equal),
    every report of the trace to 1e-6 relative (the iterates agree to ~1e-13 per iteration;
    after ~1e4 iterations the drift is far below the solve tolerance 1e-4), x / lam to 1e-6.
The oracle's factors are built from the device instance's arrays, which are already in
canonical order (asserted), i.e. build_uv's lexsort (uv.py:76) is the identity on them.
"""

import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, REPORT_FIELDS, STATE_KEYS, rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2203_05027_b200 import cfgen  # noqa: E402

ITER_TOL = 1e-9
REPORT_TOL = 1e-9
TTT_TOL = 1e-6


def _factors(inst):
    rows, cols, vals = (t.cpu().numpy() for t in (inst.rows, inst.cols, inst.vals))
    assert np.all(np.diff(cols * inst.m + rows) > 0), "instance arrays are canonical"
    fu = 1.0 / (1.0 + np.bincount(rows, weights=vals * vals, minlength=inst.m))     # uv.py:81
    fv = 1.0 / (1.0 + np.bincount(cols, minlength=inst.n))                           # uv.py:82
    return oracle.Factors(inst.m, inst.n, int(vals.size), rows, cols, vals, fu, fv)


def _iterate_and_compare(m, n, dens, kind, iters, check_at):
    inst = cfgen.generate_device(m, n, dens, kind, 0)
    plan = inst.plan
    try:
        f = _factors(inst)
        b, c = inst.b.cpu().numpy(), inst.c.cpu().numpy()
        sizes = np.asarray(inst.block_sizes, dtype=np.int64)
        st = oracle.OracleState.zeros(f)
        plan.set_state(1.0, None, export=True)
        done = 0
        for k in range(1, iters + 1):
            st = oracle.step(f, sizes, st, 1.0, b, c)
            if k not in check_at:
                continue
            plan.iterate(1.0, k - done)
            done = k
            got = plan.get_state()
            assert got["iter"] == k
            for key in STATE_KEYS:
                err = rel_err(got[key], getattr(st, key))
                assert err <= ITER_TOL, f"k={k} {key}: rel_err {err:.3e}"
            rep = plan.report(1.0)
            want = oracle.compute_report(f, st, b, c)
            for fld in REPORT_FIELDS[1:]:
                e = abs(rep[fld] - want[fld]) / (1.0 + abs(want[fld]))
                assert e <= REPORT_TOL, f"k={k} {fld}: {rep[fld]!r} vs {want[fld]!r}"
            del got
    finally:
        plan.close()
        torch.cuda.synchronize()


def test_c2_exact_instance_first_iterations():
    """C2 (m=5M, n=10M, o=1e8): iterations 1..3 from a cold start, all six vectors."""
    _iterate_and_compare(5_000_000, 10_000_000, 2e-6, "lp", 3, {1, 3})


def test_c3_exact_instance_first_iterations():
    """C3 (m=2M, n=4M, o=4e7, 1M K4 cones): iterations 1..3 from a cold start."""
    _iterate_and_compare(2_000_000, 4_000_000, 5e-6, "socp4", 3, {1, 3})


def test_c2_structure_1e7_first_25_iterations():
    """C2 structure at 1e7 nonzeros (20 per row): iterations 1..25, checked at 1, 10, 25."""
    _iterate_and_compare(500_000, 1_000_000, 2e-5, "lp", 25, {1, 10, 25})


@pytest.mark.parametrize("case", ["c2s_1e5", "c3s_20"])
def test_time_to_tolerance_matches_reference(case):
    """solve() to scs 1e-4 at the C2 / C3 structures against the reference's own solve."""
    from paper_2203_05027_b200 import SolverConfig, solve

    path = os.path.join(GOLDEN, f"headline_{case}.npz")
    d = np.load(path, allow_pickle=False)
    m, n, dens, kind = int(d["m"]), int(d["n"]), float(d["density"]), str(d["kind"])
    inst = cfgen.generate_device(m, n, dens, kind, 0, keep_plan=False)
    assert cfgen.fingerprint(inst.rows, inst.cols, inst.vals, inst.b, inst.c) == str(d["fingerprint"])
    from paper_2203_05027_b200.devgen import to_host_problem

    p = to_host_problem(inst)
    del inst
    res = solve(p, SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4))
    want = d["trace"]
    assert res.report.status == str(d["status"][-1])
    assert abs(res.report.iter - int(want[-1, 0])) <= 25, (res.report.iter, int(want[-1, 0]))
    k = min(len(res.trace), len(want))
    for i in range(k):
        got = res.trace[i]
        assert got.iter == int(want[i, 0])
        for j, fld in enumerate(REPORT_FIELDS[1:], start=1):
            e = abs(getattr(got, fld) - want[i, j]) / (1.0 + abs(want[i, j]))
            assert e <= TTT_TOL, f"report {got.iter} {fld}: {getattr(got, fld)!r} vs {want[i, j]!r}"
    if "x" in d.files:
        assert rel_err(res.x, d["x"]) <= TTT_TOL and rel_err(res.lam, d["lam"]) <= TTT_TOL
    else:
        assert rel_err(res.x[d["x_idx"]], d["x_sub"]) <= TTT_TOL
        assert rel_err(res.lam[d["lam_idx"]], d["lam_sub"]) <= TTT_TOL
        assert abs(np.linalg.norm(res.x) - float(d["x_norm"])) <= TTT_TOL * float(d["x_norm"])
