"""GPU run_bench against the reference's own run_bench rows (tests/golden/bench_rows.npz).

Every deterministic column (bench.py:22-38 minus time_ms) must match; the
residual columns to 1e-9 relative (the iterates differ only by rounding)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_run_bench_matches_reference_rows():
    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.benchrun import BENCH_COLUMNS, BenchJob, bench_csv, run_bench
    from paper_2203_05027_b200.instances import GenSpec

    g = load_golden("bench_rows.npz")
    cfg = SolverConfig(term_mode="scs", eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    jobs = [BenchJob(int(i), GenSpec(int(m), int(n), float(d), str(k), int(s)), cfg)
            for (i, m, n, s), d, k in zip(g["jobs"], g["densities"], g["kinds"])]
    rows = run_bench(jobs)
    assert [r["instance_id"] for r in rows] == list(g["instance_id"])
    for k in ("m", "n", "nnz", "iters"):
        assert [r[k] for r in rows] == [int(v) for v in g[k]], k
    for k in ("density", "mu"):
        assert [r[k] for r in rows] == [float(v) for v in g[k]], k
    for k in ("cone_kind", "term_mode", "status"):
        assert [r[k] for r in rows] == [str(v) for v in g[k]], k
    for k in ("prim_res_2", "dual_res_2", "gap", "cone_gap"):
        got = np.array([r[k] for r in rows])
        want = g[k]
        assert np.all(np.abs(got - want) <= 1e-9 * np.maximum(1.0, np.abs(want))), k
    csv = bench_csv(rows)
    assert csv.splitlines()[0] == ",".join(BENCH_COLUMNS)
    assert len(csv.splitlines()) == len(rows) + 1
    extra = bench_csv(rows, extra=True).splitlines()[0].split(",")
    assert extra[-3:] == ["iters_per_s", "hbm_gbs", "roofline_frac"]


def test_concurrent_large_jobs_equal_serial():
    """Jobs above the batch threshold solved 4 at a time (threads, one plan and stream
    each) give exactly the serial rows."""
    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.benchrun import BenchJob, run_bench
    from paper_2203_05027_b200.instances import GenSpec

    cfg = SolverConfig(max_iters=2000)
    jobs = [BenchJob(i, GenSpec(300, 900, 0.1, "lp" if i % 2 else "socp4", seed=i), cfg) for i in range(6)]
    par = run_bench(jobs, workers=4, batch_max_nnz=1000)
    ser = run_bench(jobs, workers=1, batch_max_nnz=1000)
    keys = ("instance_id", "iters", "prim_res_2", "dual_res_2", "gap", "cone_gap", "status")
    assert [[r[k] for k in keys] for r in par] == [[r[k] for k in keys] for r in ser]
