"""The robust-least-squares SOC instance (SURVEY §8d secondary mixed-cone config, bench c3m).

CPU: the generator's structure. GPU: solve() on a small instance against the oracle
(same iteration count, x/lam to rel_err 1e-8, as the other solve parity tests)."""

import numpy as np
import pytest
import torch

from conftest import rel_err

from paper_2203_05027_b200.devgen import rls_arrays
from paper_2203_05027_b200.problem import ConeSpec, ProblemInstance, TripletMatrix, validate


def _instance(K, seed=0, per_row=13):
    m, n = 3 * K, 5 * K
    g = torch.Generator()
    g.manual_seed(seed)
    rows, cols, vals, b, c, sizes = rls_arrays(torch, g, m, n, per_row / n, "cpu")
    return ProblemInstance(TripletMatrix(m, n, rows.numpy(), cols.numpy(), vals.numpy()), b.numpy(), c.numpy(),
                           ConeSpec(sizes))


def test_rls_structure():
    K = 500
    p = _instance(K)
    assert validate(p).ok                      # distinct cells, nonzero finite values, cone sum = n
    a = p.A
    assert a.nnz == 3 * K * 13
    sizes = np.asarray(p.cones.block_sizes)
    assert (sizes[:K] == 4).all() and (sizes[K:] == 1).all() and sizes.sum() == 5 * K
    cols = np.asarray(a.cols)
    assert not np.isin(np.arange(0, 4 * K, 4), cols).any()     # the t columns are free of A
    np.testing.assert_array_equal(p.c[0:4 * K:4], 1.0)
    # +f on x+ and -f on x- for every F entry
    rows, vals = np.asarray(a.rows), np.asarray(a.vals)
    plus = cols >= 4 * K
    xp = plus & (cols < 4 * K + K // 2)
    xm = cols >= 4 * K + K // 2
    key_p = rows[xp] * K + (cols[xp] - 4 * K)
    key_m = rows[xm] * K + (cols[xm] - 4 * K - K // 2)
    op, om = np.argsort(key_p), np.argsort(key_m)
    np.testing.assert_array_equal(key_p[op], key_m[om])
    np.testing.assert_array_equal(vals[xp][op], -vals[xm][om])


@pytest.mark.gpu
def test_rls_solve_matches_oracle():
    import oracle
    from paper_2203_05027_b200 import SolverConfig, solve

    p = _instance(400, seed=3)
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=20000)
    ox, olam, otr, _ = oracle.solve(p, cfg)
    res = solve(p, cfg)
    assert res.report.iter == otr[-1]["iter"] and res.report.status == otr[-1]["status"] == "solved"
    assert rel_err(res.x, ox) <= 1e-8 and rel_err(res.lam, olam) <= 1e-8


@pytest.mark.gpu
def test_rls_column_runs_bit_identical(monkeypatch):
    """A pass large enough to launch per run of one cone size (K4 tiles with the warp-shuffle
    epilogue, orthant tiles fused, the one mixed tile with the group epilogue) gives the same
    bits as the group epilogue on every tile (CF_NO_COL_RUNS=1), and matches the oracle."""
    import oracle
    from paper_2203_05027_b200.api import build_plan

    p = _instance(120_000, seed=5)
    f = oracle.build_factors(p.A)
    st = oracle.OracleState.zeros(f)
    st = oracle.iterate(f, p.cones.sizes_array(), st, 1.0, p.b, p.c, 3)

    def run(env):
        if env:
            monkeypatch.setenv("CF_NO_COL_RUNS", "1")
        else:
            monkeypatch.delenv("CF_NO_COL_RUNS", raising=False)
        with build_plan(p) as plan:
            plan.set_state(1.0, None)
            plan.iterate(1.0, 3)
            s3 = plan.get_state()
            plan.iterate(1.0, 27)
            t = plan.last_timing()
            return s3, plan.get_state(), t["launches"]

    r3, r30, runs_launches = run(False)
    g3, g30, group_launches = run(True)
    assert runs_launches > group_launches      # the run dispatch was taken
    for key in ("x", "y", "z", "lam", "gamma", "delta"):
        np.testing.assert_array_equal(r30[key], g30[key])
        assert rel_err(r3[key], getattr(st, key)) <= 1e-9, key


def _cone_problem(sizes, m, per_col=8, seed=0):
    """Random sparse problem (distinct cells, ~per_col entries per column) with the given cones."""
    rng = np.random.default_rng(seed)
    sizes = np.asarray(sizes, dtype=np.int64)
    n = int(sizes.sum())
    cols = np.repeat(np.arange(n, dtype=np.int64), per_col)
    rows = rng.integers(0, m, size=cols.size, dtype=np.int64)
    key = np.unique(cols * m + rows)
    cols, rows = key // m, key % m
    vals = rng.standard_normal(rows.size)
    vals[vals == 0.0] = 1.0
    return ProblemInstance(TripletMatrix(m, n, rows, cols, vals), rng.standard_normal(m), rng.standard_normal(n),
                           ConeSpec(sizes))


@pytest.mark.gpu
@pytest.mark.parametrize("layout", ["runs", "interleaved"])
def test_column_runs_other_sizes(monkeypatch, layout):
    """Runs of K2, K8 and orthant cones (warp epilogues of sizes 2 and 8, fused orthant), and an
    interleaved K4/K1 pattern (too many runs: the group epilogue on every tile): bit-identical
    to CF_NO_COL_RUNS and to the oracle's first iterations."""
    import oracle
    from paper_2203_05027_b200.api import build_plan

    if layout == "runs":
        sizes = [2] * 100_000 + [8] * 25_000 + [1] * 120_000 + [8] * 20_000
    else:
        sizes = [4, 1, 1] * 80_000
    p = _cone_problem(sizes, m=200_000, seed=7 if layout == "runs" else 8)
    f = oracle.build_factors(p.A)
    st = oracle.iterate(f, p.cones.sizes_array(), oracle.OracleState.zeros(f), 1.0, p.b, p.c, 3)

    def run(no_runs):
        if no_runs:
            monkeypatch.setenv("CF_NO_COL_RUNS", "1")
        else:
            monkeypatch.delenv("CF_NO_COL_RUNS", raising=False)
        with build_plan(p) as plan:
            plan.set_state(1.0, None)
            plan.iterate(1.0, 3)
            s3 = plan.get_state()
            plan.iterate(1.0, 17)
            return s3, plan.get_state(), plan.last_timing()["launches"]

    r3, r20, nl_runs = run(False)
    _, g20, nl_group = run(True)
    if layout == "runs":
        assert nl_runs > nl_group
    else:
        assert nl_runs == nl_group             # too many runs: one launch per pass
    for key in ("x", "y", "z", "lam", "gamma", "delta"):
        np.testing.assert_array_equal(r20[key], g20[key])
        assert rel_err(r3[key], getattr(st, key)) <= 1e-9, key
