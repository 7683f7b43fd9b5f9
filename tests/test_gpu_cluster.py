"""Cluster-resident solver (csrc/cf_batch.cu k_cluster, cf_cluster_solve): solve() of a
mid-size problem in one thread-block-cluster launch must return what the plan path
(cf_plan_solve, CF_NO_CLUSTER=1) returns — the same x and lam bit for bit, the same
statuses and iteration counts — and reach the oracle's iterates."""

import math

import numpy as np
import pytest

import oracle
from conftest import REPORT_FIELDS, rel_err

pytestmark = pytest.mark.gpu


def _rel(a, b):
    if a == b or (math.isnan(a) and math.isnan(b)):
        return 0.0
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def _both(p, cfg, monkeypatch):
    from paper_2203_05027_b200 import api, solve

    api._LAST_CLUSTER = 0
    got = solve(p, cfg)
    used = api._LAST_CLUSTER
    monkeypatch.setenv("CF_NO_CLUSTER", "1")
    ref = solve(p, cfg)
    monkeypatch.delenv("CF_NO_CLUSTER")
    return got, ref, used


def _same(got, ref):
    np.testing.assert_array_equal(got.x, ref.x)
    np.testing.assert_array_equal(got.lam, ref.lam)
    assert len(got.trace) == len(ref.trace)
    for a, b in zip(got.trace, ref.trace):
        assert a.status == b.status and a.iter == b.iter
        for f in REPORT_FIELDS[1:]:
            if f == "gap":   # pobj + b.lam cancels: compare against the terms' scale
                assert abs(a.gap - b.gap) <= 1e-12 * (1.0 + abs(b.pobj) + abs(b.dobj))
            else:
                assert _rel(getattr(a, f), getattr(b, f)) <= 1e-12, f


@pytest.mark.parametrize("spec,cfg_kw,cluster", [
    (("lp", 1000, 2000, 0.01, 0), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4), None),   # C1
    (("lp", 300, 500, 0.02, 5), dict(mu=0.3, max_iters=4000, check_every=10), None),
    (("socp4", 400, 800, 0.01, 7), dict(mu=0.7, max_iters=3000), None),
    (("lp", 1500, 6000, 0.0017, 9), dict(max_iters=2000, check_every=25), None),
    (("lp", 5, 9, 0.4, 99), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=5000), None),
])
def test_cluster_equals_plan(spec, cfg_kw, cluster, monkeypatch):
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate

    kind, m, n, d, seed = spec
    p = generate(GenSpec(m, n, d, kind, seed=seed))
    got, ref, used = _both(p, SolverConfig(**cfg_kw), monkeypatch)
    assert used >= 1 and (cluster is None or used == cluster)
    _same(got, ref)


def test_cluster_c1_golden(monkeypatch):
    """C1 through the default solve(): the reference's own run needs 11,375 iterations."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, api, generate, solve

    p = generate(GenSpec(1000, 2000, 0.01, "lp", seed=0))
    api._LAST_CLUSTER = 0
    res = solve(p, SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4))
    assert api._LAST_CLUSTER > 0
    assert res.report.status == "solved" and res.report.iter == 11375
    assert abs(res.report.pobj - 220.7838450224) < 1e-8


def test_cluster_mixed_cones_vs_oracle(monkeypatch):
    """Cones of mixed sizes (cone-aligned column cuts) against the oracle and the plan path."""
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, SolverConfig, TripletMatrix

    rng = np.random.default_rng(11)
    sizes = [1, 3, 1, 1, 5, 2, 4, 1, 7, 1, 3, 3, 1, 6] * 40
    n = sum(sizes)
    m = 700
    o = 6000
    lin = rng.choice(m * n, o, replace=False)
    a = TripletMatrix(m, n, lin // n, lin % n, rng.standard_normal(o))
    p = ProblemInstance(a, rng.standard_normal(m), rng.standard_normal(n), ConeSpec(tuple(sizes)))
    cfg = SolverConfig(mu=0.9, max_iters=600, check_every=20)
    got, ref, used = _both(p, cfg, monkeypatch)
    assert used >= 1
    _same(got, ref)
    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert [r.iter for r in got.trace] == [r["iter"] for r in otrace]
    assert rel_err(got.x, ox) <= 1e-9 and rel_err(got.lam, olam) <= 1e-9


def test_cluster_declines_large_and_degenerate(monkeypatch):
    """Too large for a cluster: cf_cluster_solve reports 0 and solve() runs the plan; problems
    without nonzeros or with empty rows/columns still match the plan path."""
    from paper_2203_05027_b200 import ConeSpec, GenSpec, ProblemInstance, SolverConfig, TripletMatrix, api, generate

    big = generate(GenSpec(6000, 12000, 0.002, "lp", seed=1))
    cfg = SolverConfig(max_iters=50)
    got, ref, used = _both(big, cfg, monkeypatch)
    assert used == 0
    _same(got, ref)
    empty = ProblemInstance(TripletMatrix(3, 4, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)),
                            np.array([1.0, -2.0, 0.5]), np.array([1.0, 0.0, -1.0, 2.0]), ConeSpec((1, 1, 1, 1)))
    got, ref, used = _both(empty, SolverConfig(max_iters=200), monkeypatch)
    assert used == 1
    _same(got, ref)
    a = TripletMatrix(6, 5, np.array([0, 0, 3, 5]), np.array([1, 4, 1, 0]), np.array([2.0, -1.0, 0.5, 3.0]))
    q = ProblemInstance(a, np.arange(6.0), np.ones(5), ConeSpec((1, 1, 1, 1, 1)))
    got, ref, used = _both(q, SolverConfig(max_iters=300, check_every=7), monkeypatch)
    _same(got, ref)


@pytest.mark.parametrize("size", [1, 2, 4, 8, 16])
def test_every_cluster_size_equals_plan(size, monkeypatch):
    """CF_CLUSTER_SIZE forces the cluster size: every size gives the plan's iterates."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate

    p = generate(GenSpec(300, 640, 0.02, "socp4" if size % 2 else "lp", seed=20 + size))
    monkeypatch.setenv("CF_CLUSTER_SIZE", str(size))
    got, ref, used = _both(p, SolverConfig(mu=0.8, max_iters=1500, check_every=15), monkeypatch)
    assert used == size
    _same(got, ref)
