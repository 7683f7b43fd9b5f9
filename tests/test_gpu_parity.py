"""GPU parity: the CUDA path (libcfb200 through the C ABI) against the oracle / reference fixtures.

Tolerances (north_star: iterates <= 1e-9 relative over the first 100 iterations):
  * iterates x, y, z, lam, gamma, delta:  rel_err <= 1e-9 at iterations 1..100
  * report fields:                         |got - want| / (1 + |want|) <= 1e-9
  * operators A x and A^T y:               bit-identical (sequential canonical-order sums)
  * cone projection of blocks <= 512:      bit-identical
  * whole solves: same status, same iteration count (the reduced iteration agrees
    to ~1e-13, so a check can only flip within ~1e-13 of a bound), x/lam rel_err <= 1e-8
"""

import numpy as np
import pytest

import oracle
from conftest import ITERATE_CASES, REPORT_FIELDS, STATE_KEYS, STATUS, init_from, load_golden, problem_from, rel_err

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-9
REPORT_TOL = 1e-9


def _scalar_rel(a, b):
    return abs(a - b) / (1.0 + abs(b))


def _plan(p):
    from paper_2203_05027_b200.api import build_plan

    return build_plan(p)


@pytest.mark.parametrize("case", ITERATE_CASES)
def test_iterates_match_reference(case):
    d = load_golden(f"iterates_{case}.npz")
    p = problem_from(d)
    mu = float(d["mu"])
    with _plan(p) as plan:
        plan.set_state(mu, init_from(d))
        done = 0
        for k in d["keep"]:
            plan.iterate(mu, int(k) - done)
            done = int(k)
            st = plan.get_state()
            assert st["iter"] == k
            for key in STATE_KEYS:
                err = rel_err(st[key], d[f"k{k}_{key}"])
                assert err <= ITER_TOL, f"{case} k={k} {key}: rel_err {err:.3e}"
            rep = plan.report(mu)
            want = d[f"k{k}_report"]
            for i, fld in enumerate(REPORT_FIELDS[1:], start=1):
                e = _scalar_rel(rep[fld], want[i])
                assert e <= REPORT_TOL, f"{case} k={k} {fld}: {rep[fld]!r} vs {want[i]!r}"


def _device_vec(v):
    import torch

    return torch.tensor(np.asarray(v, dtype=np.float64), device="cuda")


@pytest.mark.parametrize("case", ITERATE_CASES)
def test_operators_bit_identical(case):
    d = load_golden(f"iterates_{case}.npz")
    p = problem_from(d)
    f = oracle.build_factors(p.A)
    rng = np.random.default_rng(7)
    x = rng.standard_normal(f.n)
    y = rng.standard_normal(f.m)
    with _plan(p) as plan:
        import torch

        dx, dy = _device_vec(x), _device_vec(y)
        ax = torch.empty(f.m, dtype=torch.float64, device="cuda")
        aty = torch.empty(f.n, dtype=torch.float64, device="cuda")
        plan.apply_A(dx.data_ptr(), ax.data_ptr())
        plan.apply_At(dy.data_ptr(), aty.data_ptr())
        np.testing.assert_array_equal(ax.cpu().numpy(), oracle.apply_U(f, oracle.apply_Vt(f, x)))
        np.testing.assert_array_equal(aty.cpu().numpy(), oracle.apply_V(f, oracle.apply_Ut(f, y)))


def test_projection_bit_identical():
    import torch

    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix

    d = load_golden("projection.npz")
    sizes, w = d["sizes"], d["w"]
    n = int(sizes.sum())
    p = ProblemInstance(TripletMatrix(1, n, [0], [0], [1.0]), [1.0], np.zeros(n), ConeSpec(sizes))
    with _plan(p) as plan:
        dw = _device_vec(w)
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        plan.project(dw.data_ptr(), out.data_ptr())
        np.testing.assert_array_equal(out.cpu().numpy(), d["out_product"])
    lp_w = d["lp_w"]
    q = ProblemInstance(TripletMatrix(1, lp_w.size, [0], [0], [1.0]), [1.0], np.zeros(lp_w.size),
                        ConeSpec.orthant(lp_w.size))
    with _plan(q) as plan:
        dw = _device_vec(lp_w)
        out = torch.empty(lp_w.size, dtype=torch.float64, device="cuda")
        plan.project(dw.data_ptr(), out.data_ptr())
        got = out.cpu().numpy()
        np.testing.assert_array_equal(got, d["lp_out"])
        assert np.signbit(got).sum() == 0


def test_big_cone_projection():
    import torch

    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix

    rng = np.random.default_rng(3)
    sizes = np.array([3, 2000, 1, 700, 5, 513, 512, 4], dtype=np.int64)
    n = int(sizes.sum())
    w = rng.standard_normal(n)
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    w[starts[1]] = 60.0   # scale branch for the big cone
    w[starts[3]] = -40.0  # polar branch
    p = ProblemInstance(TripletMatrix(1, n, [0], [0], [1.0]), [1.0], np.zeros(n), ConeSpec(sizes))
    want = oracle.project_product(sizes, w)
    with _plan(p) as plan:
        assert plan.info()["big_cones"] == 4  # cones wider than kSmallCone=256
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        plan.project(_device_vec(w).data_ptr(), out.data_ptr())
        assert rel_err(out.cpu().numpy(), want) <= 1e-13


def _cfg_from(vec):
    from paper_2203_05027_b200 import SolverConfig

    mu, mi, ce, tm, ea, er, ep, ed, eg = vec
    return SolverConfig(mu=float(mu), max_iters=int(mi), check_every=int(ce),
                        term_mode=("osqp", "scs", "target")[int(tm)], eps_abs=float(ea), eps_rel=float(er),
                        eps_prim=float(ep), eps_dual=float(ed), eps_gap=float(eg))


def test_solves_match_reference():
    from test_oracle_golden import ANALYTIC_CFG, analytic_problems

    from paper_2203_05027_b200 import solve

    d = load_golden("solves.npz")
    probs = analytic_problems()
    for name in d["names"]:
        name = str(name)
        if "__" in name:
            pname, cname = name.split("__")
            p, cfg = probs[pname], ANALYTIC_CFG[cname]
        else:
            p, cfg = problem_from(d, name + "__"), _cfg_from(d[name + "__cfg"])
        res = solve(p, cfg)
        want = d[name + "__trace"]
        st = d[name + "__status"]
        assert len(res.trace) == len(want), name
        assert [STATUS.index(r.status) for r in res.trace] == list(st), name
        for r, w in zip(res.trace, want):
            assert r.iter == int(w[0])
            for i, fld in enumerate(REPORT_FIELDS[1:], start=1):
                assert _scalar_rel(getattr(r, fld), w[i]) <= 1e-8, (name, r.iter, fld)
        assert rel_err(res.x, d[name + "__x"]) <= 1e-8, name
        assert rel_err(res.lam, d[name + "__lam"]) <= 1e-8, name
        assert res.report == res.trace[-1]


def test_c1_time_to_tolerance_parity():
    """BASELINE configs[0]: the reference solves C1 in 11,375 iterations (pobj 220.7838450224)."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve

    d = load_golden("generator_c1.npz")
    p = generate(GenSpec(1000, 2000, 0.01, "lp", seed=0))
    res = solve(p, SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4))
    assert res.report.status == "solved"
    assert res.report.iter == int(d["c1__trace"][-1][0]) == 11375
    assert _scalar_rel(res.report.pobj, d["c1__trace"][-1][10]) <= 1e-9
    assert rel_err(res.x, d["c1__x"]) <= 1e-8
    assert rel_err(res.lam, d["c1__lam"]) <= 1e-8


def test_determinism_bitwise():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve

    p = generate(GenSpec(200, 600, 0.03, "socp4", seed=5))
    cfg = SolverConfig(max_iters=400, check_every=20)
    a, b = solve(p, cfg), solve(p, cfg)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.lam, b.lam)
    assert a.trace == b.trace


def _oracle_run(p, mu, iters, init=None):
    f = oracle.build_factors(p.A)
    sizes = p.cones.sizes_array()
    st = oracle.OracleState.zeros(f) if init is None else init
    return oracle.iterate(f, sizes, st, mu, p.b, p.c, iters)


def _check_against_oracle(p, mu=1.0, iters=30, tol=ITER_TOL):
    want = _oracle_run(p, mu, iters)
    with _plan(p) as plan:
        plan.set_state(mu, None)
        plan.iterate(mu, iters)
        st = plan.get_state()
    for key in STATE_KEYS:
        err = rel_err(st[key], getattr(want, key))
        assert err <= tol, f"{key}: {err:.3e}"


def test_long_rows_and_columns_chunking():
    """Rows/columns longer than the smem chunk (kCap=4096) and empty rows/columns."""
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix

    rng = np.random.default_rng(11)
    m, n = 40, 9000
    rows, cols = [], []
    rows += [0] * n; cols += list(range(n))                        # one dense row of 9000
    dense_col = 17
    rows += list(range(1, 30)); cols += [dense_col] * 29
    extra = rng.choice(np.arange(1, 30 * n), size=3000, replace=False)
    rows += list(1 + (extra // n) % 29); cols += list(extra % n)
    key = np.unique(np.array(rows) * n + np.array(cols))
    r, c = key // n, key % n
    vals = rng.standard_normal(r.size)
    b = rng.standard_normal(m)
    b[30:] = 0.0                                                    # rows 30..39 are empty
    p = ProblemInstance(TripletMatrix(m, n, r, c, vals), b, rng.standard_normal(n), ConeSpec.orthant(n))
    _check_against_oracle(p, mu=0.9, iters=25)


def test_mixed_and_big_cones_iterate():
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix

    rng = np.random.default_rng(12)
    sizes = np.array([1, 2, 600, 3, 1, 1, 1200, 4, 8, 1, 530], dtype=np.int64)
    n, m = int(sizes.sum()), 120
    dense = rng.standard_normal((m, n)) * (rng.random((m, n)) < 0.02)
    a = TripletMatrix.from_dense(dense)
    x0 = oracle.project_product(sizes, rng.standard_normal(n))
    p = ProblemInstance(a, dense @ x0, rng.standard_normal(n), ConeSpec(sizes))
    _check_against_oracle(p, mu=1.7, iters=40, tol=1e-9)


def test_warm_start_solve_matches_oracle():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, SolverState, generate, solve

    p = generate(GenSpec(50, 120, 0.05, "socp4", seed=9))
    f = oracle.build_factors(p.A)
    rng = np.random.default_rng(4)
    init = SolverState(x=rng.standard_normal(f.n), y=rng.standard_normal(f.o), z=rng.standard_normal(f.n),
                       lam=rng.standard_normal(f.m), gamma=rng.standard_normal(f.o), delta=rng.standard_normal(f.n))
    cfg = SolverConfig(mu=0.8, max_iters=3000, eps_prim=1e-5, eps_dual=1e-5, eps_gap=1e-5)
    ost = oracle.OracleState(*(getattr(init, k).copy() for k in STATE_KEYS))
    ox, olam, otrace, _ = oracle.solve(p, cfg, init=ost)
    res = solve(p, cfg, init=init)
    assert res.report.status == otrace[-1]["status"]
    assert res.report.iter == otrace[-1]["iter"]
    assert rel_err(res.x, ox) <= 1e-8 and rel_err(res.lam, olam) <= 1e-8


def test_divergence_status():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, SolverState, generate, solve

    p = generate(GenSpec(20, 50, 0.1, seed=2))
    f = oracle.build_factors(p.A)
    init = SolverState(x=np.zeros(f.n), y=np.zeros(f.o), z=np.zeros(f.n), lam=np.zeros(f.m),
                       gamma=np.zeros(f.o), delta=np.zeros(f.n))
    init.z[3] = np.inf  # x_update reads z (solver.py:173), never the old x
    cfg = SolverConfig(max_iters=100, check_every=10)
    res = solve(p, cfg, init=init)
    ost = oracle.OracleState(*(getattr(init, k).copy() for k in STATE_KEYS))
    _, _, otrace, _ = oracle.solve(p, cfg, init=ost)
    assert otrace[-1]["status"] == "diverged"
    assert res.report.status == "diverged" and res.report.iter == otrace[-1]["iter"]


def test_invalid_problems_raise_reference_messages():
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix, solve, validate

    good = dict(rows=[0, 1, 1], cols=[0, 1, 2], vals=[1.0, 2.0, 3.0])
    cases = [
        dict(rows=[0, 1, 0], cols=[0, 1, 0], vals=[1.0, 2.0, 3.0]),     # duplicate
        dict(rows=[0, 1, 1], cols=[0, 1, 2], vals=[1.0, 0.0, 3.0]),     # zero
        dict(rows=[0, 1, 1], cols=[0, 1, 2], vals=[1.0, np.nan, 3.0]),  # non-finite
        dict(rows=[0, 5, 1], cols=[0, 1, 2], vals=[1.0, 2.0, 3.0]),     # row out of range
        dict(rows=[0, 1, 1], cols=[0, 1, 7], vals=[1.0, 2.0, 3.0]),     # col out of range
    ]
    for kw in cases:
        p = ProblemInstance(TripletMatrix(2, 3, **kw), [1.0, 1.0], [1.0, 1.0, 1.0], ConeSpec.orthant(3))
        want = "invalid problem: " + "; ".join(validate(p).violations[:3])
        with pytest.raises(ValueError) as ei:
            solve(p)
        assert str(ei.value) == want
    p = ProblemInstance(TripletMatrix(2, 3, **good), [1.0, np.inf], [1.0, 1.0, 1.0], ConeSpec.orthant(3))
    with pytest.raises(ValueError, match=r"b\[1\] = inf is not finite"):
        solve(p)


def test_reference_types_accepted():
    """Duck typing: plain objects shaped like the reference's ProblemInstance work."""
    from types import SimpleNamespace

    from paper_2203_05027_b200 import SolverConfig, solve

    a = SimpleNamespace(num_rows=1, num_cols=2, rows=np.array([0, 0]), cols=np.array([0, 1]),
                        vals=np.array([1.0, 1.0]), nnz=2)
    p = SimpleNamespace(A=a, b=np.array([1.0]), c=np.array([1.0, 2.0]), cones=SimpleNamespace(block_sizes=(1, 1)))
    res = solve(p, SolverConfig(eps_prim=1e-9, eps_dual=1e-9, eps_gap=1e-9))
    assert res.report.status == "solved"
    np.testing.assert_allclose(res.x, [1.0, 0.0], atol=1e-6)
    np.testing.assert_allclose(res.lam, [-1.0], atol=1e-6)


def test_row_panels_bit_identical(monkeypatch):
    """Column panels of the row pass (CF_PANEL_MB) keep A x bit-identical and the iterates unchanged."""
    import torch

    monkeypatch.setenv("CF_PANEL_MB", "0.002")  # 2 KB of x per panel -> several panels
    d = load_golden("iterates_lp_mu1.npz")
    p = problem_from(d)
    f = oracle.build_factors(p.A)
    x = np.random.default_rng(5).standard_normal(f.n)
    with _plan(p) as plan:
        ax = torch.empty(f.m, dtype=torch.float64, device="cuda")
        plan.apply_A(_device_vec(x).data_ptr(), ax.data_ptr())
        np.testing.assert_array_equal(ax.cpu().numpy(), oracle.apply_U(f, oracle.apply_Vt(f, x)))
        plan.set_state(1.0, None)
        plan.iterate(1.0, 100)
        st = plan.get_state()
    for key in STATE_KEYS:
        assert rel_err(st[key], d[f"k100_{key}"]) <= ITER_TOL, key
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve

    q = generate(GenSpec(300, 900, 0.02, "lp", seed=8))
    cfg = SolverConfig(max_iters=600)
    res = solve(q, cfg)
    monkeypatch.setenv("CF_PANEL_MB", "1000")
    ref = solve(q, cfg)
    np.testing.assert_array_equal(res.x, ref.x)
    assert res.trace == ref.trace


def test_solve_batch_matches_solve():
    """Batched solver (C4): every problem's result equals solve(p) (same iterates, statuses, counts)."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve, solve_batch

    specs = [GenSpec(30, 60, 0.05, "lp", seed=s) for s in range(6)] + \
            [GenSpec(20, 48, 0.08, "socp4", seed=s) for s in range(3)] + [GenSpec(5, 9, 0.4, "lp", seed=99)]
    probs = [generate(s) for s in specs]
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=5000)
    batch = solve_batch(probs, cfg)
    for p, rb in zip(probs, batch):
        rs = solve(p, cfg)
        assert rb.report.status == rs.report.status and rb.report.iter == rs.report.iter
        np.testing.assert_array_equal(rb.x, rs.x)       # same sequential arithmetic as the plan passes
        np.testing.assert_array_equal(rb.lam, rs.lam)
        assert len(rb.trace) == len(rs.trace)
        for a, b in zip(rb.trace, rs.trace):
            assert a.status == b.status and a.iter == b.iter
            for fld in REPORT_FIELDS[1:]:
                assert _scalar_rel(getattr(a, fld), getattr(b, fld)) <= 1e-12
    # against the oracle too (C4 shape: 100 x 200, 5 %)
    q = generate(GenSpec(100, 200, 0.05, "lp", seed=3))
    cfg2 = SolverConfig(max_iters=3000)
    rb = solve_batch([q], cfg2)[0]
    ox, olam, otrace, _ = oracle.solve(q, cfg2)
    assert rb.report.status == otrace[-1]["status"] and rb.report.iter == otrace[-1]["iter"]
    assert rel_err(rb.x, ox) <= 1e-8 and rel_err(rb.lam, olam) <= 1e-8


def test_warp_cone_epilogue_equals_group_epilogue(monkeypatch):
    """Uniform K4 cones take the warp-shuffle epilogue; it is bit-identical to the
    shared-memory group epilogue (forced with CF_GROUP_CONES) and to the oracle's projection."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve

    p = generate(GenSpec(300, 1200, 0.02, "socp4", seed=4))
    cfg = SolverConfig(max_iters=300, check_every=25, eps_prim=1e-6, eps_dual=1e-6, eps_gap=1e-6)
    warp = solve(p, cfg)
    monkeypatch.setenv("CF_GROUP_CONES", "1")
    group = solve(p, cfg)
    assert np.array_equal(warp.x, group.x) and np.array_equal(warp.lam, group.lam)
    assert [r.iter for r in warp.trace] == [r.iter for r in group.trace]


@pytest.mark.parametrize("case", ITERATE_CASES)
def test_column_bands_match_reference(case, monkeypatch):
    """Row bands of the column pass (CF_BAND_MB: h split into L2-sized slices, partial
    column sums carried between bands) keep A^T y bit-identical and the iterates and
    reports within the parity tolerance, for every cone layout and warm starts."""
    import torch

    monkeypatch.setenv("CF_BAND_MB", "0.0005")   # 512 bytes of h per band -> several bands
    d = load_golden(f"iterates_{case}.npz")
    p = problem_from(d)
    f = oracle.build_factors(p.A)
    y = np.random.default_rng(9).standard_normal(f.m)
    mu = float(d["mu"])
    with _plan(p) as plan:
        aty = torch.empty(f.n, dtype=torch.float64, device="cuda")
        plan.apply_At(_device_vec(y).data_ptr(), aty.data_ptr())
        np.testing.assert_array_equal(aty.cpu().numpy(), oracle.apply_V(f, oracle.apply_Ut(f, y)))
        plan.set_state(mu, init_from(d))
        done = 0
        for k in d["keep"]:
            plan.iterate(mu, int(k) - done)
            done = int(k)
            st = plan.get_state()
            for key in STATE_KEYS:
                assert rel_err(st[key], d[f"k{k}_{key}"]) <= ITER_TOL, (case, int(k), key)
            rep = plan.report(mu)
            want = d[f"k{k}_report"]
            for i, fld in enumerate(REPORT_FIELDS[1:], start=1):
                assert _scalar_rel(rep[fld], want[i]) <= REPORT_TOL, (case, int(k), fld)


def test_column_bands_solve_bit_identical(monkeypatch):
    """A banded solve returns exactly what the unbanded one does (same sums, same order)."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve

    for kind in ("lp", "socp4"):
        q = generate(GenSpec(400, 800, 0.02, kind, seed=12))
        cfg = SolverConfig(max_iters=500)
        monkeypatch.setenv("CF_BAND_MB", "0.001")
        banded = solve(q, cfg)
        monkeypatch.setenv("CF_BAND_MB", "1000")
        ref = solve(q, cfg)
        np.testing.assert_array_equal(banded.x, ref.x)
        np.testing.assert_array_equal(banded.lam, ref.lam)
        assert banded.trace == ref.trace


@pytest.mark.parametrize("case", ITERATE_CASES)
def test_large_tiles_match_reference(case, monkeypatch):
    """Tiles cut with the large nonzero budget (kTileNnzLarge, used by passes too big for
    the staged dispatch; forced here on the golden cases) keep A x and A^T y bit-identical
    and the iterates within the parity tolerance, for every cone layout."""
    import torch

    monkeypatch.setenv("CF_FORCE_LARGE_TILES", "1")
    d = load_golden(f"iterates_{case}.npz")
    p = problem_from(d)
    f = oracle.build_factors(p.A)
    rng = np.random.default_rng(21)
    x, y = rng.standard_normal(f.n), rng.standard_normal(f.m)
    mu = float(d["mu"])
    with _plan(p) as plan:
        ax = torch.empty(f.m, dtype=torch.float64, device="cuda")
        aty = torch.empty(f.n, dtype=torch.float64, device="cuda")
        plan.apply_A(_device_vec(x).data_ptr(), ax.data_ptr())
        plan.apply_At(_device_vec(y).data_ptr(), aty.data_ptr())
        np.testing.assert_array_equal(ax.cpu().numpy(), oracle.apply_U(f, oracle.apply_Vt(f, x)))
        np.testing.assert_array_equal(aty.cpu().numpy(), oracle.apply_V(f, oracle.apply_Ut(f, y)))
        plan.set_state(mu, init_from(d))
        done = 0
        for k in d["keep"]:
            plan.iterate(mu, int(k) - done)
            done = int(k)
            st = plan.get_state()
            for key in STATE_KEYS:
                assert rel_err(st[key], d[f"k{k}_{key}"]) <= ITER_TOL, (case, int(k), key)


def test_large_tiles_solve_bit_identical(monkeypatch):
    """A solve on large tiles returns exactly the default tiling's iterates. Report norms
    sum per-CTA partials, whose grouping follows the tiling, so they agree to rounding."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve

    for kind in ("lp", "socp4"):
        q = generate(GenSpec(300, 900, 0.05, kind, seed=14))   # ~45 nonzeros per row
        cfg = SolverConfig(max_iters=500)
        monkeypatch.setenv("CF_FORCE_LARGE_TILES", "1")
        large = solve(q, cfg)
        monkeypatch.delenv("CF_FORCE_LARGE_TILES")
        ref = solve(q, cfg)
        np.testing.assert_array_equal(large.x, ref.x)
        np.testing.assert_array_equal(large.lam, ref.lam)
        assert len(large.trace) == len(ref.trace)
        for a, b in zip(large.trace, ref.trace):
            assert a.status == b.status and a.iter == b.iter
            for fld in REPORT_FIELDS[1:]:
                assert _scalar_rel(getattr(a, fld), getattr(b, fld)) <= 1e-12


@pytest.mark.parametrize("shape", ["no_nonzeros", "1x1", "one_dense_row", "one_dense_column", "empty_rows_cols"])
def test_degenerate_shapes_match_oracle(shape):
    """Shapes at the edges of the tiling: no nonzeros, 1x1, one dense row / column (long
    tiles), and many empty rows and columns; solve() equals the oracle's loop."""
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, SolverConfig, TripletMatrix, solve

    rng = np.random.default_rng(13)
    if shape == "no_nonzeros":
        m, n, rows, cols = 3, 5, [], []
    elif shape == "1x1":
        m, n, rows, cols = 1, 1, [0], [0]
    elif shape == "one_dense_row":
        m, n = 4, 5000
        rows, cols = [0] * n, list(range(n))
    elif shape == "one_dense_column":
        m, n = 5000, 3
        rows, cols = list(range(m)), [1] * m
    else:
        m, n = 400, 900
        rows = list(rng.choice(np.arange(0, m, 3), 600))
        cols = list(rng.choice(np.arange(0, n, 4), 600))
        key = sorted(set(zip(rows, cols)))
        rows, cols = [r for r, _ in key], [c for _, c in key]
    vals = rng.standard_normal(len(rows)) + 0.1
    a = TripletMatrix(m, n, np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64), vals)
    p = ProblemInstance(a, rng.standard_normal(m), np.abs(rng.standard_normal(n)), ConeSpec((1,) * n))
    cfg = SolverConfig(max_iters=400, check_every=25)
    res = solve(p, cfg)
    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert res.report.iter == otrace[-1]["iter"] and res.report.status == otrace[-1]["status"]
    assert rel_err(res.x, ox) <= 1e-9 and rel_err(res.lam, olam) <= 1e-9


def test_solve_batch_mixes_kernel_and_concurrent_solves():
    """Problems too large for one CTA are solved alongside the batched kernel (threads with
    their own plans); every result equals solve() on that problem, in input order."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve, solve_batch

    probs = [generate(GenSpec(60, 120, 0.05, "lp", seed=1)), generate(GenSpec(900, 2000, 0.01, "lp", seed=2)),
             generate(GenSpec(60, 120, 0.05, "socp4", seed=3)), generate(GenSpec(1000, 3000, 0.01, "socp4", seed=4))]
    cfg = SolverConfig(max_iters=3000)
    got = solve_batch(probs, cfg)
    for p, r in zip(probs, got):
        ref = solve(p, cfg)
        np.testing.assert_array_equal(r.x, ref.x)
        np.testing.assert_array_equal(r.lam, ref.lam)
        assert r.trace == ref.trace
