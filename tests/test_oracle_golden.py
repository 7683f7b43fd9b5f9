"""Pin the CPU oracle (oracle/) against fixtures produced by the unmodified reference.

tests/golden/make_golden.py ran conefree's own functions; the oracle restates
them with the same numpy operations, so agreement is required BIT FOR BIT.
"""

import hashlib

import numpy as np
import pytest

import oracle
from conftest import ITERATE_CASES, REPORT_FIELDS, STATE_KEYS, STATUS, init_from, load_golden, problem_from

from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, generate_witnessed


def test_example1_factors_and_operators():
    d = load_golden("example1.npz")

    class A:
        num_rows, num_cols = 3, 5
        rows, cols, vals = d["rows"], d["cols"], d["vals"]

    f = oracle.build_factors(A)
    for key, got in (("row_of", f.row_of), ("col_of", f.col_of), ("val", f.val), ("fu", f.fu), ("fv", f.fv)):
        np.testing.assert_array_equal(got, d[key], err_msg=key)
    # SPEC.md:96 values, independently of the fixture
    np.testing.assert_allclose(f.fu, [1 / 118, 1 / 26, 1 / 63], rtol=1e-15)
    np.testing.assert_allclose(f.fv, [1 / 3, 1 / 2, 1 / 3, 1 / 3, 1 / 2], rtol=1e-15)
    np.testing.assert_array_equal(oracle.apply_U(f, np.ones(8)), [19.0, 5.0, 12.0])
    np.testing.assert_array_equal(oracle.apply_Ut(f, np.ones(3)), np.arange(1.0, 9.0))
    np.testing.assert_array_equal(oracle.apply_V(f, np.arange(1.0, 9.0)), [3.0, 3.0, 9.0, 13.0, 8.0])
    np.testing.assert_array_equal(oracle.apply_Vt(f, np.array([10.0, 20, 30, 40, 50])),
                                  [10, 10, 20, 30, 30, 40, 40, 50])
    for key, got in (("U_y", oracle.apply_U(f, d["rand_y"])), ("Ut_s", oracle.apply_Ut(f, d["rand_s"])),
                     ("V_y", oracle.apply_V(f, d["rand_y"])), ("Vt_x_rand", oracle.apply_Vt(f, d["rand_x"])),
                     ("yfac_y", oracle.apply_y_factor(f, d["rand_y"]))):
        np.testing.assert_array_equal(got, d[key], err_msg=key)


def test_projection_golden():
    d = load_golden("projection.npz")
    sizes, w = d["sizes"], d["w"]
    np.testing.assert_array_equal(oracle.project_product(sizes, w), d["out_product"])
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1]))
    per_block = np.concatenate([oracle.project_block(w[s:s + q]) for s, q in zip(starts, sizes)])
    np.testing.assert_array_equal(per_block, d["out_block"])
    lp = oracle.project_product(np.ones(d["lp_w"].size, dtype=np.int64), d["lp_w"])
    np.testing.assert_array_equal(lp, d["lp_out"])
    assert np.signbit(lp).sum() == 0  # -0.0 and NaN map to +0.0 (cones.py:108-109)


def test_projection_spec_examples():
    np.testing.assert_array_equal(oracle.project_block([3.0, 0, 0, 4]), [3.5, 0, 0, 3.5])
    np.testing.assert_array_equal(oracle.project_block([5.0, 3, 0, 0]), [5.0, 3, 0, 0])
    np.testing.assert_array_equal(oracle.project_block([-5.0, 3, 0, 0]), [0.0, 0, 0, 0])
    np.testing.assert_array_equal(oracle.project_block([-2.0]), [0.0])
    np.testing.assert_array_equal(oracle.project_block([2.0]), [2.0])


@pytest.mark.parametrize("case", ITERATE_CASES)
def test_iterates_golden(case):
    d = load_golden(f"iterates_{case}.npz")
    p = problem_from(d)
    f = oracle.build_factors(p.A)
    sizes = p.cones.sizes_array()
    mu = float(d["mu"])
    init = init_from(d)
    st = oracle.OracleState.zeros(f) if init is None else oracle.OracleState(
        *(getattr(init, k).copy() for k in STATE_KEYS))
    done = 0
    for k in d["keep"]:
        st = oracle.iterate(f, sizes, st, mu, p.b, p.c, int(k) - done)
        done = int(k)
        for key in STATE_KEYS:
            np.testing.assert_array_equal(getattr(st, key), d[f"k{k}_{key}"], err_msg=f"{case} k={k} {key}")
        rep = oracle.compute_report(f, st, p.b, p.c)
        got = np.array([float(k)] + [rep[fld] for fld in REPORT_FIELDS[1:]])
        np.testing.assert_array_equal(got[1:], d[f"k{k}_report"][1:], err_msg=f"{case} k={k} report")


def test_dense_mirror_agrees():
    d = load_golden("iterates_socp4_mu5.npz")
    p = problem_from(d)
    f = oracle.build_factors(p.A)
    sizes = p.cones.sizes_array()
    a = oracle.OracleState.zeros(f)
    b = oracle.OracleState.zeros(f)
    for _ in range(50):
        a = oracle.step(f, sizes, a, 5.0, p.b, p.c)
        b = oracle.dense_iterate(f, sizes, b, 5.0, p.b, p.c)
    for key in STATE_KEYS:
        want = getattr(a, key)
        assert np.max(np.abs(getattr(b, key) - want)) / (1 + np.max(np.abs(want))) < 1e-10


def _cfg_from(vec):
    mu, mi, ce, tm, ea, er, ep, ed, eg = vec
    return SolverConfig(mu=float(mu), max_iters=int(mi), check_every=int(ce), term_mode=("osqp", "scs", "target")[int(tm)],
                        eps_abs=float(ea), eps_rel=float(er), eps_prim=float(ep), eps_dual=float(ed), eps_gap=float(eg))


ANALYTIC_CFG = {
    "scs1e-3": SolverConfig(),
    "scs1e-9": SolverConfig(eps_prim=1e-9, eps_dual=1e-9, eps_gap=1e-9),
    "osqp": SolverConfig(term_mode="osqp", eps_abs=1e-6, eps_rel=1e-6),
    "target": SolverConfig(term_mode="target", target_prim_res=1e-7, target_gap=1e-7),
    "max7": SolverConfig(max_iters=7, check_every=3),
}


def analytic_problems():
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, TripletMatrix

    return {
        "lp1x1": ProblemInstance(TripletMatrix(1, 1, [0], [0], [1.0]), [1.0], [1.0], ConeSpec.orthant(1)),
        "lp2var": ProblemInstance(TripletMatrix(1, 2, [0, 0], [0, 1], [1.0, 1.0]), [1.0], [1.0, 2.0],
                                  ConeSpec.orthant(2)),
        "socp4": ProblemInstance(TripletMatrix(1, 4, [0], [0], [1.0]), [2.0], [0.0, 0.0, 0.0, -1.0], ConeSpec((4,))),
    }


def _trace_array(trace):
    return np.array([[float(r[f]) for f in REPORT_FIELDS] for r in trace])


def test_solves_golden():
    d = load_golden("solves.npz")
    probs = analytic_problems()
    for name in d["names"]:
        name = str(name)
        if "__" in name:
            pname, cname = name.split("__")
            p, cfg = probs[pname], ANALYTIC_CFG[cname]
        else:
            p, cfg = problem_from(d, name + "__"), _cfg_from(d[name + "__cfg"])
        x, lam, trace, _ = oracle.solve(p, cfg)
        np.testing.assert_array_equal(_trace_array(trace), d[name + "__trace"], err_msg=name)
        assert [STATUS.index(r["status"]) for r in trace] == list(d[name + "__status"]), name
        np.testing.assert_array_equal(x, d[name + "__x"])
        np.testing.assert_array_equal(lam, d[name + "__lam"])


def test_generator_golden():
    d = load_golden("generator_c1.npz")
    for name in ("g_lp", "g_socp", "g_raw", "g_dense"):
        m, n, dens, kind, seed, bounded = d[name + "__spec"]
        spec = GenSpec(int(m), int(n), float(dens), ("lp", "socp4")[int(kind)], seed=int(seed),
                       bounded_mode=bool(bounded))
        g = generate_witnessed(spec)
        want = problem_from(d, name + "__")
        for attr in ("rows", "cols", "vals"):
            np.testing.assert_array_equal(getattr(g.problem.A, attr), getattr(want.A, attr), err_msg=name + attr)
        np.testing.assert_array_equal(g.problem.b, want.b, err_msg=name)
        np.testing.assert_array_equal(g.problem.c, want.c, err_msg=name)
        np.testing.assert_array_equal(g.x_feas, d[name + "__x_feas"])
        assert g.problem.cones == want.cones
    c1 = generate(GenSpec(1000, 2000, 0.01, "lp", seed=0))
    h = hashlib.sha256()
    for a in (c1.A.rows, c1.A.cols, c1.A.vals, c1.b, c1.c):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(d["c1_sha"])


def test_c1_golden_solve():
    """C1 (BASELINE configs[0]): 11,375 iterations to scs 1e-4, bit-identical trace."""
    d = load_golden("generator_c1.npz")
    p = generate(GenSpec(1000, 2000, 0.01, "lp", seed=0))
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    x, lam, trace, _ = oracle.solve(p, cfg)
    assert trace[-1]["iter"] == 11375 and trace[-1]["status"] == "solved"
    np.testing.assert_array_equal(_trace_array(trace), d["c1__trace"])
    np.testing.assert_array_equal(x, d["c1__x"])
    np.testing.assert_array_equal(lam, d["c1__lam"])
