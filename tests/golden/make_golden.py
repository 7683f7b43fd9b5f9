"""Generate the golden parity fixtures by running the UNMODIFIED reference.

Run ONLY in the build container, where the reference is mounted read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Nothing at test time imports the reference (it does not exist on the GPU box);
the tests read the ``.npz`` files this script writes next to it. Every array
here is produced by calling the reference's own public functions
(``conefree.build_uv``, ``apply_*``, ``project_block``, ``x_update`` …
``dual_update``, ``compute_report``, ``solve``, ``generate``), so the fixtures
pin both the oracle restatement in ``oracle/`` and the CUDA path.
"""

from __future__ import annotations

import hashlib
import os
import sys
from dataclasses import asdict

import numpy as np

REF_SRC = "/root/reference/pkg/src"
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

import conefree as cf  # noqa: E402  (the reference package)
from conefree import solver as ref_solver  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

REPORT_FIELDS = (
    "iter", "prim_res_inf", "prim_res_2", "dual_res_inf", "dual_res_2",
    "stat_res_inf", "stat_res_2", "ax_inf", "atl_inf", "cone_gap",
    "pobj", "dobj", "gap",
)
STATUS = ("running", "solved", "max_iters", "diverged")


def _problem_arrays(p, prefix=""):
    return {
        prefix + "m": np.int64(p.A.num_rows),
        prefix + "n": np.int64(p.A.num_cols),
        prefix + "rows": p.A.rows.copy(),
        prefix + "cols": p.A.cols.copy(),
        prefix + "vals": p.A.vals.copy(),
        prefix + "b": p.b.copy(),
        prefix + "c": p.c.copy(),
        prefix + "block_sizes": np.asarray(p.cones.block_sizes, dtype=np.int64),
    }


def _trace_arrays(trace, prefix=""):
    tab = np.array([[float(getattr(r, f)) for f in REPORT_FIELDS] for r in trace])
    st = np.array([STATUS.index(r.status) for r in trace], dtype=np.int64)
    return {prefix + "trace": tab, prefix + "status": st}


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# --------------------------------------------------------------------------
# 1. Example 1 (PAPER Example 1 / conftest.py:8-14) and the operator examples
# --------------------------------------------------------------------------
def example1():
    dense = np.array(
        [[1.0, 0.0, 4.0, 6.0, 8.0],
         [0.0, 0.0, 5.0, 0.0, 0.0],
         [2.0, 3.0, 0.0, 7.0, 0.0]]
    )
    a = cf.TripletMatrix.from_dense(dense)
    # shuffle the triplets so canonicalisation is exercised
    perm = np.array([5, 2, 7, 0, 3, 6, 1, 4])
    a_shuf = cf.TripletMatrix(3, 5, a.rows[perm], a.cols[perm], a.vals[perm])
    f = cf.build_uv(a_shuf)
    rng = np.random.default_rng(11)
    y = rng.standard_normal(f.o)
    s = rng.standard_normal(f.m)
    x = rng.standard_normal(f.n)
    out = dict(
        dense=dense, rows=a_shuf.rows.copy(), cols=a_shuf.cols.copy(), vals=a_shuf.vals.copy(),
        row_of=f.row_of.copy(), col_of=f.col_of.copy(), val=f.val.copy(),
        fu=f.fu_diag.copy(), fv=f.fv_diag.copy(),
        U_ones=cf.apply_U(f, np.ones(f.o)), Ut_ones=cf.apply_Ut(f, np.ones(f.m)),
        V_seq=cf.apply_V(f, np.arange(1.0, 9.0)), Vt_x=cf.apply_Vt(f, np.array([10.0, 20, 30, 40, 50])),
        rand_y=y, rand_s=s, rand_x=x,
        U_y=cf.apply_U(f, y), Ut_s=cf.apply_Ut(f, s), V_y=cf.apply_V(f, y), Vt_x_rand=cf.apply_Vt(f, x),
        yfac_y=cf.apply_y_factor(f, y),
    )
    np.savez_compressed(os.path.join(OUT, "example1.npz"), **out)


# --------------------------------------------------------------------------
# 2. Cone projections (cones.py:76-110): SPEC examples + random blocks 1..16
#    including the alpha = +-w0 boundary ties.
# --------------------------------------------------------------------------
def projections():
    rng = np.random.default_rng(12)
    blocks = [np.array([3.0, 0, 0, 4]), np.array([5.0, 3, 0, 0]), np.array([-5.0, 3, 0, 0]),
              np.array([-2.0]), np.array([2.0]), np.array([0.0]), np.array([-0.0]),
              np.array([3.0, 4.0]), np.array([-3.0, 4.0]), np.array([5.0, 3.0, 4.0]),
              np.array([-5.0, 3.0, 4.0]), np.array([0.0, 0.0, 0.0])]
    for _ in range(2000):
        q = int(rng.integers(1, 17))
        w = rng.standard_normal(q) * (10.0 ** rng.integers(-3, 4))
        if q > 1 and rng.random() < 0.1:  # boundary tie alpha == |w0| (exact in fp for a single tail entry)
            w[1:] = 0.0
            w[1 + int(rng.integers(0, q - 1))] = abs(w[0]) * (1 if rng.random() < 0.5 else -1)
        blocks.append(w)
    sizes = np.array([b.size for b in blocks], dtype=np.int64)
    w = np.concatenate(blocks)
    out_block = np.concatenate([cf.project_block(b) for b in blocks])
    view = cf.ConeWorkview.from_spec(cf.ConeSpec(tuple(int(s) for s in sizes)))
    out_product = cf.project_product(view, w)
    # LP shortcut path (cones.py:108-109) incl. NaN / -0.0 semantics
    lp_w = np.array([-1.0, 2.0, -0.0, 0.0, np.nan, np.inf, -np.inf, 1e-300, -1e-300])
    lp_view = cf.ConeWorkview.from_spec(cf.ConeSpec.orthant(lp_w.size))
    lp_out = cf.project_product(lp_view, lp_w)
    np.savez_compressed(os.path.join(OUT, "projection.npz"), sizes=sizes, w=w, out_block=out_block,
                        out_product=out_product, lp_w=lp_w, lp_out=lp_out)


# --------------------------------------------------------------------------
# 3. Per-iteration states x,y,z,lam,gamma,delta from the reference step
#    functions, driven exactly like solve() (solver.py:312-317).
# --------------------------------------------------------------------------
KEEP = (1, 2, 3, 4, 5, 10, 25, 50, 75, 100)


def _iterate(p, cfg, init, iters):
    f = cf.build_uv(p.A)
    view = cf.ConeWorkview.from_spec(p.cones)
    st = init.copy() if init is not None else ref_solver.SolverState.zeros(f)
    kept = {}
    for k in range(1, iters + 1):
        st.x = ref_solver.x_update(f, st, cfg, p.c)
        st.y = ref_solver.y_update(f, st, cfg, p.b)
        st.z = ref_solver.z_update(view, st, cfg)
        st.lam, st.gamma, st.delta = ref_solver.dual_update(f, st, cfg, p.b)
        st.iter = k
        if k in KEEP:
            kept[k] = (st.copy(), ref_solver.compute_report(p, f, st))
    return kept


def iterates():
    cases = [
        ("lp_mu1", cf.GenSpec(24, 60, 0.08, "lp", seed=3), 1.0, False),
        ("lp_mu03", cf.GenSpec(30, 50, 0.1, "lp", seed=4), 0.3, False),
        ("socp4_mu5", cf.GenSpec(20, 48, 0.1, "socp4", seed=5), 5.0, False),
        ("socp4_mu07_warm", cf.GenSpec(25, 64, 0.08, "socp4", seed=6), 0.7, True),
        ("lp_raw_mu1_warm", cf.GenSpec(16, 40, 0.12, "lp", seed=7, bounded_mode=False), 1.0, True),
    ]
    for name, spec, mu, warm in cases:
        p = cf.generate(spec)
        f = cf.build_uv(p.A)
        cfg = cf.SolverConfig(mu=mu)
        init = None
        out = _problem_arrays(p)
        out["mu"] = np.float64(mu)
        if warm:
            rng = np.random.default_rng(100 + spec.seed)
            init = ref_solver.SolverState(
                x=rng.standard_normal(f.n), y=rng.standard_normal(f.o), z=rng.standard_normal(f.n),
                lam=rng.standard_normal(f.m), gamma=rng.standard_normal(f.o),
                delta=rng.standard_normal(f.n), iter=0,
            )
            for key in ("x", "y", "z", "lam", "gamma", "delta"):
                out["init_" + key] = getattr(init, key).copy()
        kept = _iterate(p, cfg, init, max(KEEP))
        out["keep"] = np.array(KEEP, dtype=np.int64)
        for k, (st, rep) in kept.items():
            for key in ("x", "y", "z", "lam", "gamma", "delta"):
                out[f"k{k}_{key}"] = getattr(st, key)
            out[f"k{k}_report"] = np.array([float(getattr(rep, fld)) for fld in REPORT_FIELDS])
        np.savez_compressed(os.path.join(OUT, f"iterates_{name}.npz"), **out)


# --------------------------------------------------------------------------
# 4. Whole solves: SPEC analytic fixtures + random instances
# --------------------------------------------------------------------------
def solves():
    analytic = {
        "lp1x1": cf.ProblemInstance(cf.TripletMatrix(1, 1, [0], [0], [1.0]), [1.0], [1.0], cf.ConeSpec.orthant(1)),
        "lp2var": cf.ProblemInstance(cf.TripletMatrix(1, 2, [0, 0], [0, 1], [1.0, 1.0]), [1.0], [1.0, 2.0],
                                     cf.ConeSpec.orthant(2)),
        "socp4": cf.ProblemInstance(cf.TripletMatrix(1, 4, [0], [0], [1.0]), [2.0], [0.0, 0.0, 0.0, -1.0],
                                    cf.ConeSpec((4,))),
    }
    cfgs = {
        "scs1e-3": cf.SolverConfig(),
        "scs1e-9": cf.SolverConfig(eps_prim=1e-9, eps_dual=1e-9, eps_gap=1e-9),
        "osqp": cf.SolverConfig(term_mode="osqp", eps_abs=1e-6, eps_rel=1e-6),
        "target": cf.SolverConfig(term_mode="target", target_prim_res=1e-7, target_gap=1e-7),
        "max7": cf.SolverConfig(max_iters=7, check_every=3),
    }
    out = {}
    names = []
    for pname, p in analytic.items():
        for cname, cfg in cfgs.items():
            r = cf.solve(p, cfg)
            key = f"{pname}__{cname}"
            names.append(key)
            out.update(_trace_arrays(r.trace, key + "__"))
            out[key + "__x"] = r.x
            out[key + "__lam"] = r.lam
    # random instances to a 1e-4 scs tolerance; iteration counts pin termination parity
    rand = {
        "lp_small": (cf.GenSpec(60, 150, 0.05, "lp", seed=21), cf.SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)),
        "socp_small": (cf.GenSpec(40, 120, 0.06, "socp4", seed=22), cf.SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)),
        "lp_mixed_mu2": (cf.GenSpec(50, 100, 0.05, "lp", seed=23), cf.SolverConfig(mu=2.0, check_every=10, term_mode="osqp")),
        "lp_maxiters": (cf.GenSpec(40, 90, 0.05, "lp", seed=24), cf.SolverConfig(max_iters=130, check_every=25)),
    }
    for rname, (spec, cfg) in rand.items():
        p = cf.generate(spec)
        r = cf.solve(p, cfg)
        names.append(rname)
        out.update(_problem_arrays(p, rname + "__"))
        out.update(_trace_arrays(r.trace, rname + "__"))
        out[rname + "__x"] = r.x
        out[rname + "__lam"] = r.lam
        out[rname + "__cfg"] = np.array([cfg.mu, cfg.max_iters, cfg.check_every, ["osqp", "scs", "target"].index(cfg.term_mode),
                                         cfg.eps_abs, cfg.eps_rel, cfg.eps_prim, cfg.eps_dual, cfg.eps_gap])
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(OUT, "solves.npz"), **out)


def mixed_cones():
    """A hand-built mixed-cone problem (sizes 1,2,3,5,1,7,...) incl. a big block of 40."""
    rng = np.random.default_rng(31)
    sizes = [1, 2, 3, 5, 1, 7, 1, 1, 4, 40, 2, 1, 3]
    n = sum(sizes)
    m = 15
    dense = rng.standard_normal((m, n)) * (rng.random((m, n)) < 0.15)
    a = cf.TripletMatrix.from_dense(dense)
    view = cf.ConeWorkview.from_spec(cf.ConeSpec(tuple(sizes)))
    x_feas = cf.project_product(view, rng.standard_normal(n))
    b = dense @ x_feas
    s_feas = cf.project_product(view, rng.standard_normal(n))
    c = s_feas - dense.T @ rng.standard_normal(m)
    p = cf.ProblemInstance(a, b, c, cf.ConeSpec(tuple(sizes)))
    cfg = cf.SolverConfig(mu=1.3)
    kept = _iterate(p, cfg, None, max(KEEP))
    out = _problem_arrays(p)
    out["mu"] = np.float64(1.3)
    out["keep"] = np.array(KEEP, dtype=np.int64)
    for k, (st, rep) in kept.items():
        for key in ("x", "y", "z", "lam", "gamma", "delta"):
            out[f"k{k}_{key}"] = getattr(st, key)
        out[f"k{k}_report"] = np.array([float(getattr(rep, fld)) for fld in REPORT_FIELDS])
    np.savez_compressed(os.path.join(OUT, "iterates_mixed_cones.npz"), **out)


# --------------------------------------------------------------------------
# 5. Generator (generate.py:103-140): small instances verbatim, C1 by hash,
#    plus the C1 golden solve (11,375 iterations at scs 1e-4).
# --------------------------------------------------------------------------
def generator():
    out = {}
    specs = {
        "g_lp": cf.GenSpec(10, 30, 0.1, "lp", seed=0),
        "g_socp": cf.GenSpec(12, 32, 0.2, "socp4", seed=9),
        "g_raw": cf.GenSpec(8, 20, 0.3, "lp", seed=123, bounded_mode=False),
        "g_dense": cf.GenSpec(6, 10, 0.7, "lp", seed=5),  # permutation branch (2*count >= total)
    }
    for name, spec in specs.items():
        g = cf.generate_witnessed(spec)
        out.update(_problem_arrays(g.problem, name + "__"))
        out[name + "__x_feas"] = g.x_feas
        out[name + "__spec"] = np.array([spec.m, spec.n, spec.density, ["lp", "socp4"].index(spec.cone_kind),
                                         spec.seed, int(spec.bounded_mode)])
    c1 = cf.generate(cf.GenSpec(1000, 2000, 0.01, "lp", seed=0))
    out["c1_sha"] = np.array(sha(c1.A.rows, c1.A.cols, c1.A.vals, c1.b, c1.c))
    cfg = cf.SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    r = cf.solve(c1, cfg)
    out.update(_trace_arrays(r.trace, "c1__"))
    out["c1__x"] = r.x
    out["c1__lam"] = r.lam
    np.savez_compressed(os.path.join(OUT, "generator_c1.npz"), **out)
    print("C1:", r.report.iter, r.report.status, r.report.pobj)


if __name__ == "__main__":
    np.seterr(all="ignore")
    example1()
    projections()
    iterates()
    mixed_cones()
    solves()
    generator()
    for fn in sorted(os.listdir(OUT)):
        if fn.endswith(".npz"):
            print(fn, os.path.getsize(os.path.join(OUT, fn)))
