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
import conefree.bench  # noqa: E402,F401
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


BENCH_JOBS = (
    # (instance_id, m, n, density, cone_kind, seed): C4-shaped jobs (batched on the GPU),
    # an SOCP one, and one above benchrun.BATCH_MAX_NNZ (solved alone)
    (0, 100, 200, 0.05, "lp", 0), (1, 100, 200, 0.05, "lp", 1), (2, 100, 200, 0.05, "lp", 2),
    (3, 100, 200, 0.05, "lp", 3), (4, 100, 200, 0.05, "socp4", 7), (5, 200, 800, 0.15, "lp", 3),
)


def bench_rows():
    """The reference's own run_bench (bench.py:96-106) over BENCH_JOBS: deterministic columns."""
    cfg = cf.SolverConfig(term_mode="scs", eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    jobs = [cf.bench.BenchJob(i, cf.GenSpec(m, n, dens, kind, seed), cfg) for i, m, n, dens, kind, seed in BENCH_JOBS]
    rows = cf.bench.run_bench(jobs, workers=1)
    num = ("instance_id", "m", "n", "nnz", "density", "mu", "iters", "prim_res_2", "dual_res_2", "gap", "cone_gap")
    out = {k: np.array([r[k] for r in rows]) for k in num}
    out["cone_kind"] = np.array([r["cone_kind"] for r in rows])
    out["term_mode"] = np.array([r["term_mode"] for r in rows])
    out["status"] = np.array([r["status"] for r in rows])
    out["jobs"] = np.array([[i, m, n, seed] for i, m, n, dens, kind, seed in BENCH_JOBS], dtype=np.int64)
    out["densities"] = np.array([dens for _, _, _, dens, _, _ in BENCH_JOBS])
    out["kinds"] = np.array([kind for _, _, _, _, kind, _ in BENCH_JOBS])
    np.savez_compressed(os.path.join(OUT, "bench_rows.npz"), **out)
    print("bench_rows:", [(r["instance_id"], r["iters"], r["status"]) for r in rows])


def _coneprob_cases():
    """Valid and malformed CONEPROB texts (mutations of one small instance)."""
    from conefree import fileio

    p = cf.generate(cf.GenSpec(4, 8, 0.5, "socp4", seed=5))
    base = fileio.write_problem(p)
    L = base.splitlines()
    nnz = p.A.nnz
    e0, e_last = 3, 3 + nnz - 1            # 0-based line indices of the first/last entry
    b0, c0 = 3 + nnz, 3 + nnz + 4
    cases = [base, base.replace("\n", "\r\n"), base.replace("\n", "\r"), "# comment\n\n" + base,
             base.replace("\n", "\n  # note\n", 5), base.replace("\n", "\x0b", 3), base.replace("\n", "\x0c", 4),
             base.replace("\n", "\x1c", 2), base.replace(" ", "\t"), base.replace(" ", " \x1f "), "", "\n\n",
             "CONEPROB 2\n", "coneprob 1\n", "CONEPROB  1\n", "CONEPROB 1", "CONEPROB 1\n4 8\n",
             "CONEPROB 1\n4 8 x\n", "CONEPROB 1\n4 1.5 3\n", "CONEPROB 1\n0 8 3\n", "CONEPROB 1\n4 8 -1\n",
             "CONEPROB 1\n4 8 1_0\nCONE 1 8\n", "CONEPROB 1\n+4 8 0\nCONES\n", "CONEPROB 1\n4 8 0\nCONES x\n",
             "CONEPROB 1\n4 8 0\nCONES 2 4\n", "CONEPROB 1\n4 8 0\nCONES 2 4 y\n", "CONEPROB 1\n4 8 0\nCONES 2 8 0\n",
             "CONEPROB 1\n4 8 0\nCONES 2 4 3\n", "CONEPROB 1\n4 8 0\nCONES 2 4 4\n",
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 1_0.5\n1e1_0\n-2\n",
             "CONEPROB 1\n1 1 0\nCONES 1 1\n1\n2\n3\n", "CONEPROB 1\n1 1 0\nCONES 1 1\n1 2\n2\n",
             "CONEPROB 1\n1 1 0\nCONES 1 1\ninf\n2\n", "CONEPROB 1\n1 1 0\nCONES 1 1\n1\n-NaN\n",
             "CONEPROB 1\n4 8 0\nCONES 2 4 4\n" + "1\n" * 4 + "1\n" * 7,
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 it's\n", 'CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 "q\n',
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 a\\b'\"\n", "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 1e-400\n",
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 -0.0\n", "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 1e999\n",
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 0x10\n", "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 1__0\n",
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 .5\n1.\n-.5e+3\n", "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 1e\n",
             "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 +Infinity\n", "CONEPROB 1\n1 1 1\nCONES 1 1\n00 0_0 7\n1\n1\n",
             "CONEPROB 1\n99999999999999999999 1 0\nCONES 1 1\n", "CONEPROB 1\n1 1 1\nCONES 1 1\n0 0 7 # x\n",
             "# caf\u00e9\n" + base, base.replace("\n", "\u2028", 1), "CONEPROB 1\n2 1 2\nCONES 1 1\n0 0 1\n0 0 2\n1\n1\n1\n"]
    muts = {
        e0 + 1: "1 2", e0 + 2: "x 0 1.0", e0 + 3: "0 y 1.0", e_last: "0 0 z", e0: "9 0 1.0", e0 + 4: "0 -1 1.0",
        e_last - 1: "0 0 nan", b0: "b?", c0 + 2: "inf", c0 + 7: "1 2",
    }
    for li, text in muts.items():
        lines = list(L)
        lines[li] = text
        cases.append("\n".join(lines) + "\n")
    # duplicates: an entry repeated later; and a zero-valued duplicate (zero wins on that line)
    for a, bq, txt in ((e0, e0 + 5, None), (e0 + 2, e_last, "zero")):
        lines = list(L)
        i, j, _ = lines[a].split()
        lines[bq] = f"{i} {j} {'0.0' if txt else '2.5'}"
        cases.append("\n".join(lines) + "\n")
    lines = list(L)
    lines[e0 + 6] = lines[e0 + 1]
    lines[e0 + 3] = "3 x 1"
    cases.append("\n".join(lines) + "\n")
    cases += ["\n".join(L[:e0 + 3]) + "\n", "\n".join(L[:b0 + 2]) + "\n", "\n".join(L[:-1]) + "\n",
              base + "extra\n", base + "# trailing comment\n\n"]
    return cases


def coneprob_cases():
    """parse_problem on valid and malformed texts: ParseError line/message or a hash of the arrays."""
    from conefree import fileio

    texts, lines, msgs, hashes = [], [], [], []
    for t in _coneprob_cases():
        try:
            p = fileio.parse_problem(t)
            lines.append(-1)
            msgs.append("")
            hashes.append(sha(p.A.rows, p.A.cols, p.A.vals, p.b, p.c, np.asarray(p.cones.block_sizes)))
        except fileio.ParseError as e:
            lines.append(e.line)
            msgs.append(e.message)
            hashes.append("")
        except Exception as e:   # e.g. numpy refusing a huge m: the same exception is expected
            lines.append(-2)
            msgs.append(f"{type(e).__name__}: {e}")
            hashes.append("")
        texts.append(t)
    np.savez_compressed(os.path.join(OUT, "coneprob_cases.npz"), texts=np.array(texts), lines=np.array(lines),
                        messages=np.array(msgs), hashes=np.array(hashes))
    print("coneprob_cases:", len(texts), "cases,", sum(1 for x in lines if x >= 0), "errors")


if __name__ == "__main__":
    np.seterr(all="ignore")
    example1()
    projections()
    iterates()
    mixed_cones()
    solves()
    generator()
    bench_rows()
    coneprob_cases()
    for fn in sorted(os.listdir(OUT)):
        if fn.endswith(".npz"):
            print(fn, os.path.getsize(os.path.join(OUT, fn)))
