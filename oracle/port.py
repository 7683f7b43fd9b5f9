"""Literal numpy restatement of the reference iteration (TEST INFRASTRUCTURE ONLY).

Every function cites the reference line it restates (paths relative to
/root/reference/pkg/src/conefree). The arithmetic is the reference's: the
same numpy calls in the same order, so on the same inputs the results are
bit-identical to the reference (verified against tests/golden).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

REPORT_FIELDS = ("iter", "prim_res_inf", "prim_res_2", "dual_res_inf", "dual_res_2", "stat_res_inf",
                 "stat_res_2", "ax_inf", "atl_inf", "cone_gap", "pobj", "dobj", "gap")


@dataclass(frozen=True)
class Factors:
    """UVFactors (uv.py:34-55) without the group tuples."""

    m: int
    n: int
    o: int
    row_of: np.ndarray
    col_of: np.ndarray
    val: np.ndarray
    fu: np.ndarray
    fv: np.ndarray


def build_factors(a) -> Factors:
    """build_uv (uv.py:64-98): canonical column-major order, cached diagonals."""
    m, n = int(a.num_rows), int(a.num_cols)
    rows, cols, vals = np.asarray(a.rows, np.int64), np.asarray(a.cols, np.int64), np.asarray(a.vals, np.float64)
    perm = np.lexsort((rows, cols))                                       # uv.py:76
    r, c, v = rows[perm], cols[perm], vals[perm]
    fu = 1.0 / (1.0 + np.bincount(r, weights=v * v, minlength=m))         # uv.py:81
    fv = 1.0 / (1.0 + np.bincount(c, minlength=n))                        # uv.py:82
    return Factors(m, n, int(v.size), r, c, v, fu, fv)


# ------------------------------------------------------------------ operators (uv.py:106-143)
def apply_U(f: Factors, y):
    return np.bincount(f.row_of, weights=f.val * np.asarray(y, np.float64), minlength=f.m)


def apply_Ut(f: Factors, s):
    return f.val * np.asarray(s, np.float64)[f.row_of]


def apply_V(f: Factors, g):
    return np.bincount(f.col_of, weights=np.asarray(g, np.float64), minlength=f.n)


def apply_Vt(f: Factors, x):
    return np.asarray(x, np.float64)[f.col_of]


def apply_y_factor(f: Factors, t):
    """(I + U^T U)^-1 t by the inversion lemma (uv.py:134-143)."""
    return t - apply_Ut(f, f.fu * apply_U(f, t))


# ------------------------------------------------------------------ cones (cones.py:67-110)
def _segments(sizes):
    sizes = np.asarray(sizes, dtype=np.int64)
    starts = np.concatenate(([0], np.cumsum(sizes)[:-1])).astype(np.int64) if sizes.size else sizes
    owner = np.repeat(np.arange(sizes.size, dtype=np.int64), sizes)
    return sizes, starts, owner


def project_product(sizes, w):
    """project_product (cones.py:103-110) incl. the all-unit shortcut (:108-109)."""
    sizes, starts, owner = _segments(sizes)
    w = np.asarray(w, dtype=np.float64)
    if sizes.size == 0 or sizes.max() == 1:
        return np.where(w > 0.0, w, 0.0)
    w1 = w[starts]                                                         # cones.py:69
    sq = w * w
    sq[starts] = 0.0
    alpha = np.sqrt(np.bincount(owner, weights=sq, minlength=sizes.size))  # cones.py:72
    zero_blk = alpha <= -w1                                                # cones.py:78-80
    keep_blk = ~zero_blk & (alpha <= w1)
    scale_blk = ~(zero_blk | keep_blk)
    factor = np.zeros(alpha.shape)
    factor[scale_blk] = w1[scale_blk] / (2.0 * alpha[scale_blk])           # cones.py:83
    out = 0.5 * w + factor[owner] * w                                      # cones.py:84
    out[keep_blk[owner]] = w[keep_blk[owner]]
    out[zero_blk[owner]] = 0.0
    out[starts[scale_blk]] = 0.5 * w1[scale_blk] + 0.5 * alpha[scale_blk]  # cones.py:91
    return out


def project_block(w):
    w = np.asarray(w, dtype=np.float64)
    return project_product(np.array([w.size]), w)


# ------------------------------------------------------------------ iteration (solver.py:168-197)
@dataclass
class OracleState:
    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    lam: np.ndarray
    gamma: np.ndarray
    delta: np.ndarray
    iter: int = 0

    @classmethod
    def zeros(cls, f: Factors):
        return cls(np.zeros(f.n), np.zeros(f.o), np.zeros(f.n), np.zeros(f.m), np.zeros(f.o), np.zeros(f.n))

    def copy(self):
        return OracleState(self.x.copy(), self.y.copy(), self.z.copy(), self.lam.copy(), self.gamma.copy(),
                           self.delta.copy(), self.iter)


def step(f: Factors, sizes, st: OracleState, mu: float, b, c) -> OracleState:
    """One iteration in Gauss-Seidel order x -> y -> z -> duals (solver.py:313-317)."""
    x = f.fv * (apply_V(f, st.y + st.gamma / mu) + st.z + st.delta / mu - c / mu)       # :171-176
    t = apply_Ut(f, b - st.lam / mu) + apply_Vt(f, x) - st.gamma / mu                  # :182
    y = apply_y_factor(f, t)                                                            # :183
    z = project_product(sizes, x - st.delta / mu)                                       # :188
    lam = st.lam + mu * (apply_U(f, y) - b)                                             # :194
    gamma = st.gamma + mu * (y - apply_Vt(f, x))                                        # :195
    delta = st.delta + mu * (z - x)                                                     # :196
    return OracleState(x, y, z, lam, gamma, delta, st.iter + 1)


def iterate(f, sizes, st, mu, b, c, n_iters):
    for _ in range(n_iters):
        st = step(f, sizes, st, mu, b, c)
    return st


def _norms(v):
    """solver.py:200-203."""
    if v.size == 0:
        return 0.0, 0.0
    return float(np.max(np.abs(v))), float(math.sqrt(np.dot(v, v)))


def compute_report(f: Factors, st: OracleState, b, c) -> dict:
    """compute_report (solver.py:206-242) as a dict with a 'status' key."""
    finite = all(np.isfinite(v).all() for v in (st.x, st.y, st.z, st.lam, st.gamma, st.delta))
    ax = apply_U(f, apply_Vt(f, st.x))
    prim = ax - b
    atl = apply_V(f, apply_Ut(f, st.lam))
    dual = atl + c
    stat = dual - st.delta
    pobj = float(np.dot(c, st.x))
    blam = float(np.dot(b, st.lam))
    rep = {"iter": st.iter}
    rep["prim_res_inf"], rep["prim_res_2"] = _norms(prim)
    rep["dual_res_inf"], rep["dual_res_2"] = _norms(dual)
    rep["stat_res_inf"], rep["stat_res_2"] = _norms(stat)
    rep["ax_inf"] = _norms(ax)[0]
    rep["atl_inf"] = _norms(atl)[0]
    rep["cone_gap"] = float(np.max(np.abs(st.x - st.z))) if st.x.size else 0.0
    rep["pobj"], rep["dobj"], rep["gap"] = pobj, -blam, pobj + blam
    rep["status"] = "running" if finite else "diverged"
    return rep


def check_termination(rep: dict, cfg, b, c) -> str:
    """check_termination (solver.py:245-272)."""
    if rep["status"] != "running":
        return rep["status"]
    if cfg.term_mode == "osqp":
        ep = cfg.eps_abs + cfg.eps_rel * max(rep["ax_inf"], _norms(b)[0])
        ed = cfg.eps_abs + cfg.eps_rel * max(rep["atl_inf"], _norms(c)[0])
        ok = rep["prim_res_inf"] < ep and rep["stat_res_inf"] < ed
    elif cfg.term_mode == "scs":
        ok = (rep["prim_res_2"] <= cfg.eps_prim * (1.0 + _norms(b)[1])
              and rep["stat_res_2"] <= cfg.eps_dual * (1.0 + _norms(c)[1])
              and abs(rep["gap"]) <= cfg.eps_gap * (1.0 + abs(rep["pobj"]) + abs(rep["dobj"])))
    else:
        ok = rep["prim_res_2"] < cfg.target_prim_res and abs(rep["gap"]) < cfg.target_gap
    return "solved" if ok else "running"


def solve(p, cfg, init: OracleState | None = None, max_wall_s: float | None = None):
    """The solve() loop (solver.py:299-334); returns (x, lam, trace of report dicts, state).

    max_wall_s bounds a CPU-baseline sample: the loop stops (status
    'sampled') after the first iteration that crosses it.
    """
    import time

    b, c = np.asarray(p.b, np.float64), np.asarray(p.c, np.float64)
    sizes = np.asarray(p.cones.block_sizes, dtype=np.int64) if not hasattr(p.cones, "sizes_array") \
        else p.cones.sizes_array()
    f = build_factors(p.A)
    st = init.copy() if init is not None else OracleState.zeros(f)
    trace = []
    t0 = time.perf_counter()
    for k in range(1, cfg.max_iters + 1):
        st = step(f, sizes, st, cfg.mu, b, c)
        st.iter = k
        if k % cfg.check_every == 0 or k == cfg.max_iters:
            rep = compute_report(f, st, b, c)
            status = check_termination(rep, cfg, b, c)
            if status == "running" and k == cfg.max_iters:
                status = "max_iters"
            rep["status"] = status
            trace.append(rep)
            if status != "running":
                break
        if max_wall_s is not None and time.perf_counter() - t0 > max_wall_s:
            trace.append({"iter": k, "status": "sampled"})
            break
    return st.x.copy(), st.lam.copy(), trace, st


def dense_iterate(f: Factors, sizes, st: OracleState, mu, b, c) -> OracleState:
    """Dense explicit-matrix mirror (oracle.py:84-102) for tiny problems."""
    u = np.zeros((f.m, f.o))
    v = np.zeros((f.n, f.o))
    u[f.row_of, np.arange(f.o)] = f.val
    v[f.col_of, np.arange(f.o)] = 1.0
    fu = 1.0 / (1.0 + np.diag(u @ u.T))
    fv = 1.0 / (1.0 + np.diag(v @ v.T))
    x = fv * (v @ (st.y + st.gamma / mu) + st.z + st.delta / mu - c / mu)
    t = u.T @ (b - st.lam / mu) + v.T @ x - st.gamma / mu
    y = t - u.T @ (fu * (u @ t))
    z = project_product(sizes, x - st.delta / mu)
    lam = st.lam + mu * (u @ y - b)
    gamma = st.gamma + mu * (y - v.T @ x)
    delta = st.delta + mu * (z - x)
    return OracleState(x, y, z, lam, gamma, delta, st.iter + 1)
