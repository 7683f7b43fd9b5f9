"""The drop-in solver API: ``solve(p, cfg=None, init=None) -> SolveResult``.

Same signature, types, semantics and errors as the reference
``conefree.solver`` (solver.py:61-334):

* ``SolverConfig`` (solver.py:61-103) — same fields, defaults and ValueErrors.
* ``SolverState`` (:106-138), ``IterationReport`` (:141-158),
  ``SolveResult`` (:161-165).
* ``check_termination`` (:245-272) — host restatement; ``solve`` uses it to
  re-decide every device report and refuses to return if the device and the
  host disagree (they evaluate the same IEEE expressions on the same numbers).
* ``solve`` (:275-334) — validate, build, warm start, loop with a report every
  ``check_every`` iterations and at ``max_iters``, early exit on a terminal
  status. The loop body runs on the GPU only (libcfb200, sm_100a); there is no
  CPU path.

The ``p``, ``cfg`` and ``init`` arguments are duck-typed, so the reference's
own ``ProblemInstance`` / ``SolverConfig`` / ``SolverState`` objects work too.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass, replace
from typing import NamedTuple

import numpy as np

from .engine import DevicePlan, ProblemRejected, config_struct
from .problem import cone_sizes_array, validate

__all__ = [
    "solve_batch",
    "SolverConfig",
    "SolverState",
    "IterationReport",
    "SolveResult",
    "check_termination",
    "solve",
    "norms",
]

TERM_MODES = ("osqp", "scs", "target")


@dataclass(frozen=True)
class SolverConfig:
    """Penalty, iteration budget and termination test (solver.py:61-103)."""

    mu: float = 1.0
    max_iters: int = 100_000
    check_every: int = 25
    term_mode: str = "scs"
    eps_abs: float = 1e-4
    eps_rel: float = 1e-3
    eps_prim: float = 1e-3
    eps_dual: float = 1e-3
    eps_gap: float = 1e-3
    target_prim_res: float | None = None
    target_gap: float | None = None

    def __post_init__(self):
        if not self.mu > 0:
            raise ValueError("mu must be > 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.check_every < 1:
            raise ValueError("check_every must be >= 1")
        if self.term_mode not in TERM_MODES:
            raise ValueError(f"term_mode must be one of {TERM_MODES}")
        for field in ("eps_abs", "eps_rel", "eps_prim", "eps_dual", "eps_gap"):
            if getattr(self, field) < 0:
                raise ValueError(f"{field} must be >= 0")
        if self.term_mode == "target" and (self.target_prim_res is None or self.target_gap is None):
            raise ValueError("target mode needs target_prim_res and target_gap")


@dataclass
class SolverState:
    """Iterates x, y, z and multipliers lam, gamma, delta (solver.py:106-138).

    y and gamma are o-length, in canonical (column-major) nonzero order.
    """

    x: np.ndarray
    y: np.ndarray
    z: np.ndarray
    lam: np.ndarray
    gamma: np.ndarray
    delta: np.ndarray
    iter: int = 0

    @classmethod
    def zeros(cls, f) -> "SolverState":
        """Cold start for anything with m, n, o (e.g. the reference's UVFactors)."""
        m, n, o = int(f.m), int(f.n), int(f.o)
        return cls(x=np.zeros(n), y=np.zeros(o), z=np.zeros(n), lam=np.zeros(m), gamma=np.zeros(o),
                   delta=np.zeros(n))

    def copy(self) -> "SolverState":
        return SolverState(x=self.x.copy(), y=self.y.copy(), z=self.z.copy(), lam=self.lam.copy(),
                           gamma=self.gamma.copy(), delta=self.delta.copy(), iter=self.iter)


@dataclass(frozen=True)
class IterationReport:
    """Residual norms, objectives and status at one evaluated iteration."""

    iter: int
    prim_res_inf: float
    prim_res_2: float
    dual_res_inf: float
    dual_res_2: float
    stat_res_inf: float
    stat_res_2: float
    ax_inf: float
    atl_inf: float
    cone_gap: float
    pobj: float
    dobj: float
    gap: float
    status: str = "running"


class SolveResult(NamedTuple):
    x: np.ndarray
    lam: np.ndarray
    report: IterationReport
    trace: tuple


def norms(v) -> tuple:
    """(inf-norm, 2-norm) exactly as solver.py:200-203."""
    v = np.asarray(v, dtype=np.float64)
    if v.size == 0:
        return 0.0, 0.0
    return float(np.max(np.abs(v))), float(math.sqrt(np.dot(v, v)))


def _decide(report, cfg, b_norms, c_norms) -> str:
    """check_termination with the problem norms precomputed (solver.py:245-272)."""
    if report.status == "diverged":
        return "diverged"
    if report.status != "running":
        return report.status
    if cfg.term_mode == "osqp":
        eps_prim = cfg.eps_abs + cfg.eps_rel * max(report.ax_inf, b_norms[0])
        eps_dual = cfg.eps_abs + cfg.eps_rel * max(report.atl_inf, c_norms[0])
        ok = report.prim_res_inf < eps_prim and report.stat_res_inf < eps_dual
    elif cfg.term_mode == "scs":
        ok = (
            report.prim_res_2 <= cfg.eps_prim * (1.0 + b_norms[1])
            and report.stat_res_2 <= cfg.eps_dual * (1.0 + c_norms[1])
            and abs(report.gap) <= cfg.eps_gap * (1.0 + abs(report.pobj) + abs(report.dobj))
        )
    else:
        ok = report.prim_res_2 < cfg.target_prim_res and abs(report.gap) < cfg.target_gap
    return "solved" if ok else "running"


def check_termination(report, cfg, p) -> str:
    """Map a report onto solved/running/diverged for the configured mode."""
    return _decide(report, cfg, norms(p.b), norms(p.c))


def _host_shapes_ok(p) -> bool:
    a = p.A
    if np.asarray(p.b).size != a.num_rows or np.asarray(p.c).size != a.num_cols:
        return False
    sizes = cone_sizes_array(p.cones)
    return bool(sizes.size == 0 or sizes.min() >= 1) and int(sizes.sum()) == a.num_cols


def _raise_invalid(p):
    rep = validate(p)
    if rep.ok:  # pragma: no cover - the device and host checks disagree
        raise RuntimeError("device validation rejected a problem the host validate() accepts")
    raise ValueError("invalid problem: " + "; ".join(rep.violations[:3]))


def _to_report(d: dict) -> IterationReport:
    return IterationReport(
        iter=d["iter"], prim_res_inf=d["prim_res_inf"], prim_res_2=d["prim_res_2"],
        dual_res_inf=d["dual_res_inf"], dual_res_2=d["dual_res_2"], stat_res_inf=d["stat_res_inf"],
        stat_res_2=d["stat_res_2"], ax_inf=d["ax_inf"], atl_inf=d["atl_inf"], cone_gap=d["cone_gap"],
        pobj=d["pobj"], dobj=d["dobj"], gap=d["gap"],
        status="diverged" if d["nonfinite"] else "running",
    )


def build_plan(p, stream: int | None = None) -> DevicePlan:
    """validate + build_uv on the device; raises ValueError like solver.py:300-307."""
    if not _host_shapes_ok(p):
        _raise_invalid(p)
    try:
        return DevicePlan.from_problem(p, stream=stream)
    except ProblemRejected:
        _raise_invalid(p)


def run_plan(plan: DevicePlan, p, cfg, b_norms=None, c_norms=None) -> SolveResult:
    """Run the solve() loop on an existing plan from its current state."""
    b_norms = norms(p.b) if b_norms is None else b_norms
    c_norms = norms(p.c) if c_norms is None else c_norms
    x, lam, raw = plan.run(config_struct(cfg, b_norms, c_norms))
    trace = []
    for d in raw:
        rep = _to_report(d)
        status = _decide(rep, cfg, b_norms, c_norms)
        if status == "running" and rep.iter == cfg.max_iters:
            status = "max_iters"
        if status != d["status"]:
            raise RuntimeError(
                f"device termination test ({d['status']}) disagrees with check_termination ({status}) "
                f"at iteration {rep.iter}")
        trace.append(replace(rep, status=status))
    return SolveResult(x=x, lam=lam, report=trace[-1], trace=tuple(trace))


def solve(p, cfg: SolverConfig | None = None, init: SolverState | None = None) -> SolveResult:
    """Run the ADMM loop on the GPU until a terminal status (solver.py:275-334)."""
    cfg = cfg or SolverConfig()
    # the host norms (numpy, GIL released) overlap the device setup (ctypes, GIL released)
    box = {}

    def _norms():
        try:
            box["b"], box["c"] = norms(p.b), norms(p.c)
        except Exception:   # re-raised by run_plan computing them again
            pass

    if init is None and _cluster_candidate(p):
        res = _solve_cluster(p, cfg)
        if res is not None:
            return res
    th = threading.Thread(target=_norms, daemon=True)
    th.start()
    try:
        plan = build_plan(p)
    finally:
        th.join()
    try:
        if init is not None:
            plan.set_state(cfg.mu, init, export=False)
        return run_plan(plan, p, cfg, box.get("b"), box.get("c"))
    finally:
        plan.close()


# Mid-size problems run in the cluster-resident kernel (csrc/cf_batch.cu k_cluster): one
# launch for the whole loop, iterates in the distributed shared memory of up to 16 CTAs.
# The estimate below is conservative; cf_cluster_solve makes the exact decision.
_CLUSTER_TRACE_MAX = 1 << 16   # cf_batch.cu kMaxClusterTrace
_LAST_CLUSTER = 0   # cluster size of the last cf_cluster_solve call (0: did not fit), for tests

_PLAN_KNOBS = ("CF_PANEL_MB", "CF_BAND_MB", "CF_FORCE_LARGE_TILES", "CF_NO_LARGE_TILES", "CF_GROUP_CONES",
               "CF_NO_COL_RUNS", "CF_LIB_PATH")


def _cluster_candidate(p) -> bool:
    import os

    if os.environ.get("CF_NO_CLUSTER", "") not in ("", "0") or not _host_shapes_ok(p):
        return False
    if any(os.environ.get(k) for k in _PLAN_KNOBS):   # a plan-engine configuration was asked for
        return False
    m, n, o = int(p.A.num_rows), int(p.A.num_cols), int(np.asarray(p.A.vals).size)
    if m < 1 or n < 1:
        return False
    own = 1.3 * (24 * o + 36 * m + 52 * n) / 16
    return 8 * (n + 3 * m) + own + 4096 <= 227 * 1024


def _solve_cluster(p, cfg, timing: dict | None = None) -> SolveResult | None:
    """solve() in one cluster launch (cf_cluster_solve); None when the problem does not fit.
    ``timing``, if given, receives the loop kernel's device time and the cluster size."""
    import ctypes

    from ._lib import CF_EPROBLEM, CfChecks, CfReport, check, lib
    from .engine import report_to_dict

    m, n = int(p.A.num_rows), int(p.A.num_cols)
    rows = np.ascontiguousarray(p.A.rows, dtype=np.int64)
    cols = np.ascontiguousarray(p.A.cols, dtype=np.int64)
    vals = np.ascontiguousarray(p.A.vals, dtype=np.float64)
    b = np.ascontiguousarray(p.b, dtype=np.float64)
    c = np.ascontiguousarray(p.c, dtype=np.float64)
    sizes = np.ascontiguousarray(cone_sizes_array(p.cones), dtype=np.int64)
    bn, cn = norms(b), norms(c)
    cs = config_struct(cfg, bn, cn)
    x = np.empty(n)
    lam = np.empty(m)
    final = CfReport()
    nrep = ctypes.c_int32()
    cap = -(-int(cfg.max_iters) // int(cfg.check_every))
    if cap > _CLUSTER_TRACE_MAX:   # the cluster kernel keeps its trace on the device: plan path
        return None
    tr = (CfReport * cap)()
    chk = CfChecks()
    used = ctypes.c_int32()
    el = ctypes.c_double()

    def ptr(a):
        return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)

    rc = lib().cf_cluster_solve(m, n, int(vals.size), ptr(rows), ptr(cols), ptr(vals), ptr(b), ptr(c),
                                int(sizes.size), ptr(sizes), ctypes.byref(cs), ptr(x), ptr(lam),
                                ctypes.byref(final), ctypes.byref(nrep), tr, cap, ctypes.byref(chk),
                                ctypes.byref(used), ctypes.byref(el))
    if rc == CF_EPROBLEM:
        _raise_invalid(p)
    check(rc, "cf_cluster_solve")
    global _LAST_CLUSTER
    _LAST_CLUSTER = int(used.value)
    if used.value == 0:
        return None
    if timing is not None:
        timing["kernel_ms"] = el.value
        timing["cluster"] = int(used.value)
    trace = []
    for j in range(int(nrep.value)):
        d = report_to_dict(tr[j])
        rep = _to_report(d)
        status = _decide(rep, cfg, bn, cn)
        if status == "running" and rep.iter == cfg.max_iters:
            status = "max_iters"
        if status != d["status"]:
            raise RuntimeError(f"device termination test ({d['status']}) disagrees with check_termination "
                               f"({status}) at iteration {rep.iter}")
        trace.append(replace(rep, status=status))
    return SolveResult(x=x, lam=lam, report=trace[-1], trace=tuple(trace))


# shared memory of the batched kernel for a batch whose largest dimensions are m, n, o, k
# (cf_batch.cu batch_smem) and the per-CTA opt-in limit of sm_100
_BATCH_SMEM_LIMIT = 227 * 1024


def _batch_smem(m: int, n: int, o: int, k: int) -> int:
    # + the length-ranked row and column orders (CF_BATCH_RANK)
    return 8 * (2 * o + 7 * m + 7 * n + 32) + 4 * (2 * o + m + 1 + n + 1 + k + 1 + m + n) + 16


def solve_batch(problems, cfg: SolverConfig | None = None, trace: bool = True, timing: dict | None = None,
                workers: int = 8) -> list:
    """Solve many independent problems at once: ``[solve(p, cfg) for p in problems]``.

    The reference batches with a process pool over ``solve`` (bench.py:96-106).
    Here the problems that fit one CTA's shared memory run in the batched
    kernel (csrc/cf_batch.cu, SURVEY config C4): one CTA per problem, every
    iterate on chip, per-problem termination. The others are solved
    ``workers`` at a time, each with its own plan and CUDA stream. Each result
    is the SolveResult ``solve(p, cfg)`` returns (same iterates, statuses and
    iteration counts; ``trace=False`` keeps only the final report), in input
    order. ``timing``, if given, receives the device time of the batched kernel.
    """
    problems = list(problems)
    # greedy: smallest first while the batch's dimension caps still fit
    dims = []
    for i, p in enumerate(problems):
        k = len(cone_sizes_array(p.cones)) if _host_shapes_ok(p) else 0
        dims.append((int(p.A.num_rows), int(p.A.num_cols), int(np.asarray(p.A.vals).size), k, i))
    order = sorted(dims, key=lambda t: _batch_smem(*t[:4]))
    fit, cm, cn, co, ck = [], 0, 0, 0, 0
    for m, n, o, k, i in order:
        nm, nn, no, nk = max(cm, m), max(cn, n), max(co, o), max(ck, k)
        if _batch_smem(nm, nn, no, nk) > _BATCH_SMEM_LIMIT:
            break
        fit.append(i)
        cm, cn, co, ck = nm, nn, no, nk
    rest = sorted(set(range(len(problems))) - set(fit))
    out = [None] * len(problems)
    if fit:
        fit.sort()
        for i, r in zip(fit, _solve_batch_kernel([problems[i] for i in fit], cfg, trace, timing, ids=fit)):
            out[i] = r
    if rest:
        from concurrent.futures import ThreadPoolExecutor

        def one(i):
            r = solve(problems[i], cfg)
            return r if trace else r._replace(trace=(r.report,))

        with ThreadPoolExecutor(max_workers=max(1, int(workers))) as pool:
            for i, r in zip(rest, pool.map(one, rest)):
                out[i] = r
    return out


def _solve_batch_kernel(problems, cfg: SolverConfig | None = None, trace: bool = True,
                        timing: dict | None = None, ids=None) -> list:
    """The batched kernel on problems that fit one CTA each (see solve_batch); ids: the
    problems' positions in the caller's list (error messages)."""
    import ctypes

    from . import _lib
    from ._lib import CfChecks, CfReport, check, lib
    from .engine import config_struct, report_to_dict

    cfg = cfg or SolverConfig()
    problems = list(problems)
    P = len(problems)
    if P == 0:
        return []
    for i, p in enumerate(problems):
        if not _host_shapes_ok(p):
            rep = validate(p)
            raise ValueError(f"problem {ids[i] if ids else i}: invalid problem: " + "; ".join(rep.violations[:3]))
    ms = np.array([p.A.num_rows for p in problems], dtype=np.int64)
    ns = np.array([p.A.num_cols for p in problems], dtype=np.int64)
    row_off = np.concatenate(([0], np.cumsum(ms))).astype(np.int64)
    col_off = np.concatenate(([0], np.cumsum(ns))).astype(np.int64)
    rows = np.concatenate([np.asarray(p.A.rows, np.int64) + row_off[i] for i, p in enumerate(problems)])
    cols = np.concatenate([np.asarray(p.A.cols, np.int64) + col_off[i] for i, p in enumerate(problems)])
    vals = np.concatenate([np.asarray(p.A.vals, np.float64) for p in problems])
    b = np.concatenate([np.asarray(p.b, np.float64) for p in problems])
    c = np.concatenate([np.asarray(p.c, np.float64) for p in problems])
    sizes = np.concatenate([cone_sizes_array(p.cones) for p in problems]).astype(np.int64)
    bn = [norms(p.b) for p in problems]
    cn = [norms(p.c) for p in problems]
    cfgs = (_lib.CfConfig * P)(*[config_struct(cfg, bn[i], cn[i]) for i in range(P)])
    M, N = int(row_off[-1]), int(col_off[-1])
    x = np.empty(N)
    lam = np.empty(M)
    finals = (CfReport * P)()
    nrep = np.zeros(P, dtype=np.int32)
    cap = -(-int(cfg.max_iters) // int(cfg.check_every)) if trace else 0
    if trace and P * cap * ctypes.sizeof(CfReport) > (4 << 30):
        raise ValueError("solve_batch: the full traces would need more than 4 GiB; pass trace=False")
    tr = (CfReport * max(P * cap, 1))()
    chk = CfChecks()
    el = ctypes.c_double()

    def ptr(a):
        return ctypes.c_void_p(a.ctypes.data) if a.size else ctypes.c_void_p(0)

    rc = lib().cf_batch_solve(P, ptr(row_off), ptr(col_off), int(vals.size), ptr(rows), ptr(cols), ptr(vals),
                              ptr(b), ptr(c), int(sizes.size), ptr(sizes), cfgs, ptr(x), ptr(lam), finals,
                              ptr(nrep), tr if cap else None, cap, ctypes.byref(chk), ctypes.byref(el))
    if rc == _lib.CF_EPROBLEM:
        for i, p in enumerate(problems):
            rep = validate(p)
            if not rep.ok:
                raise ValueError(f"problem {ids[i] if ids else i}: invalid problem: " + "; ".join(rep.violations[:3]))
    check(rc, "cf_batch_solve")
    if timing is not None:
        timing["kernel_ms"] = el.value
    out = []
    for i, p in enumerate(problems):
        def host_report(d):
            rep = _to_report(d)
            status = _decide(rep, cfg, bn[i], cn[i])
            if status == "running" and rep.iter == cfg.max_iters:
                status = "max_iters"
            if status != d["status"]:
                raise RuntimeError(f"problem {ids[i] if ids else i}: device termination ({d['status']}) disagrees with "
                                   f"check_termination ({status}) at iteration {rep.iter}")
            return replace(rep, status=status)

        final = host_report(report_to_dict(finals[i]))
        if cap:
            k = int(nrep[i])
            reps = tuple(host_report(report_to_dict(tr[i * cap + j])) for j in range(k))
        else:
            reps = (final,)
        out.append(SolveResult(x=x[col_off[i]:col_off[i + 1]].copy(), lam=lam[row_off[i]:row_off[i + 1]].copy(),
                               report=final, trace=reps))
    return out
