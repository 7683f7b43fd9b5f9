"""DevicePlan: one problem instance resident on the B200 (a ``cf_plan``).

Thin Python owner of the C-ABI handle. It stages the reference's input
types into the library (host numpy arrays, or device pointers for
HBM-resident inputs), exposes the per-iteration probing API used by the
parity tests (set_state / iterate / get_state / report) and the whole-loop
``run`` used by :func:`paper_2203_05027_b200.api.solve`.
"""

from __future__ import annotations

import ctypes
from ctypes import byref, c_double, c_int32, c_int64, c_void_p

import numpy as np

from . import _lib
from ._lib import CfChecks, CfConfig, CfReport, check, lib
from .problem import cone_sizes_array

__all__ = ["DevicePlan", "ProblemRejected", "report_to_dict"]


class ProblemRejected(Exception):
    """The device checks of cf_plan_create found validate() violations."""

    def __init__(self, checks: CfChecks, msg: str):
        super().__init__(msg)
        self.checks = checks


def _ptr(arr) -> c_void_p:
    return c_void_p(arr.ctypes.data) if arr is not None and arr.size else c_void_p(0)


def _as(arr, dtype) -> np.ndarray:
    return np.ascontiguousarray(arr, dtype=dtype)


REPORT_FIELDS = ("prim_res_inf", "prim_res_2", "dual_res_inf", "dual_res_2", "stat_res_inf",
                 "stat_res_2", "ax_inf", "atl_inf", "cone_gap", "pobj", "dobj", "gap")


def report_to_dict(r: CfReport) -> dict:
    d = {"iter": int(r.iter), "status": _lib.STATUS_NAMES[r.status], "nonfinite": bool(r.nonfinite)}
    for f in REPORT_FIELDS:
        d[f] = float(getattr(r, f))
    return d


CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: the legacy default stream (torch's default stream)


class DevicePlan:
    """Owner of a cf_plan handle (device copy of A in CSR + CSC, cones, iterates)."""

    def __init__(self, handle: c_void_p, m: int, n: int, o: int):
        self._h = handle
        self.m, self.n, self.o = m, n, o

    # ------------------------------------------------------------------ creation
    @classmethod
    def from_problem(cls, p, stream: int | None = None) -> "DevicePlan":
        """Host ProblemInstance (this package's or the reference's) -> device plan."""
        a = p.A
        m, n = int(a.num_rows), int(a.num_cols)
        rows, cols, vals = _as(a.rows, np.int64), _as(a.cols, np.int64), _as(a.vals, np.float64)
        b, c = _as(p.b, np.float64), _as(p.c, np.float64)
        sizes = _as(cone_sizes_array(p.cones), np.int64)
        return cls._create(m, n, int(vals.size), _ptr(rows), _ptr(cols), _ptr(vals), _ptr(b), _ptr(c),
                           sizes, on_device=0, stream=stream)

    @classmethod
    def from_device(cls, m, n, o, rows_ptr, cols_ptr, vals_ptr, b_ptr, c_ptr, block_sizes,
                    stream: int | None = None) -> "DevicePlan":
        """Inputs already resident in HBM (int64 rows/cols, f64 vals/b/c device pointers)."""
        sizes = _as(block_sizes, np.int64)
        return cls._create(int(m), int(n), int(o), c_void_p(rows_ptr), c_void_p(cols_ptr), c_void_p(vals_ptr),
                           c_void_p(b_ptr), c_void_p(c_ptr), sizes, on_device=1, stream=stream)

    @classmethod
    def _create(cls, m, n, o, rows, cols, vals, b, c, sizes, on_device, stream):
        """stream: None = the plan creates its own stream; an int = that cudaStream_t. torch's
        default stream has handle 0, which the C ABI reads as "create one", so 0 is passed as
        cudaStreamLegacy (1): the plan's kernels are then ordered with torch's work on it."""
        h = c_void_p()
        chk = CfChecks()
        handle = None if stream is None else (CUDA_STREAM_LEGACY if int(stream) == 0 else int(stream))
        rc = lib().cf_plan_create(m, n, o, rows, cols, vals, b, c, int(sizes.size), _ptr(sizes), on_device,
                                  c_void_p(handle), byref(chk), byref(h))
        if rc == _lib.CF_EPROBLEM:
            raise ProblemRejected(chk, _lib.last_error())
        check(rc, "cf_plan_create")
        return cls(h, m, n, o)

    # ------------------------------------------------------------------ lifetime
    def close(self):
        if self._h:
            lib().cf_plan_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> c_void_p:
        if not self._h:
            raise ValueError("plan is closed")
        return self._h

    def info(self) -> dict:
        vals = [c_int64() for _ in range(6)]
        au = c_int32()
        check(lib().cf_plan_info(self.handle, *[byref(v) for v in vals], byref(au)))
        keys = ("m", "n", "o", "row_tiles", "col_tiles", "big_cones")
        d = {k: int(v.value) for k, v in zip(keys, vals)}
        d["all_unit"] = bool(au.value)
        return d

    # ------------------------------------------------------------------ state
    def set_export(self, keep: bool = True):
        """Keep b - r each iteration so get_state() can rebuild y (parity probing)."""
        check(lib().cf_plan_set_export(self.handle, 1 if keep else 0))

    def set_state(self, mu: float, state=None, export: bool = True):
        """Warm start from a SolverState-like object (None = cold start).

        export=True also keeps b - r so get_state() can return y after iterating."""
        self.set_export(export)
        if state is None:
            check(lib().cf_plan_set_state(self.handle, float(mu), None, None, None, None, None, None))
            return
        x, z, dl = (_as(getattr(state, k), np.float64) for k in ("x", "z", "delta"))
        y, g = (_as(getattr(state, k), np.float64) for k in ("y", "gamma"))
        lam = _as(state.lam, np.float64)
        for name, arr, ln in (("x", x, self.n), ("z", z, self.n), ("delta", dl, self.n), ("lam", lam, self.m),
                              ("y", y, self.o), ("gamma", g, self.o)):
            if arr.shape != (ln,):
                raise ValueError(f"init.{name}: expected shape ({ln},), got {arr.shape}")
        keep = (x, y, z, lam, g, dl)  # alive until the call returns
        check(lib().cf_plan_set_state(self.handle, float(mu), *[c_void_p(a.ctypes.data) for a in keep]))

    def get_state(self, want_yg: bool = True) -> dict:
        out = {
            "x": np.empty(self.n), "z": np.empty(self.n), "delta": np.empty(self.n), "lam": np.empty(self.m),
            "y": np.empty(self.o) if want_yg else None, "gamma": np.empty(self.o) if want_yg else None,
        }
        it = c_int64()

        def p(a):
            return c_void_p(a.ctypes.data) if a is not None and a.size else None

        check(lib().cf_plan_get_state(self.handle, p(out["x"]), p(out["y"]), p(out["z"]), p(out["lam"]),
                                      p(out["gamma"]), p(out["delta"]), byref(it)))
        out["iter"] = int(it.value)
        return out

    # ------------------------------------------------------------------ loop
    def iterate(self, mu: float, n_iters: int = 1):
        check(lib().cf_plan_iterate(self.handle, float(mu), int(n_iters)))

    def report(self, mu: float = 1.0) -> dict:
        r = CfReport()
        check(lib().cf_plan_report(self.handle, float(mu), byref(r)))
        return report_to_dict(r)

    def run(self, cfg: CfConfig, want_x: bool = True):
        """The solve() loop; returns (x, lam, list of report dicts)."""
        # a bounded first buffer; a longer trace is fetched afterwards (the plan keeps every
        # report), so max_iters=10**9 costs nothing until the reports exist
        n_chunks = -(-int(cfg.max_iters) // int(cfg.check_every))
        cap = max(1, min(n_chunks, 4096))
        trace = (CfReport * cap)()
        nrep = c_int64()
        x = np.empty(self.n) if want_x else None
        lam = np.empty(self.m) if want_x else None
        check(lib().cf_plan_solve(self.handle, byref(cfg), _ptr(x) if want_x else None,
                                  _ptr(lam) if want_x else None, trace, cap, byref(nrep)),
              "cf_plan_solve")
        out = [report_to_dict(trace[i]) for i in range(min(cap, nrep.value))]
        if nrep.value > cap:
            rest = (CfReport * (nrep.value - cap))()
            check(lib().cf_plan_trace(self.handle, cap, nrep.value - cap, rest), "cf_plan_trace")
            out.extend(report_to_dict(r) for r in rest)
        return x, lam, out

    def last_timing(self) -> dict:
        ms, rms, cms = c_double(), c_double(), c_double()
        nl, it = c_int64(), c_int64()
        check(lib().cf_plan_last_timing(self.handle, byref(ms), byref(nl), byref(rms), byref(cms), byref(it)))
        return {"loop_ms": ms.value, "launches": nl.value, "row_pass_ms": rms.value, "col_pass_ms": cms.value,
                "iters": it.value}

    def set_profiling(self, enable, stride: int = 1):
        """Per-pass CUDA events on every ``stride``-th iteration of the next loops (off: False)."""
        check(lib().cf_plan_set_profiling(self.handle, max(1, int(stride)) if enable else 0))

    # ------------------------------------------------------------------ operators (device pointers)
    def apply_A(self, x_ptr: int, y_ptr: int):
        check(lib().cf_apply_A(self.handle, c_void_p(x_ptr), c_void_p(y_ptr)))

    def apply_At(self, y_ptr: int, x_ptr: int):
        check(lib().cf_apply_At(self.handle, c_void_p(y_ptr), c_void_p(x_ptr)))

    def project(self, w_ptr: int, out_ptr: int):
        check(lib().cf_project(self.handle, c_void_p(w_ptr), c_void_p(out_ptr)))

    def set_rhs(self, b_ptr=None, c_ptr=None, on_device: bool = True):
        check(lib().cf_plan_set_rhs(self.handle, c_void_p(b_ptr) if b_ptr else None,
                                    c_void_p(c_ptr) if c_ptr else None, 1 if on_device else 0))

    def sync(self):
        check(lib().cf_plan_sync(self.handle))


def config_struct(cfg, b_norms, c_norms) -> CfConfig:
    """SolverConfig -> cf_config with the norm-dependent bounds of solver.py:252-271."""
    s = CfConfig()
    s.mu = float(cfg.mu)
    s.max_iters = int(cfg.max_iters)
    s.check_every = int(cfg.check_every)
    s.term_mode = _lib.TERM_MODES.index(cfg.term_mode)
    s.eps_abs = float(cfg.eps_abs)
    s.eps_rel = float(cfg.eps_rel)
    s.b_inf = b_norms[0]
    s.c_inf = c_norms[0]
    s.scs_prim_bound = cfg.eps_prim * (1.0 + b_norms[1])
    s.scs_dual_bound = cfg.eps_dual * (1.0 + c_norms[1])
    s.eps_gap = float(cfg.eps_gap)
    s.target_prim_res = float(cfg.target_prim_res) if cfg.target_prim_res is not None else float("nan")
    s.target_gap = float(cfg.target_gap) if cfg.target_gap is not None else float("nan")
    return s


_ = ctypes  # keep the module import explicit for readers of the signatures
