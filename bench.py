#!/usr/bin/env python
"""Benchmark of the B200 iteration engine on BASELINE.json's headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c3m|c1|c4|c5] [--impl ours|reference]

A *step* is one ADMM iteration (solver.py:313-317) of the C2 LP (m=5M, n=10M,
o=100M, fp64) with the solve loop's report cadence (check_every=25, solver.py:319)
included, inputs resident in HBM. ``value`` = iterations/s over exactly K timed
iterations (CUDA events on the plan's stream, barrier + synchronize on both sides,
max over ranks), measured after a >= 2 s warm-up so the GPU sits at its sustained
(power-capped) clock rather than a cold-start burst.

Instances: C2 and C3 come from cfgen, a counter-based generator whose numpy and CUDA
halves return bit-identical arrays (tests/test_gpu_gen.py). The GPU arm builds them on
the device; the CPU reference arm builds the SAME arrays with numpy (it never loads
libcfb200); both lines carry ``config.instance_fingerprint``. C1 is the reference's
own instance (GenSpec(1000, 2000, 0.01, "lp", seed=0), PCG64, bit-identical).

Also on the GPU line:
  time_to_tol  full solve() to scs eps=1e-4 from a cold start, device-resident inputs
  e2e          the same metric through the public API solve(p, cfg) from HOST numpy
               buffers (N>1: solve_distributed) — iterations / wall seconds
  roofline     dominant kernel (per-pass CUDA events inside the timed region):
               algorithmic bytes (SURVEY §8d split per pass) / average duration
  cpu_baseline the reference's step functions (baseline/_ref conefree, else the oracle
               port) on the same arrays, 1 core of os.cpu_count() (rank 0, N=1)
  clocks       nvidia-smi sampled during the timed region
  gather_bound the dominant pass against the measured random-gather ceiling

N>1 (torchrun): the SAME C2 instance strong-scaled over the ranks through the sharded
engine (sharded.choose_sharding picks columns for m < n: NCCL reduce-scatter of A x,
each rank updates its block of rows, all-gather of h), ``scaling: "strong"``; the full-scale 1e9-nonzero C5 row/column-
sharded number rides along as ``c5``.

--impl reference: the unmodified reference (baseline/_ref/conefree: validate,
build_uv, then its x/y/z/dual step functions) on the same arrays, timed on the host
cores by rank 0; other ranks exit 0. C2/C3: setup + min(K, 3) full-size iterations
from the cold start (no warm-up: numpy has nothing to warm); C1: the full solve() to 1e-4; C4: the reference's run_bench over a
process pool on every host core.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp64 solver iterations/sec and time-to-1e-4 residual; HBM GB/s vs roofline"
UNIT = "iterations/s"
REF_PATH = os.path.join(ROOT, "baseline", "_ref")

CONFIGS = {
    "c2": dict(m=5_000_000, n=10_000_000, density=2e-6, cone_kind="lp", gen="cfgen",
               workload="C2: synthetic sparse LP m=5,000,000 n=10,000,000 o=100,000,000 (20 nnz/row) fp64"),
    "c3": dict(m=2_000_000, n=4_000_000, density=5e-6, cone_kind="socp4", gen="cfgen",
               workload="C3: synthetic SOCP m=2,000,000 n=4,000,000 o=40,000,000, 1,000,000 K4 cones fp64"),
    "c3m": dict(m=3_000_000, n=5_000_000, density=2.6e-6, cone_kind="rls", gen="rls",
                workload="C3 secondary (SURVEY §8d): robust least squares in SOC form, 1,000,000 K4 blocks "
                         "(t_i, u_i) + x+/x- in R+^1,000,000; m=3,000,000 n=5,000,000 o=39,000,000 fp64"),
    "c1": dict(m=1000, n=2000, density=0.01, cone_kind="lp", gen="reference",
               workload="C1: the reference's instance GenSpec(1000, 2000, 0.01, 'lp', seed=0), o=20,000 fp64"),
    "c5": dict(m=50_000_000, n=100_000_000, density=2e-7, cone_kind="lp", sharded=True,
               workload="C5: row-sharded synthetic sparse LP m=50,000,000 n=100,000,000 o=1,000,000,000 fp64"),
    "c4": dict(m=100, n=200, density=0.05, cone_kind="lp", batch=4096,
               workload="C4: batch of 4096 independent sparse LPs m=100 n=200 o=1,000 (5%) fp64, seeds 0..4095"),
}
DATA_LABEL = {
    "cfgen": "synthetic: cfgen counter-based generator (reference recipe generate.py:103-140, own random stream); "
             "numpy and CUDA halves produce bit-identical arrays, so the GPU arm (device) and the reference arm "
             "(host numpy) run the same instance (config.instance_fingerprint)",
    "reference": "synthetic: the reference's own generator and seed (PCG64, generate.py:103-140), bit-identical",
    "rls": "synthetic (GPU generator devgen.rls_arrays: N(0,1) F with 6 distinct columns per row, g ~ N(0,1))",
}
WARM_SECONDS = 2.0      # GPU arm: warm-up long enough to reach the sustained (power-capped) clock
REF_MAX_STEPS = 3       # reference arm: full-size C2/C3 iterations timed


def algorithmic_bytes(m, n, o):
    """B_alg = 24o + 44m + 68n per iteration, split per pass."""
    row = 12 * o + 4 * m + 8 * n + 32 * m      # CSR val+idx, rowptr, x gather, b/lam read + lam/h write
    col = 12 * o + 4 * n + 8 * m + 56 * n      # CSC val+idx, colptr, h gather, x/z/delta/c read + x/z/delta write
    return row, col


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# Random fp64 gathers from an L2-resident vector retire at ~1.03 per SM-cycle
# (one L1TEX->L2 request each; profiles/r01_probes.md, scratch/gather_probe2.cu).
# Every pass does one gather per nonzero, so this — not HBM — bounds a pass.
GATHERS_PER_SM_CYCLE = 1.03
N_SMS = 148


def gather_bound(o, pass_ms, clocks):
    """The dominant pass against the gather-request ceiling at the sampled SM clock."""
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = GATHERS_PER_SM_CYCLE * N_SMS * mhz * 1e6 / 1e9
    achieved = o / (pass_ms / 1000.0) / 1e9
    return {"achieved": achieved, "peak": peak, "unit": "Ggathers/s", "frac": achieved / peak,
            "sm_mhz": mhz, "source": "probe: 1.03 random fp64 gathers per SM-cycle (profiles/r01_probes.md)"}


# The ideal C2 iteration (scratch/ideal_iter_probe.cu, profiles/r02_probes.md): uniform
# 10-nonzero segments in ELL layout, every load a full aligned line, the same bytes and
# gathers as C2 — 0.888 ms per iteration sustained (0.567 of the measured HBM peak) with
# the request port 88 % busy. No implementation of C2's access pattern beats it on this
# power-capped part, so it is the practical ceiling the line is compared with.
PROF_STRIDE = 10        # per-pass CUDA events on every 10th timed iteration (see run_ours)
IDEAL_C2_MS = 0.888
IDEAL_C2_MHZ = 1965.0   # its sustained SM clock (below the 1 kW cap: 860-910 W)


def native_so_loaded():
    """Shared objects of this repo mapped into the process (the reference arm must show none)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if line.strip() else ""
                if path.endswith(".so") and path.startswith(ROOT) and "/baseline/" not in path:
                    out.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(out)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled in the background."""

    FIELDS = ("timestamp", "clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "power.draw")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.windows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for t, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            rows.append((t, parts))
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        inside = [r for r in rows if any(a - 0.15 <= r[0] <= b + 0.15 for a, b in self.windows)] or rows
        sm = [float(p[1]) for _, p in inside if p[1].replace(".", "").isdigit()]
        mx = [float(p[2]) for _, p in inside if p[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({nm for _, p in inside for nm, v in zip(names, p[3:7]) if v.lower() == "active"})
        pw = [float(p[7]) for _, p in inside if p[7].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------------------ instances
def o_of(spec):
    return int(round(spec["m"] * spec["n"] * spec["density"]))


def host_arrays(spec, seed):
    """The instance on the host, numpy only (never loads libcfb200): dict of canonical arrays."""
    import numpy as np

    if spec["gen"] == "reference":
        ref = load_reference()
        if ref is not None:
            from conefree.generate import GenSpec as RGenSpec
            from conefree.generate import generate as rgenerate

            p = rgenerate(RGenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=seed))
        else:
            from paper_2203_05027_b200.instances import GenSpec, generate

            p = generate(GenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=seed))
        return dict(m=spec["m"], n=spec["n"], rows=np.asarray(p.A.rows), cols=np.asarray(p.A.cols),
                    vals=np.asarray(p.A.vals), b=np.asarray(p.b), c=np.asarray(p.c),
                    sizes=np.asarray(p.cones.block_sizes, dtype=np.int64))
    if spec["gen"] != "cfgen":
        raise SystemExit(f"config {spec['workload']!r} has no host generator")
    from paper_2203_05027_b200 import cfgen

    h = cfgen.generate_host(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed)
    return dict(m=h.m, n=h.n, rows=h.rows, cols=h.cols, vals=h.vals, b=h.b, c=h.c, sizes=h.block_sizes)


def device_instance(spec, seed, stream):
    """(DeviceInstance with its plan, generator description)."""
    import torch

    if spec["gen"] == "cfgen":
        from paper_2203_05027_b200 import cfgen

        return cfgen.generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed, stream=stream)
    if spec["gen"] == "rls":
        from paper_2203_05027_b200.devgen import generate_device

        return generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=seed, stream=stream)
    from paper_2203_05027_b200.devgen import DeviceInstance
    from paper_2203_05027_b200.engine import DevicePlan
    from paper_2203_05027_b200.instances import GenSpec, generate

    p = generate(GenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=seed))
    t = {k: torch.as_tensor(v).cuda() for k, v in (("rows", p.A.rows), ("cols", p.A.cols), ("vals", p.A.vals),
                                                   ("b", p.b), ("c", p.c))}
    sizes = p.cones.sizes_array()
    torch.cuda.synchronize()
    plan = DevicePlan.from_device(p.m, p.n, int(p.A.nnz), t["rows"].data_ptr(), t["cols"].data_ptr(),
                                  t["vals"].data_ptr(), t["b"].data_ptr(), t["c"].data_ptr(), sizes, stream=stream)
    return DeviceInstance(p.m, p.n, int(p.A.nnz), spec["cone_kind"], t["rows"], t["cols"], t["vals"], t["b"], t["c"],
                          sizes, plan)


def fingerprint(a):
    from paper_2203_05027_b200 import cfgen

    return cfgen.fingerprint(a["rows"], a["cols"], a["vals"], a["b"], a["c"])


# ------------------------------------------------------------------------------ the reference on the CPU
def load_reference():
    """The unmodified reference installed in baseline/_ref (pip --target), or None."""
    if os.path.isdir(os.path.join(REF_PATH, "conefree")) and REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    try:
        import conefree  # noqa: F401

        return conefree
    except ImportError:
        return None


def _ref_problem(a):
    from conefree.model import ConeSpec, ProblemInstance, TripletMatrix

    return ProblemInstance(TripletMatrix(a["m"], a["n"], a["rows"], a["cols"], a["vals"]), a["b"], a["c"],
                           ConeSpec(tuple(int(s) for s in a["sizes"])))


def reference_iterations(a, warmup, steps, full_setup, budget_s=1e9):
    """Time the reference's iteration (solver.py:313-317: its own x/y/z/dual_update) on the arrays ``a``.

    full_setup: time solve()'s setup first (validate + build_uv + ConeWorkview,
    solver.py:300-307); else assemble UVFactors from the (already canonical) arrays with
    build_uv's formulas (uv.py:76-98, the unused index groups left empty) — a bounded
    sample. Falls back to the oracle port when baseline/_ref is absent.
    Returns dict(s_per_iter, iters, setup_s, kind, what)."""
    import numpy as np

    ref = load_reference()
    setup_s = None
    times = []
    if ref is not None:
        from conefree.cones import ConeWorkview
        from conefree.model import validate
        from conefree.solver import SolverConfig, SolverState, dual_update, x_update, y_update, z_update
        from conefree.uv import UVFactors, build_uv

        p = _ref_problem(a)
        t0 = time.perf_counter()
        if full_setup:
            rep = validate(p)
            if not rep.ok:
                raise RuntimeError("reference validate rejected the instance: " + "; ".join(rep.violations[:3]))
            f = build_uv(p.A)
            view = ConeWorkview.from_spec(p.cones)
            setup_s = time.perf_counter() - t0
        else:
            r, c, v = a["rows"], a["cols"], a["vals"]
            f = UVFactors(m=a["m"], n=a["n"], o=int(v.size), row_of=r, col_of=c, val=v,
                          fu_diag=1.0 / (1.0 + np.bincount(r, weights=v * v, minlength=a["m"])),
                          fv_diag=1.0 / (1.0 + np.bincount(c, minlength=a["n"])), row_groups=(), col_groups=())
            view = ConeWorkview.from_spec(p.cones)
        cfg = SolverConfig()
        st = SolverState.zeros(f)

        def step():
            st.x = x_update(f, st, cfg, p.c)
            st.y = y_update(f, st, cfg, p.b)
            st.z = z_update(view, st, cfg)
            st.lam, st.gamma, st.delta = dual_update(f, st, cfg, p.b)

        kind, what = "reference", "baseline/_ref conefree (unmodified reference) x/y/z/dual_update, solver.py:313-317"
    else:
        import oracle

        p = None
        t0 = time.perf_counter()
        f = oracle.build_factors(type("A", (), dict(num_rows=a["m"], num_cols=a["n"], rows=a["rows"],
                                                    cols=a["cols"], vals=a["vals"]))())
        if full_setup:
            setup_s = time.perf_counter() - t0
        box = {"st": oracle.OracleState.zeros(f)}

        def step():
            box["st"] = oracle.step(f, a["sizes"], box["st"], 1.0, a["b"], a["c"])

        kind, what = "port", "oracle port (literal numpy restatement of solver.py:168-197; baseline/_ref absent)"
    for _ in range(warmup):
        step()
    t_start = time.perf_counter()
    for _ in range(steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s:
            break
    return dict(s_per_iter=sum(times) / len(times), iters=len(times), setup_s=setup_s, kind=kind, what=what)


def reference_solve(a, eps):
    """The reference's full solve() to eps (small configs): (iterations, seconds, report, kind)."""
    ref = load_reference()
    if ref is not None:
        from conefree.solver import SolverConfig, solve

        p = _ref_problem(a)
        t0 = time.perf_counter()
        res = solve(p, SolverConfig(eps_prim=eps, eps_dual=eps, eps_gap=eps))
        secs = time.perf_counter() - t0
        return res.report.iter, secs, res.report, "reference"
    import oracle
    from paper_2203_05027_b200 import ConeSpec, ProblemInstance, SolverConfig, TripletMatrix

    p = ProblemInstance(TripletMatrix(a["m"], a["n"], a["rows"], a["cols"], a["vals"]), a["b"], a["c"],
                        ConeSpec(a["sizes"]))
    t0 = time.perf_counter()
    _, _, tr, _ = oracle.solve(p, SolverConfig(eps_prim=eps, eps_dual=eps, eps_gap=eps))
    secs = time.perf_counter() - t0
    rep = type("R", (), tr[-1])()
    return tr[-1]["iter"], secs, rep, "port"


def reference_batch_baseline(args, spec):
    """C4 CPU baseline: the reference's own run_bench (bench.py:96-106, a process pool over
    solve()) on every host core, over a bounded prefix of the batch (the oracle port in the
    same scheme without baseline/_ref). Returns a cpu_baseline dict in problem-iterations/s."""
    workers = os.cpu_count() or 1
    P = min(spec["batch"], 16 * workers)
    cfg_kw = dict(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps)
    ref = load_reference()
    if ref is not None:
        from conefree.bench import BenchJob, run_bench
        from conefree.generate import GenSpec
        from conefree.solver import SolverConfig

        jobs = [BenchJob(s, GenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=s),
                         SolverConfig(**cfg_kw)) for s in range(P)]
        t0 = time.perf_counter()
        rows = run_bench(jobs, workers=workers)
        wall = time.perf_counter() - t0
        its = sum(r["iters"] for r in rows)
        cpu = {"value": its / wall, "unit": "problem-iterations/s", "cores": workers, "host_cores": workers,
               "kind": "reference",
               "sample": f"the reference's run_bench (baseline/_ref conefree, {workers}-process pool) on problems "
                         f"0..{P - 1} of the batch to eps={args.eps}: {its} iterations in {wall:.1f} s wall "
                         "(includes its per-job generate, as the reference's bench does)"}
    else:
        from paper_2203_05027_b200 import GenSpec, SolverConfig, generate

        probs = [generate(GenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=s)) for s in range(P)]
        cpu = cpu_batch_pool(probs, SolverConfig(**cfg_kw), args.eps, args.cpu_budget)
    return cpu


def run_reference_batch(args, spec):
    """C4 reference arm: reference_batch_baseline on every host core."""
    workers = os.cpu_count() or 1
    cpu = reference_batch_baseline(args, spec)
    value = cpu["value"]
    line = {
        "metric": METRIC, "value": value, "unit": "problem-iterations/s", "n_gpus": args.gpus, "steps": 1,
        "warmup": 0, "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": DATA_LABEL["reference"] + " (seeds 0..4095)",
        "impl": "reference",
        "config": {"workload": spec["workload"], "problems": spec["batch"], "parallelism": f"{workers}-process pool"},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "problem-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_so_loaded": native_so_loaded(),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args, spec, rank):
    """--impl reference: the reference on the host cores, same instance as the GPU arm."""
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if "batch" in spec:
        return run_reference_batch(args, spec)
    if spec.get("sharded"):
        print(json.dumps({"impl": "reference", "unavailable": "C5 (1e9 nonzeros) exceeds the reference's host "
                          "memory (~160 GB RSS, SURVEY §8d); no CPU arm"}), flush=True)
        return 0
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    a = host_arrays(spec, args.seed)
    gen_s = time.perf_counter() - t0
    fp = fingerprint(a)
    o = int(a["vals"].size)
    config = {"workload": spec["workload"], "m": a["m"], "n": a["n"], "o": o, "mu": 1.0, "check_every": 25,
              "parallelism": "single process (the reference is single-threaded numpy)",
              "instance_fingerprint": fp}
    if o < 1_000_000:
        # small configs: the full solve() to eps, as BASELINE.md §3 prescribes for C1
        iters, secs, rep, kind = reference_solve(a, args.eps)
        value = iters / secs
        steps = iters
        sample = (f"{'the unmodified reference (baseline/_ref conefree.solve)' if kind == 'reference' else 'the oracle port'}"
                  f": full solve to scs eps={args.eps} from a cold start, {iters} iterations in {secs:.3f} s "
                  f"(1 core of {cores})")
        extra = {"time_to_tol": {"seconds": secs, "iters": int(iters), "status": rep.status, "eps": args.eps,
                                 "pobj": float(rep.pobj)}}
    else:
        steps = max(1, min(args.steps, REF_MAX_STEPS))
        r = reference_iterations(a, 0, steps, full_setup=True)
        kind = r["kind"]
        value = 1.0 / r["s_per_iter"]
        steps = r["iters"]
        sample = (f"{r['what']}: solve()'s setup (validate + build_uv + ConeWorkview, solver.py:300-307) "
                  f"{r['setup_s']:.1f} s, then {steps} timed full-size iterations from the cold start, "
                  f"{r['s_per_iter']:.3f} s/iteration (1 core of {cores}; requested --steps {args.steps} capped "
                  f"at {REF_MAX_STEPS})")
        extra = {"setup_s": r["setup_s"], "s_per_iteration": r["s_per_iter"]}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": 0, "ms_per_step": 1000.0 / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA_LABEL[spec["gen"]],
        "impl": "reference", "config": config,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "host_cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "instance_build_s": gen_s,
        "native_so_loaded": native_so_loaded(),
        **extra,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ our arm, one GPU
def run_ours(args, spec, rank, world, local_rank):
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.api import norms, solve
    from paper_2203_05027_b200.devgen import to_host_problem
    from paper_2203_05027_b200.engine import config_struct

    torch.cuda.set_device(local_rank)
    stream = torch.cuda.current_stream()
    inst = device_instance(spec, args.seed, stream.cuda_stream)
    plan = inst.plan
    m, n, o = inst.m, inst.n, inst.o
    fp = fingerprint(dict(rows=inst.rows, cols=inst.cols, vals=inst.vals, b=inst.b, c=inst.c))
    b_host, c_host = inst.b.cpu().numpy(), inst.c.cpu().numpy()
    bn, cn = norms(b_host), norms(c_host)

    def never(k):
        return config_struct(SolverConfig(max_iters=k, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0),
                             bn, cn)

    # ---------------- warm-up: W iterations, then enough more for >= WARM_SECONDS of load
    plan.set_state(1.0, None, export=False)
    plan.run(never(args.warmup), want_x=False)
    per_it = plan.last_timing()["loop_ms"] / 1000.0 / args.warmup
    warm_more = int(min(200_000, max(0, args.warm_seconds / max(per_it, 1e-7))))
    if warm_more:
        plan.run(never(warm_more), want_x=False)
    # ---------------- timed iterations (device-resident inputs), from a cold start
    plan.set_state(1.0, None, export=False)
    sampler = ClockSampler(local_rank).start() if rank == 0 else None
    time.sleep(0.4 if sampler else 0.0)
    if warm_more:   # the sampler start cost the GPU its load: re-warm briefly
        plan.run(never(max(1, warm_more // 4)), want_x=False)
        plan.set_state(1.0, None, export=False)
    # per-pass CUDA events inside the timed region break the passes' programmatic-launch
    # overlap (~11 us per bracketed iteration at C2, 1 %): they bracket every PROF_STRIDE-th
    # iteration of the timed loop and the pass times are the sampled launches' average.
    # Small problems (where even that matters) time their split in a separate run.
    profile_in_timed = o >= 1_000_000 and not os.environ.get("CF_BENCH_NO_EVENTS")
    plan.set_profiling(profile_in_timed, stride=PROF_STRIDE)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(stream)
    _, _, trace = plan.run(never(args.steps), want_x=False)
    e1.record(stream)
    torch.cuda.synchronize()
    w1 = time.time()
    plan.set_profiling(False)
    if sampler:
        sampler.mark(w0, w1)
    ms = e0.elapsed_time(e1)
    tim = plan.last_timing()
    assert tim["iters"] == args.steps and trace[-1]["status"] == "max_iters", (tim, trace[-1])
    pass_tim = tim
    if not profile_in_timed:
        plan.set_state(1.0, None, export=False)
        plan.set_profiling(True)
        plan.run(never(args.steps), want_x=False)
        plan.set_profiling(False)
        pass_tim = plan.last_timing()
    ms_max = ms
    value = args.steps / (ms_max / 1000.0)

    # ---------------- small problems: solve() runs them in the cluster-resident kernel
    # (k_cluster, one launch for the whole loop); its device time is the headline then
    engine = {"name": "plan (k_pass chain)"}
    hp = None
    if o < 1_000_000:
        from paper_2203_05027_b200 import api as _api

        hp = to_host_problem(inst)
        if _api._cluster_candidate(hp):
            zero = SolverConfig(max_iters=args.steps, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
            _api._solve_cluster(hp, SolverConfig(max_iters=args.warmup, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0))
            ct = {}
            cres = _api._solve_cluster(hp, zero, timing=ct)
            if cres is not None and cres.report.iter == args.steps:
                engine = {"name": f"cluster (k_cluster, {ct['cluster']} CTAs, distributed shared memory)",
                          "ms_per_step": ct["kernel_ms"] / args.steps,
                          "plan_engine": {"value": value, "ms_per_step": ms_max / args.steps}}
                ms_max = ct["kernel_ms"]
                value = args.steps / (ms_max / 1000.0)

    # ---------------- roofline of the dominant pass (per-pass events inside the timed region)
    row_b, col_b = algorithmic_bytes(m, n, o)
    peak, peak_src = hbm_peak()
    row_ms = pass_tim["row_pass_ms"] / args.steps
    col_ms = pass_tim["col_pass_ms"] / args.steps
    passes = {"row_pass": (row_b, row_ms), "col_pass": (col_b, col_ms)}
    dom = max(passes, key=lambda k: passes[k][1])
    dbytes, dms = passes[dom]
    achieved = dbytes / (dms / 1000.0) / 1e9
    per_iter_ms = ms / args.steps
    it_achieved = (row_b + col_b) / (per_iter_ms / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"ncu_traffic_{args.config}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": f"k_{dom}", "bytes_per_launch": dbytes, "avg_launch_ms": dms,
                "peak_source": peak_src,
                # both passes (the two take nearly the same time, so "dominant" flips between runs)
                "passes": {k: {"bytes_per_launch": b_, "avg_launch_ms": t_,
                               "frac": (b_ / (t_ / 1000.0) / 1e9) / peak if t_ > 0 else None}
                           for k, (b_, t_) in passes.items()}}
    iteration_roofline = {"achieved": it_achieved, "frac": it_achieved / peak, "bytes_per_iteration": row_b + col_b,
                          "ms_per_iteration": per_iter_ms, "row_pass_ms": row_ms, "col_pass_ms": col_ms,
                          "report_and_launch_ms": (per_iter_ms - row_ms - col_ms) if profile_in_timed else None,
                          "pass_times": (f"timed region, CUDA events around the passes of every {PROF_STRIDE}th iteration"
                                         if profile_in_timed else "separate profiled run")}

    # ---------------- time to tolerance (device-resident, cold start)
    ttt = None
    if not args.skip_ttt:
        tol = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps)
        plan.set_state(1.0, None, export=False)
        torch.cuda.synchronize()
        w0 = time.time()
        _, _, ttrace = plan.run(config_struct(tol, bn, cn), want_x=False)
        w1 = time.time()
        if sampler:
            sampler.mark(w0, w1)
        tt = plan.last_timing()
        ttt = {"seconds": tt["loop_ms"] / 1000.0, "iters": int(ttrace[-1]["iter"]), "status": ttrace[-1]["status"],
               "eps": args.eps, "term_mode": "scs", "pobj": ttrace[-1]["pobj"],
               "prim_res_2": ttrace[-1]["prim_res_2"], "stat_res_2": ttrace[-1]["stat_res_2"],
               "gap": ttrace[-1]["gap"], "iterations_per_s": int(ttrace[-1]["iter"]) / (tt["loop_ms"] / 1000.0)}
    if ttt is not None and engine["name"].startswith("cluster"):
        from paper_2203_05027_b200 import api as _api

        ct = {}
        cres = _api._solve_cluster(hp, SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps),
                                   timing=ct)
        engine["plan_engine"]["time_to_tol"] = ttt
        ttt = {"seconds": ct["kernel_ms"] / 1000.0, "iters": cres.report.iter, "status": cres.report.status,
               "eps": args.eps, "term_mode": "scs", "pobj": cres.report.pobj,
               "prim_res_2": cres.report.prim_res_2, "stat_res_2": cres.report.stat_res_2, "gap": cres.report.gap}
    if sampler:
        sampler.stop()
    plan.close()

    # ---------------- e2e through the public API from host buffers
    p = to_host_problem(inst) if hp is None else hp
    arrays = dict(m=m, n=n, rows=p.A.rows, cols=p.A.cols, vals=p.A.vals, b=p.b, c=p.c,
                  sizes=p.cones.sizes_array())
    del inst
    torch.cuda.empty_cache()
    e2e = None
    if not args.skip_e2e:
        tol = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps,
                           max_iters=args.e2e_max_iters or 100_000)
        # one untimed warm-up step: first-use costs of a fresh process (lazy kernel-module loading,
        # first mapping of the memory pool) are not per-solve costs
        solve(p, SolverConfig(max_iters=25))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solve(p, tol)
        secs = time.perf_counter() - t0
        e2e = {"value": res.report.iter / secs, "unit": UNIT,
               "h2d_bytes_per_step": 24 * o + 8 * m + 8 * n, "d2h_bytes_per_step": 8 * (m + n),
               "seconds": secs, "iters": res.report.iter, "status": res.report.status,
               "step": "one solve(p, SolverConfig(eps=%g)) from host numpy buffers" % args.eps}
        if ttt is not None and res.report.iter != ttt["iters"]:
            e2e["note"] = "iteration count differs from the device-resident run"

    # ---------------- CPU baseline: the reference's iteration on the same arrays (rank 0, N=1)
    cpu = None
    if rank == 0 and not args.skip_cpu:
        cores = os.cpu_count() or 1
        if o < 1_000_000:
            iters, secs, rep, kind = reference_solve(arrays, args.eps)
            cpu = {"value": iters / secs, "unit": UNIT, "cores": 1, "host_cores": cores, "kind": kind,
                   "sample": f"full solve to eps={args.eps} on the same instance: {iters} iterations in "
                             f"{secs:.3f} s (1 core of {cores})"}
        else:
            r = reference_iterations(arrays, 0, 2, full_setup=False, budget_s=args.cpu_budget)
            cpu = {"value": 1.0 / r["s_per_iter"], "unit": UNIT, "cores": 1, "host_cores": cores, "kind": r["kind"],
                   "sample": f"{r['what']} on the same arrays (fingerprint {fp}): {r['iters']} "
                             f"full-size iterations from the cold start, {r['s_per_iter']:.3f} s/iteration (1 core of {cores}); "
                             "UVFactors assembled from the canonical arrays with build_uv's formulas "
                             "(the reference's own setup is timed by --impl reference)"}
            if ttt is not None:
                cpu["extrapolated_time_to_tol_s"] = ttt["iters"] * r["s_per_iter"]

    clocks = sampler.summary() if sampler else None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "warmup_extra_iterations": warm_more, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA_LABEL[spec["gen"]],
        "config": {"workload": spec["workload"], "m": m, "n": n, "o": o, "mu": 1.0, "check_every": 25,
                   "parallelism": "single", "instance_fingerprint": fp,
                   "l2": "inputs larger than L2 " f"({(row_b + col_b) / 1e9:.2f} GB streamed per iteration vs 126 MB L2)"
                   if row_b + col_b > 126e6 else "inputs L2-resident (small config; latency-bound)"},
        "gpu_launches": 1 if engine["name"].startswith("cluster") else tim["launches"], "engine": engine,
        "roofline": roofline, "iteration_roofline": iteration_roofline,
        "time_to_tol": ttt, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
        "gather_bound": gather_bound(o, dms, clocks),
    }
    if args.config == "c2":
        mhz = (clocks or {}).get("sm_mhz") or IDEAL_C2_MHZ
        per_it = ms_max / args.steps
        line["ideal_bound"] = {"ideal_ms_per_iteration": IDEAL_C2_MS, "frac": IDEAL_C2_MS / per_it,
                               "ideal_mhz": IDEAL_C2_MHZ,
                               # the probe runs below the power cap at the top clock; this line's
                               # engine runs at the cap: the same comparison at this line's clock
                               "frac_at_this_clock": IDEAL_C2_MS * IDEAL_C2_MHZ / mhz / per_it,
                               "source": "scratch/ideal_iter_probe.cu: the same bytes and gathers with uniform "
                                         "segments in a perfectly coalesced ELL layout, sustained on this pool's "
                                         "B200 at 1,965 MHz and 860-910 W (profiles/r02_probes.md); 0.567 of the "
                                         "HBM peak"}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ our arm, N GPUs
def distributed_backend(inst_or_problem, mode, rank, world, group=None):
    """This rank's shard of the instance for ``mode`` (sharded.choose_sharding).

    Device instance (bench): slice the device arrays and build the rank's plan on the GPU.
    Host problem (tests): the sharded module's own slicing and the numpy test backends are
    passed through ``backend_factory`` by the caller instead (see run_strong)."""
    import numpy as np
    import torch

    from paper_2203_05027_b200.engine import DevicePlan
    from paper_2203_05027_b200.sharded import (CudaColBackend, CudaRankBackend, column_cuts,
                                               row_cuts_from_counts)

    inst = inst_or_problem
    m, n = inst.m, inst.n
    sizes = np.asarray(inst.block_sizes, dtype=np.int64)
    col_cuts = column_cuts(sizes, n, world)
    stream = torch.cuda.current_stream().cuda_stream
    if mode == "cols":
        c0, c1 = col_cuts[rank], col_cuts[rank + 1]
        sel = (inst.cols >= c0) & (inst.cols < c1)
        rows, cols, vals = inst.rows[sel].contiguous(), (inst.cols[sel] - c0).contiguous(), inst.vals[sel].contiguous()
        c_s = inst.c[c0:c1].contiguous()
        starts = np.concatenate(([0], np.cumsum(sizes)))
        q0, q1 = int(np.searchsorted(starts, c0)), int(np.searchsorted(starts, c1))
        torch.cuda.synchronize()
        plan = DevicePlan.from_device(m, c1 - c0, int(vals.numel()), rows.data_ptr(), cols.data_ptr(),
                                      vals.data_ptr(), inst.b.data_ptr(), c_s.data_ptr(), sizes[q0:q1], stream=stream)
        return CudaColBackend(None, plan=plan), None, col_cuts
    counts = torch.bincount(inst.rows, minlength=m).cpu().numpy()
    row_cuts = row_cuts_from_counts(counts, world)
    r0, r1 = row_cuts[rank], row_cuts[rank + 1]
    sel = (inst.rows >= r0) & (inst.rows < r1)
    rows, cols, vals = (inst.rows[sel] - r0).contiguous(), inst.cols[sel].contiguous(), inst.vals[sel].contiguous()
    b_l = inst.b[r0:r1].contiguous()
    torch.cuda.synchronize()
    plan = DevicePlan.from_device(r1 - r0, n, int(vals.numel()), rows.data_ptr(), cols.data_ptr(), vals.data_ptr(),
                                  b_l.data_ptr(), inst.c.data_ptr(), np.ones(n, dtype=np.int64), stream=stream)
    lo, hi = col_cuts[rank], col_cuts[rank + 1]
    starts = np.concatenate(([0], np.cumsum(sizes)))
    cone_slice = None
    if sizes.size and int(sizes.max()) > 1:
        q0, q1 = np.searchsorted(starts, lo), np.searchsorted(starts, hi)
        cone_slice = (starts[q0:q1 + 1] - lo).astype(np.int32)
    be = CudaRankBackend.from_plan(plan, lo, hi, inst.c[lo:hi].clone(), cone_slice)
    return be, row_cuts, col_cuts


def run_strong(args, spec, rank, world, local_rank, group=None, factories=None, problem=None):
    """N>1: ONE C2 instance strong-scaled over the ranks through the sharded engine.

    ``problem`` (a host ProblemInstance) and ``factories`` ({"rows": ..., "cols": ...} rank
    backends) let tests/test_bench_strong.py run this exact code on gloo with the numpy
    rank backends, sliced by the sharded module's own partition; by default every rank
    builds the instance on its GPU (cfgen, identical on every rank) and slices its shard
    there. Prints the rank-0 line."""
    import torch
    import torch.distributed as dist

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.api import norms
    from paper_2203_05027_b200.sharded import (choose_sharding, exchange_bytes, run_col_sharded, run_sharded,
                                               solve_distributed)

    on_gpu = factories is None
    if on_gpu:
        torch.cuda.set_device(local_rank)
        inst = device_instance(spec, args.seed, torch.cuda.current_stream().cuda_stream)
        inst.plan.close()
        inst.plan = None
        m, n, o = inst.m, inst.n, inst.o
        fp = fingerprint(dict(rows=inst.rows, cols=inst.cols, vals=inst.vals, b=inst.b, c=inst.c))
        bn, cn = norms(inst.b.cpu().numpy()), norms(inst.c.cpu().numpy())
    else:
        m, n, o = int(problem.A.num_rows), int(problem.A.num_cols), int(problem.A.nnz)
        fp = None
        bn, cn = norms(problem.b), norms(problem.c)
    mode = choose_sharding(m, n, world) if args.layout == "auto" else args.layout

    def backend():
        if on_gpu:
            return distributed_backend(inst, mode, rank, world, group)
        from paper_2203_05027_b200.sharded import _cone_ptr_slice, local_columns, local_problem, partition

        row_cuts, col_cuts = partition(problem, world)
        lo, hi = col_cuts[rank], col_cuts[rank + 1]
        if mode == "cols":
            return factories["cols"](local_columns(problem, lo, hi)), None, col_cuts
        lp = local_problem(problem, row_cuts[rank], row_cuts[rank + 1])
        return factories["rows"](lp, lo, hi, _cone_ptr_slice(problem, lo, hi), None), row_cuts, col_cuts

    def loop(cfg, timing):
        be, row_cuts, col_cuts = backend()
        try:
            dist.barrier(group=group)
            if on_gpu:
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            if mode == "cols":
                res = run_col_sharded(be, col_cuts, cfg, bn, cn, group=group, timing=timing, gather_result=False)
            else:
                res = run_sharded(be, row_cuts, col_cuts, cfg, bn, cn, group=group, timing=timing,
                                  gather_result=False)
            if on_gpu:
                torch.cuda.synchronize()
            timing.setdefault("loop_ms", (time.perf_counter() - t0) * 1000.0)
            return res
        finally:
            if hasattr(be, "close"):
                be.close()

    def max_over_ranks(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda" if on_gpu else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return float(t.item())

    zero = dict(check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    loop(SolverConfig(max_iters=args.warmup, **zero), {})               # warm-up (fresh state after)
    sampler = ClockSampler(local_rank).start() if (on_gpu and rank == 0) else None
    tim = {}
    w0 = time.time()
    res = loop(SolverConfig(max_iters=args.steps, **zero), tim)
    if sampler:
        sampler.mark(w0, time.time())
        sampler.stop()
    assert res.report.iter == args.steps and res.report.status == "max_iters", res.report
    ms = max_over_ranks(tim["loop_ms"])
    value = args.steps / (ms / 1000.0)
    ttt = None
    if not args.skip_ttt:
        tt = {}
        tres = loop(SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps), tt)
        secs = max_over_ranks(tt["loop_ms"]) / 1000.0
        ttt = {"seconds": secs, "iters": tres.report.iter, "status": tres.report.status, "eps": args.eps,
               "pobj": tres.report.pobj, "prim_res_2": tres.report.prim_res_2,
               "stat_res_2": tres.report.stat_res_2, "gap": tres.report.gap}
    e2e = None
    if not args.skip_e2e:
        if on_gpu:
            from paper_2203_05027_b200.devgen import to_host_problem

            problem = to_host_problem(inst)
            del inst
            torch.cuda.empty_cache()
        tol = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps,
                           max_iters=args.e2e_max_iters or 100_000)
        kw = {} if on_gpu else {"backend_factory": factories[mode]}
        # one untimed warm-up solve, as on the single-GPU line: first-use costs of a fresh
        # process (lazy kernel-module loading, first touch of the host pages) are not per-solve
        solve_distributed(problem, SolverConfig(max_iters=25), group=group, mode=mode, **kw)
        dist.barrier(group=group)
        t0 = time.perf_counter()
        eres = solve_distributed(problem, tol, group=group, mode=mode, **kw)   # the loop's layout
        secs = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": eres.report.iter / secs, "unit": UNIT, "seconds": secs, "iters": eres.report.iter,
               "status": eres.report.status,
               # every rank uploads its own shard of the triplets plus its vectors
               "h2d_bytes_per_step": 24 * o + world * 8 * (m + n), "d2h_bytes_per_step": 8 * (m + n),
               "step": f"one solve_distributed(p, SolverConfig(eps={args.eps}), mode={mode!r}) per rank from host "
                       "numpy buffers (the layout choice, the host slicing, the per-rank plan setup, the loop "
                       "and the x/lam gather)"}
    c5 = None
    if on_gpu and args.c5_extra and args.c5_scale > 0:
        # an extra: a failure here (e.g. memory on a small part) must not void the C2 line
        try:
            c5 = run_sharded_bench(args, CONFIGS["c5"], rank, world, local_rank, emit=False)
        except Exception as exc:   # noqa: BLE001
            c5 = {"error": f"{type(exc).__name__}: {exc}"[:300]}
            torch.cuda.synchronize()
    if rank == 0:
        row_b, col_b = algorithmic_bytes(m, n, o)
        peak, src = hbm_peak()
        per_it = ms / args.steps / 1000.0
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": DATA_LABEL[spec["gen"]],
            "config": {"workload": spec["workload"], "m": m, "n": n, "o": o, "mu": 1.0, "check_every": 25,
                       "instance_fingerprint": fp,
                       "parallelism": f"{mode}-sharded x{world} (sharded.choose_sharding: "
                                      + ("NCCL reduce-scatter of A x, per-rank row block update, all-gather of h" if mode == "cols" else
                                         "per-slice NCCL reduce of A^T h + all-gather of x") + ")"},
            "gpu_launches": args.steps * 4 + (args.steps // 25) * 5,
            "iteration_roofline": {"bytes_per_iteration_total": row_b + col_b,
                                   "achieved_per_gpu_GBs": (row_b + col_b) / world / per_it / 1e9,
                                   "frac_per_gpu": (row_b + col_b) / world / per_it / 1e9 / peak,
                                   "nvlink_bytes_per_rank_per_iteration": exchange_bytes(m, n, world, mode),
                                   "peak": peak, "peak_source": src},
            "time_to_tol": ttt, "e2e": e2e, "c5": c5,
            "clocks": sampler.summary() if sampler else None,
        }
        # per GPU over the whole sharded iteration (its passes and the exchange), device time
        # max over ranks: the rank's share of the algorithmic bytes / the iteration time
        ach = (row_b + col_b) / world / per_it / 1e9
        line["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                            "traffic": None, "kernel": f"whole {mode}-sharded iteration per GPU", "peak_source": src}
        print(json.dumps(line), flush=True)
    return 0


def run_sharded_bench(args, spec, rank, world, local_rank, emit=True):
    """C5: rows (or columns) of one 1e9-nonzero instance split over the ranks (strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_shard
    from paper_2203_05027_b200.sharded import CudaRankBackend, run_sharded

    torch.cuda.set_device(local_rank)
    own_group = False
    if world == 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1)
        own_group = True
    scale = args.c5_scale
    m, n = int(spec["m"] * scale), int(spec["n"] * scale)
    stream = torch.cuda.current_stream()
    mode = args.c5_mode
    if mode == "auto":
        from paper_2203_05027_b200.sharded import choose_sharding

        mode = choose_sharding(m, n, world)
    steps = args.steps if emit else min(args.steps, 20)
    if mode == "cols":
        return run_col_sharded_bench(args, spec, rank, world, m, n, scale, stream, own_group, steps, emit)
    build = lambda: generate_device_shard(  # noqa: E731
        m, n, spec["density"] / scale, spec["cone_kind"], args.seed, rank, world, stream=stream.cuda_stream)
    plan, row_cuts, col_cuts, c_slice, bn, cn, cones = build()
    be = CudaRankBackend.from_plan(plan, col_cuts[rank], col_cuts[rank + 1], c_slice, cones)
    o_t = torch.tensor([float(plan.o)], dtype=torch.float64, device="cuda")
    dist.all_reduce(o_t)
    p2p = mode == "p2p"
    warm = SolverConfig(max_iters=max(args.warmup, 1), check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    run_sharded(be, row_cuts, col_cuts, warm, bn, cn, gather_result=False, p2p=p2p)
    be.close()
    del be
    plan, row_cuts, col_cuts, c_slice, bn, cn, cones = build()
    be = CudaRankBackend.from_plan(plan, col_cuts[rank], col_cuts[rank + 1], c_slice, cones)
    cfg = SolverConfig(max_iters=steps, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    dist.barrier()
    torch.cuda.synchronize()
    tim = {}
    res = run_sharded(be, row_cuts, col_cuts, cfg, bn, cn, timing=tim, gather_result=False, p2p=p2p)
    torch.cuda.synchronize()
    assert tim["iters"] == steps and res.report.status == "max_iters", (tim, res.report)
    ms = torch.tensor([tim["loop_ms"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    be.close()
    if own_group:
        dist.destroy_process_group()
    return _c5_line(args, spec, rank, world, m, n, scale, int(o_t.item()), ms, steps, emit,
                    "row-sharded x%d " % world + (
                        "(fused P2P step: partial A^T h in peer memory, one reduce+update+broadcast kernel)"
                        if p2p else "(per-slice NCCL reduce overlapped with the column pass + all-gather)"),
                    steps * 4 + (steps // 25) * 5)


def _c5_line(args, spec, rank, world, m, n, scale, o_total, ms, steps, emit, parallelism, launches):
    row_b, col_b = algorithmic_bytes(m, n, o_total)
    peak, src = hbm_peak()
    value = steps / (ms / 1000.0)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (per-rank GPU generator, reference recipe)",
        "config": {"workload": spec["workload"] if scale == 1.0 else f"C5 structure scaled by {scale}: m={m} n={n}",
                   "m": m, "n": n, "o": o_total, "parallelism": parallelism},
        "gpu_launches": launches,
        "iteration_roofline": {"bytes_per_iteration_total": row_b + col_b,
                               "achieved_per_gpu_GBs": (row_b + col_b) / world / (ms / steps / 1000) / 1e9,
                               "peak": peak, "peak_source": src},
    }
    if emit and rank == 0:
        print(json.dumps(line), flush=True)
    return 0 if emit else line


def run_col_sharded_bench(args, spec, rank, world, m, n, scale, stream, own_group, steps, emit):
    """C5 with A's columns split over the ranks: one all-reduce of the m-vector A x per iteration."""
    import torch
    import torch.distributed as dist

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device_colshard
    from paper_2203_05027_b200.sharded import CudaColBackend, run_col_sharded

    def build():
        plan, col_cuts, bn, cn = generate_device_colshard(m, n, spec["density"] / scale, spec["cone_kind"],
                                                          args.seed, rank, world, stream=stream.cuda_stream)
        return CudaColBackend(None, plan=plan), col_cuts, bn, cn

    be, col_cuts, bn, cn = build()
    o_t = torch.tensor([float(be.plan.o)], dtype=torch.float64, device="cuda")
    dist.all_reduce(o_t)
    run_col_sharded(be, col_cuts, SolverConfig(max_iters=max(args.warmup, 1), check_every=25, eps_prim=0.0,
                                               eps_dual=0.0, eps_gap=0.0), bn, cn, gather_result=False)
    be.close()
    be, col_cuts, bn, cn = build()
    cfg = SolverConfig(max_iters=steps, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    dist.barrier()
    torch.cuda.synchronize()
    tim = {}
    res = run_col_sharded(be, col_cuts, cfg, bn, cn, timing=tim, gather_result=False)
    torch.cuda.synchronize()
    assert tim["iters"] == steps and res.report.status == "max_iters", (tim, res.report)
    ms = torch.tensor([tim["loop_ms"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    be.close()
    if own_group:
        dist.destroy_process_group()
    return _c5_line(args, spec, rank, world, m, n, scale, int(o_t.item()), ms, steps, emit,
                    f"column-sharded x{world} (NCCL reduce-scatter of A x, all-gather of h)", steps * 4 + (steps // 25) * 5)


def _oracle_iters(p, cfg, budget_s):
    import oracle

    _, _, tr, _ = oracle.solve(p, cfg, max_wall_s=budget_s)
    return tr[-1]["iter"]


def cpu_batch_pool(probs, cfg, eps, budget_s):
    """C4 CPU baseline fallback (no baseline/_ref): the oracle port in a process pool on every
    host core, the reference's batching scheme (bench.py:96-106)."""
    from concurrent.futures import FIRST_COMPLETED, ProcessPoolExecutor, wait

    workers = os.cpu_count() or 1
    its, done = 0, 0
    with ProcessPoolExecutor(max_workers=workers) as pool:
        t_start = time.perf_counter()
        pending = {pool.submit(_oracle_iters, probs[s], cfg, budget_s) for s in range(min(len(probs), 64 * workers))}
        wall = 0.0
        while pending:
            left = budget_s - (time.perf_counter() - t_start)
            if left <= 0:
                break
            finished, pending = wait(pending, timeout=left, return_when=FIRST_COMPLETED)
            for fu in finished:
                its += fu.result()
                done += 1
            if finished:
                wall = time.perf_counter() - t_start
        for fu in pending:
            fu.cancel()
    wall = max(wall, 1e-9)
    return {"value": its / wall, "unit": "problem-iterations/s", "cores": workers, "host_cores": workers,
            "kind": "port",
            "sample": f"oracle port solving {done} problems of the batch (dealt in order) to eps={eps} in a "
                      f"{workers}-process pool (the reference's run_bench scheme): {its} iterations in "
                      f"{wall:.1f} s wall"}


def run_batch(args, spec, rank, world):
    """C4: solve_batch over 4096 generated problems; value = problem-iterations/s of the batch kernel."""
    import numpy as np

    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve_batch

    P = spec["batch"]
    probs = [generate(GenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=s)) for s in range(P)]
    cfg = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps)
    solve_batch(probs, SolverConfig(max_iters=100), trace=False)   # warm-up (same batch: pinned staging, setup)
    tim = {}
    t0 = time.perf_counter()
    res = solve_batch(probs, cfg, trace=False, timing=tim)
    t1 = time.perf_counter()
    iters = np.array([r.report.iter for r in res])
    total = int(iters.sum())
    value = total / (tim["kernel_ms"] / 1000.0)
    statuses = {}
    for r in res:
        statuses[r.report.status] = statuses.get(r.report.status, 0) + 1
    cpu = None
    if not args.skip_cpu:
        cpu = reference_batch_baseline(args, spec)
    line = {
        "metric": METRIC, "value": value, "unit": "problem-iterations/s", "n_gpus": world, "steps": 1,
        "warmup": args.warmup, "ms_per_step": tim["kernel_ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": DATA_LABEL["reference"] + " (seeds 0..4095)",
        "config": {"workload": spec["workload"], "problems": P, "parallelism": "one CTA per problem"},
        "gpu_launches": 1,
        "time_to_tol": {"seconds": tim["kernel_ms"] / 1000.0, "iters_total": total, "iters_median": float(np.median(iters)),
                        "iters_max": int(iters.max()), "statuses": statuses, "eps": args.eps},
        "e2e": {"value": total / (t1 - t0), "unit": "problem-iterations/s", "seconds": t1 - t0,
                "h2d_bytes_per_step": int(sum(24 * p.A.nnz + 8 * (p.m + p.n) for p in probs)),
                "d2h_bytes_per_step": int(sum(8 * (p.m + p.n) for p in probs)),
                "step": "one solve_batch(4096 problems) from host numpy buffers"},
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=25)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--eps", type=float, default=1e-4)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-ttt", action="store_true")
    ap.add_argument("--e2e-max-iters", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=30.0)
    ap.add_argument("--c5-scale", type=float, default=1.0, help="shrink C5 (m, n) by this factor (same nnz/row)")
    ap.add_argument("--c5-mode", choices=("rows", "cols", "p2p", "auto"), default="rows",
                    help="C5: split A's rows (exchange n-vectors) or columns (all-reduce the m-vector A x); "
                         "auto: by shape (sharded.choose_sharding)")
    ap.add_argument("--strong", action="store_true",
                    help="run the N>1 strong-scaling path even at N=1 (an NCCL group of one; tests the code path)")
    ap.add_argument("--layout", choices=("auto", "rows", "cols"), default="auto",
                    help="N>1 path: sharding layout (auto: sharded.choose_sharding by shape)")
    ap.add_argument("--warm-seconds", type=float, default=WARM_SECONDS,
                    help="GPU arm: extra warm-up time so the timed steps run at the sustained clock (0: W steps only)")
    ap.add_argument("--no-c5-extra", dest="c5_extra", action="store_false",
                    help="N>1: skip the full-scale C5 number carried as the 'c5' key")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    return args


def main():
    args = parse_args()
    spec = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, spec, rank)
    distributed = world > 1 or (args.strong and not spec.get("sharded") and "batch" not in spec)
    if distributed:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            tdist.init_process_group("nccl", rank=0, world_size=1)
        else:
            tdist.init_process_group("nccl")
    try:
        if "batch" in spec:
            return run_batch(args, spec, rank, world)
        if spec.get("sharded"):
            return run_sharded_bench(args, spec, rank, world, local_rank)
        if distributed:
            return run_strong(args, spec, rank, world, local_rank)
        return run_ours(args, spec, rank, world, local_rank)
    finally:
        if distributed:
            import torch.distributed as tdist

            tdist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
