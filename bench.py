#!/usr/bin/env python
"""Benchmark of the B200 iteration engine on BASELINE.json's headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c3m|c1|c4|c5] [--impl ours|reference]

A *step* is one ADMM iteration (solver.py:313-317) of the C2 LP
(m=5M, n=10M, o=100M, fp64) with the solve loop's report cadence
(check_every=25, solver.py:319) included, inputs resident in HBM:
``value`` = iterations/s over exactly K timed iterations (CUDA events on the
plan's stream, barrier + synchronize on both sides, max over ranks).

Also on the line:
  time_to_tol  full solve() to scs eps=1e-4 from a cold start, device-resident inputs
  e2e          the same metric through the public API solve(p, cfg) from HOST
               numpy buffers: H2D of the triplets/b/c, device validate + build_uv,
               the loop to 1e-4, D2H of x and lam — iterations / wall seconds
  roofline     dominant kernel (per-pass CUDA events inside the timed region):
               algorithmic bytes (SURVEY §8d split per pass) / average duration,
               against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline the oracle port (numpy, literal reference iteration) on a bounded
               1/20-scale sample of the same workload (rank 0, N=1)
  clocks       nvidia-smi sampled during the timed region
  gather_bound the dominant pass against the measured random-gather ceiling
               (1.03 fp64 gathers per SM-cycle x 148 SMs x sampled clock)

The C2 instance fits one GPU, so N>1 runs N independent replicas ("replicas
only"): value = N*K / max-over-ranks time, scaling "weak".

--impl reference: the reference's CPU implementation of the path (the oracle
port — the reference is pure Python and has no compiled part to build) timed
on the host cores by rank 0; other ranks exit 0.
"""

from __future__ import annotations

import argparse
import json
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

CONFIGS = {
    "c2": dict(m=5_000_000, n=10_000_000, density=2e-6, cone_kind="lp",
               workload="C2: synthetic sparse LP m=5,000,000 n=10,000,000 o=100,000,000 (20 nnz/row) fp64"),
    "c3": dict(m=2_000_000, n=4_000_000, density=5e-6, cone_kind="socp4",
               workload="C3: synthetic SOCP m=2,000,000 n=4,000,000 o=40,000,000, 1,000,000 K4 cones fp64"),
    "c3m": dict(m=3_000_000, n=5_000_000, density=2.6e-6, cone_kind="rls",
                workload="C3 secondary (SURVEY §8d): robust least squares in SOC form, 1,000,000 K4 blocks "
                         "(t_i, u_i) + x+/x- in R+^1,000,000; m=3,000,000 n=5,000,000 o=39,000,000 fp64",
                data="synthetic (GPU generator devgen.rls_arrays: N(0,1) F with 6 distinct columns per row, "
                     "g ~ N(0,1); same arrays for every arm)"),
    "c1": dict(m=1000, n=2000, density=0.01, cone_kind="lp",
               workload="C1: synthetic sparse LP m=1,000 n=2,000 o=20,000 fp64"),
    "c5": dict(m=50_000_000, n=100_000_000, density=2e-7, cone_kind="lp", sharded=True,
               workload="C5: row-sharded synthetic sparse LP m=50,000,000 n=100,000,000 o=1,000,000,000 fp64"),
    "c4": dict(m=100, n=200, density=0.05, cone_kind="lp", batch=4096,
               workload="C4: batch of 4096 independent sparse LPs m=100 n=200 o=1,000 (5%) fp64, seeds 0..4095"),
}
CPU_SAMPLE_SCALE = 20  # the CPU baseline runs a 1/20-scale instance of the same structure


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
# (one L1TEX->L2 request each; profiles/r01_probes.md, scratch/gather_probe2.cu),
# and a fully coalesced idx/val stream next to them costs ~7 % more
# (scratch/stream_probe.cu: 100M gathers + stream in 0.394 ms). Every pass does
# one gather per nonzero, so this — not HBM — is the ceiling of a pass.
GATHERS_PER_SM_CYCLE = 1.03
N_SMS = 148


def gather_bound(o, pass_ms, clocks):
    """The dominant pass against the gather-request ceiling at the sampled SM clock."""
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    peak = GATHERS_PER_SM_CYCLE * N_SMS * mhz * 1e6 / 1e9
    achieved = o / (pass_ms / 1000.0) / 1e9
    return {"achieved": achieved, "peak": peak, "unit": "Ggathers/s", "frac": achieved / peak,
            "sm_mhz": mhz, "source": "probe: 1.03 random fp64 gathers per SM-cycle (profiles/r01_probes.md)"}


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


# ------------------------------------------------------------------------------ CPU baseline (oracle port)
def cpu_sample(spec, warmup, steps, budget_s=20.0, seed=0):
    """Time the oracle port's iteration on a 1/CPU_SAMPLE_SCALE instance of the same structure.

    Returns (C2-equivalent iterations/s, description, per-iteration seconds)."""
    import numpy as np

    import oracle
    from paper_2203_05027_b200.devgen import generate_device, to_host_problem

    # large configs run a 1/20-scale sample; small ones (per-call numpy overhead, not nnz,
    # sets their time) run the full instance
    s = CPU_SAMPLE_SCALE if spec["m"] * spec["n"] * spec["density"] >= 5e6 else 1
    m, n = max(1, spec["m"] // s), max(1, spec["n"] // s)
    if spec["cone_kind"] == "socp4":
        n -= n % 4
    density = spec["density"] * s  # same nonzeros per row and per column
    inst = generate_device(m, n, density, spec["cone_kind"], seed=seed)
    p = to_host_problem(inst)
    inst.plan.close()
    del inst
    f = oracle.build_factors(p.A)
    sizes = p.cones.sizes_array()
    st = oracle.OracleState.zeros(f)
    b, c = p.b, p.c
    for _ in range(warmup):
        st = oracle.step(f, sizes, st, 1.0, b, c)
    times = []
    t_start = time.perf_counter()
    for k in range(steps):
        t0 = time.perf_counter()
        st = oracle.step(f, sizes, st, 1.0, b, c)
        if (k + 1) % 25 == 0:
            oracle.compute_report(f, st, b, c)  # the loop's report cadence
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s and len(times) >= 3:
            break
    t_iter = sum(times) / len(times)
    o_full = int(round(spec["m"] * spec["n"] * spec["density"]))
    scale = o_full / f.o
    value = 1.0 / (t_iter * scale)
    desc = (f"oracle port (numpy, literal reference iteration solver.py:168-197, 1 thread) on "
            f"{'the full instance' if s == 1 else f'a 1/{s}-scale instance of the same structure'} (m={m}, n={n}, o={f.o}): {len(times)} iterations after {warmup} "
            f"warm-up, {t_iter:.4f} s/iteration; value scaled to the full workload by nnz ratio {scale:.2f} "
            f"(per-iteration cost is linear in nnz, SPEC acceptance #7)")
    return value, desc, t_iter


def run_reference_batch(args, spec):
    """C4 reference arm: the batch metric (problem-iterations/s) of the reference's own
    batching scheme, a process pool over solve() on every host core (cpu_batch_pool)."""
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate

    workers = os.cpu_count() or 1
    P = min(spec["batch"], 64 * workers)
    probs = [generate(GenSpec(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=s)) for s in range(P)]
    cfg = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps)
    cpu = cpu_batch_pool(probs, cfg, args.eps, args.cpu_budget)
    value = cpu["value"]
    line = {
        "metric": METRIC, "value": value, "unit": "problem-iterations/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seeds 0..4095)",
        "impl": "reference",
        "config": {"workload": spec["workload"], "problems": spec["batch"], "parallelism": f"{workers}-process pool"},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": "problem-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args, spec, rank):
    if rank != 0:
        return 0
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if "batch" in spec:
        return run_reference_batch(args, spec)
    value, desc, t_iter = cpu_sample(spec, max(args.warmup, 1), max(args.steps, 3), budget_s=args.cpu_budget)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 / value, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": spec["workload"], "m": spec["m"], "n": spec["n"],
                   "o": int(round(spec["m"] * spec["n"] * spec["density"])), "mu": 1.0, "check_every": 25,
                   "parallelism": "replicas" if args.gpus > 1 else "single"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------ our arm
def run_ours(args, spec, rank, world, local_rank):
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.api import norms, solve
    from paper_2203_05027_b200.devgen import generate_device, to_host_problem
    from paper_2203_05027_b200.engine import config_struct

    torch.cuda.set_device(local_rank)
    dist = world > 1
    if dist:
        import torch.distributed as tdist

    def barrier():
        if dist:
            tdist.barrier()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    inst = generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=args.seed,
                           stream=stream.cuda_stream)
    plan = inst.plan
    m, n, o = inst.m, inst.n, inst.o
    b_host, c_host = inst.b.cpu().numpy(), inst.c.cpu().numpy()
    bn, cn = norms(b_host), norms(c_host)

    # ---------------- timed iterations (device-resident inputs)
    never = SolverConfig(max_iters=max(args.warmup, 1), check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    plan.set_state(1.0, None, export=False)
    plan.run(config_struct(never, bn, cn), want_x=False)  # warm-up iterations
    timed_cfg = SolverConfig(max_iters=args.steps, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    cs = config_struct(timed_cfg, bn, cn)
    sampler = ClockSampler(local_rank).start() if rank == 0 else None
    time.sleep(0.4 if sampler else 0.0)
    # per-pass CUDA events inside the timed region cost ~10 us per iteration of
    # launch overlap: negligible at C2 (1.2 ms/iteration), not for small problems,
    # whose pass split comes from a separate profiled run of the same length
    profile_in_timed = o >= 1_000_000 and not os.environ.get("CF_BENCH_NO_EVENTS")
    plan.set_profiling(profile_in_timed)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(stream)
    _, _, trace = plan.run(cs, want_x=False)
    e1.record(stream)
    barrier()
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
        plan.run(cs, want_x=False)
        plan.set_profiling(False)
        pass_tim = plan.last_timing()
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if dist:
        tdist.all_reduce(ms_t, op=tdist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * args.steps / (ms_max / 1000.0)

    # ---------------- small problems: solve() runs them in the cluster-resident kernel
    # (k_cluster, one launch for the whole loop). Its device time over the same K
    # iterations is the headline then; the plan engine's number stays on the line.
    engine = {"name": "plan (k_pass chain)"}
    if world == 1 and o < 1_000_000:
        from paper_2203_05027_b200 import api as _api

        hp = to_host_problem(inst)
        if _api._cluster_candidate(hp):
            _api._solve_cluster(hp, SolverConfig(max_iters=args.warmup, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0))
            ct = {}
            cres = _api._solve_cluster(hp, timed_cfg, timing=ct)
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
                "peak_source": peak_src}
    iteration_roofline = {"achieved": it_achieved, "frac": it_achieved / peak, "bytes_per_iteration": row_b + col_b,
                          "ms_per_iteration": per_iter_ms, "row_pass_ms": row_ms, "col_pass_ms": col_ms,
                          "report_and_launch_ms": (per_iter_ms - row_ms - col_ms) if profile_in_timed else None,
                          "pass_times": "timed region" if profile_in_timed else "separate profiled run"}

    # ---------------- time to tolerance (device-resident, cold start)
    ttt = None
    if not args.skip_ttt:
        tol = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps)
        plan.set_state(1.0, None, export=False)
        barrier()
        w0 = time.time()
        _, _, ttrace = plan.run(config_struct(tol, bn, cn), want_x=False)
        w1 = time.time()
        if sampler:
            sampler.mark(w0, w1)
        tt = plan.last_timing()
        ttt = {"seconds": tt["loop_ms"] / 1000.0, "iters": int(ttrace[-1]["iter"]), "status": ttrace[-1]["status"],
               "eps": args.eps, "term_mode": "scs", "pobj": ttrace[-1]["pobj"],
               "prim_res_2": ttrace[-1]["prim_res_2"], "stat_res_2": ttrace[-1]["stat_res_2"],
               "gap": ttrace[-1]["gap"]}
    if ttt is not None and engine["name"].startswith("cluster"):
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
    e2e = None
    if not args.skip_e2e:
        p = to_host_problem(inst)
        del inst
        torch.cuda.empty_cache()
        tol = SolverConfig(eps_prim=args.eps, eps_dual=args.eps, eps_gap=args.eps,
                           max_iters=args.e2e_max_iters or 100_000)
        # one untimed warm-up step: first-use costs of a fresh process (lazy kernel-module loading,
        # first mapping of the memory pool) are not per-solve costs
        solve(p, SolverConfig(max_iters=25))
        barrier()
        t0 = time.perf_counter()
        res = solve(p, tol)
        t1 = time.perf_counter()
        secs = t1 - t0
        if dist:   # replicas: the job's solves over the slowest rank's wall time
            s_t = torch.tensor([secs], dtype=torch.float64, device="cuda")
            tdist.all_reduce(s_t, op=tdist.ReduceOp.MAX)
            secs = float(s_t.item())
        e2e = {"value": world * res.report.iter / secs, "unit": UNIT,
               "h2d_bytes_per_step": 24 * o + 8 * m + 8 * n, "d2h_bytes_per_step": 8 * (m + n),
               "seconds": secs, "iters": res.report.iter, "status": res.report.status,
               "step": "one solve(p, SolverConfig(eps=%g)) from host numpy buffers per rank" % args.eps}
        if ttt is not None and res.report.iter != ttt["iters"]:
            e2e["note"] = "iteration count differs from the device-resident run"
    else:
        del inst

    # ---------------- CPU baseline (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        v, desc, _ = cpu_sample(spec, 1, 60, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "port", "sample": desc}

    if rank == 0:
        clocks = sampler.summary() if sampler else None
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": spec.get("data", "synthetic (GPU generator, reference recipe generate.py:103-140; same arrays "
                                     "for every arm)"),
            "config": {"workload": spec["workload"], "m": m, "n": n, "o": o, "mu": 1.0, "check_every": 25,
                       "parallelism": "replicas" if world > 1 else "single", "l2": "inputs larger than L2 "
                       f"({(row_b + col_b) / 1e9:.2f} GB streamed per iteration vs 126 MB L2)"},
            "gpu_launches": 1 if engine["name"].startswith("cluster") else tim["launches"], "engine": engine,
            "roofline": roofline, "iteration_roofline": iteration_roofline,
            "time_to_tol": ttt, "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "gather_bound": gather_bound(o, dms, clocks),
        }
        print(json.dumps(line), flush=True)
    return 0


def run_sharded_bench(args, spec, rank, world, local_rank):
    """C5: rows of one instance split over the ranks (strong scaling), NCCL reduce-scatter + all-gather."""
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
    if args.c5_mode == "auto":
        from paper_2203_05027_b200.sharded import choose_sharding

        args.c5_mode = choose_sharding(m, n, world)
    if args.c5_mode == "cols":
        return run_col_sharded_bench(args, spec, rank, world, m, n, scale, stream, own_group)
    plan, row_cuts, col_cuts, c_slice, bn, cn, cones = generate_device_shard(
        m, n, spec["density"] / scale, spec["cone_kind"], args.seed, rank, world, stream=stream.cuda_stream)
    be = CudaRankBackend.from_plan(plan, col_cuts[rank], col_cuts[rank + 1], c_slice, cones)
    o_local = plan.o
    o_t = torch.tensor([float(o_local)], dtype=torch.float64, device="cuda")
    dist.all_reduce(o_t)
    warm = SolverConfig(max_iters=max(args.warmup, 1), check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    p2p = args.c5_mode == "p2p"
    run_sharded(be, row_cuts, col_cuts, warm, bn, cn, gather_result=False, p2p=p2p)
    # fresh state for the timed run
    be.close()
    del be
    plan, row_cuts, col_cuts, c_slice, bn, cn, cones = generate_device_shard(
        m, n, spec["density"] / scale, spec["cone_kind"], args.seed, rank, world, stream=stream.cuda_stream)
    be = CudaRankBackend.from_plan(plan, col_cuts[rank], col_cuts[rank + 1], c_slice, cones)
    cfg = SolverConfig(max_iters=args.steps, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    dist.barrier()
    torch.cuda.synchronize()
    tim = {}
    res = run_sharded(be, row_cuts, col_cuts, cfg, bn, cn, timing=tim, gather_result=False, p2p=p2p)
    torch.cuda.synchronize()
    assert tim["iters"] == args.steps and res.report.status == "max_iters", (tim, res.report)
    ms = torch.tensor([tim["loop_ms"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    value = args.steps / (ms / 1000.0)
    o_total = int(o_t.item())
    row_b, col_b = algorithmic_bytes(m, n, o_total)
    peak, src = hbm_peak()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (per-rank GPU generator, reference recipe)",
            "config": {"workload": spec["workload"] if scale == 1.0 else f"C5 structure scaled by {scale}: m={m} n={n}",
                       "m": m, "n": n, "o": o_total, "parallelism": f"row-sharded x{world} " + (
                           "(fused P2P step: partial A^T h in peer memory, one reduce+update+broadcast kernel)"
                           if p2p else "(per-slice NCCL reduce overlapped with the column pass + all-gather)")},
            # per iteration: partial A^T h, column update, row pass (per panel); + report kernels every 25
            "gpu_launches": args.steps * 4 + (args.steps // 25) * 5,
            "iteration_roofline": {"bytes_per_iteration_total": row_b + col_b,
                                   "achieved_per_gpu_GBs": (row_b + col_b) / world / (ms / args.steps / 1000) / 1e9,
                                   "peak": peak, "peak_source": src},
        }
        print(json.dumps(line), flush=True)
    be.close()
    if own_group:
        dist.destroy_process_group()
    return 0


def _oracle_iters(p, cfg, budget_s):
    import oracle

    _, _, tr, _ = oracle.solve(p, cfg, max_wall_s=budget_s)
    return tr[-1]["iter"]


def run_col_sharded_bench(args, spec, rank, world, m, n, scale, stream, own_group):
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
    cfg = SolverConfig(max_iters=args.steps, check_every=25, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    dist.barrier()
    torch.cuda.synchronize()
    tim = {}
    res = run_col_sharded(be, col_cuts, cfg, bn, cn, timing=tim, gather_result=False)
    torch.cuda.synchronize()
    assert tim["iters"] == args.steps and res.report.status == "max_iters", (tim, res.report)
    ms = torch.tensor([tim["loop_ms"]], dtype=torch.float64, device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms)
    value = args.steps / (ms / 1000.0)
    o_total = int(o_t.item())
    row_b, col_b = algorithmic_bytes(m, n, o_total)
    peak, src = hbm_peak()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (per-rank GPU generator, reference recipe)",
            "config": {"workload": spec["workload"] if scale == 1.0 else f"C5 structure scaled by {scale}: m={m} n={n}",
                       "m": m, "n": n, "o": o_total,
                       "parallelism": f"column-sharded x{world} (NCCL all-reduce of A x)"},
            "gpu_launches": args.steps * 4 + (args.steps // 25) * 5,
            "iteration_roofline": {"bytes_per_iteration_total": row_b + col_b,
                                   "achieved_per_gpu_GBs": (row_b + col_b) / world / (ms / args.steps / 1000) / 1e9,
                                   "peak": peak, "peak_source": src},
        }
        print(json.dumps(line), flush=True)
    be.close()
    if own_group:
        dist.destroy_process_group()
    return 0


def cpu_batch_pool(probs, cfg, eps, budget_s):
    """C4 CPU baseline: the reference batches with a process pool over solve()
    (bench.py:96-106), so run the oracle port on every host core, problems dealt in order,
    for a bounded wall time. Returns a cpu_baseline dict in problem-iterations/s."""
    from concurrent.futures import FIRST_COMPLETED, ProcessPoolExecutor, wait

    workers = os.cpu_count() or 1
    its, done = 0, 0
    with ProcessPoolExecutor(max_workers=workers) as pool:
        t_start = time.perf_counter()
        pending = {pool.submit(_oracle_iters, probs[s], cfg, budget_s) for s in range(min(len(probs), 64 * workers))}
        wall = 0.0
        # count every solve that finished inside the budget, in completion order; the
        # clock stops at the last counted completion (in-flight solves are not counted)
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
    return {"value": its / wall, "unit": "problem-iterations/s", "cores": workers, "kind": "port",
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
        cpu = cpu_batch_pool(probs, cfg, args.eps, args.cpu_budget)
    line = {
        "metric": METRIC, "value": value, "unit": "problem-iterations/s", "n_gpus": world, "steps": 1,
        "warmup": args.warmup, "ms_per_step": tim["kernel_ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generator, seeds 0..4095)",
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


def main():
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
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--c5-scale", type=float, default=1.0, help="shrink C5 (m, n) by this factor (same nnz/row)")
    ap.add_argument("--c5-mode", choices=("rows", "cols", "p2p", "auto"), default="rows",
                    help="C5: split A's rows (exchange n-vectors) or columns (all-reduce the m-vector A x); "
                         "auto: by shape (sharded.choose_sharding)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    spec = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, spec, rank)
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl")
    try:
        if "batch" in spec:
            return run_batch(args, spec, rank, world)
        if spec.get("sharded"):
            return run_sharded_bench(args, spec, rank, world, local_rank)
        return run_ours(args, spec, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist

            tdist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
