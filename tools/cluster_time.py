"""Per-iteration time of the cluster-resident solver against the plan path on C1-like problems."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes  # noqa: E402

import numpy as np  # noqa: E402

from paper_2203_05027_b200 import GenSpec, SolverConfig, api, generate, solve  # noqa: E402

for spec in [GenSpec(1000, 2000, 0.01, "lp", seed=0), GenSpec(400, 800, 0.01, "socp4", seed=7),
             GenSpec(1500, 6000, 0.0017, "lp", seed=9)]:
    p = generate(spec)
    cfg = SolverConfig(max_iters=20000, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    for mode in ("cluster", "plan"):
        if mode == "plan":
            os.environ["CF_NO_CLUSTER"] = "1"
        solve(p, SolverConfig(max_iters=100))
        t0 = time.perf_counter()
        r = solve(p, cfg)
        dt = time.perf_counter() - t0
        os.environ.pop("CF_NO_CLUSTER", None)
        print(f"{spec.m}x{spec.n} {spec.cone_kind} {mode:8s} cluster={api._LAST_CLUSTER if mode == 'cluster' else 0} "
              f"iters={r.report.iter} wall={dt * 1e3:.1f} ms -> {r.report.iter / dt:,.0f} it/s", flush=True)
