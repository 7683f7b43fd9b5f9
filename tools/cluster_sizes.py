"""Per-iteration device time of k_cluster at every cluster size that fits (CF_CLUSTER_SIZE)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_05027_b200 import GenSpec, SolverConfig, api, generate  # noqa: E402

cfg = SolverConfig(max_iters=5000, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
for spec in [GenSpec(1000, 2000, 0.01, "lp", seed=0), GenSpec(400, 800, 0.01, "socp4", seed=7),
             GenSpec(1500, 6000, 0.0017, "lp", seed=9), GenSpec(300, 500, 0.02, "lp", seed=5),
             GenSpec(2000, 4000, 0.003, "lp", seed=3)]:
    out = []
    for c in (1, 2, 4, 8, 16):
        os.environ["CF_CLUSTER_SIZE"] = str(c)
        t = {}
        api._solve_cluster(generate(spec), SolverConfig(max_iters=100), timing={})
        r = api._solve_cluster(generate(spec), cfg, timing=t)
        if r is not None:
            out.append(f"C={c}: {t['kernel_ms'] * 1000 / r.report.iter:.2f} us")
    print(f"{spec.m}x{spec.n} {spec.cone_kind} o~{int(spec.m * spec.n * spec.density)}: " + ", ".join(out), flush=True)
