"""One cluster-kernel solve of C1 (2,000 iterations) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_05027_b200 import GenSpec, SolverConfig, api, generate, solve  # noqa: E402

p = generate(GenSpec(1000, 2000, 0.01, "lp", seed=0))
t = {}
r = api._solve_cluster(p, SolverConfig(max_iters=2000, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0), timing=t)
print(t, r.report.iter, t["kernel_ms"] * 1000 / r.report.iter, "us/iteration")
