"""Break down the e2e solve() time on a config (C2 default): host prep, plan create stages, loop, D2H."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CF_VERBOSE"] = "1"


def main():
    import torch

    from bench import CONFIGS
    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.api import build_plan, norms, run_plan
    from paper_2203_05027_b200.devgen import generate_device, to_host_problem

    spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    inst = generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=0)
    inst.plan.close()
    p = to_host_problem(inst)
    del inst
    torch.cuda.empty_cache()
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    for rep in range(2):
        t0 = time.perf_counter()
        plan = build_plan(p)
        t1 = time.perf_counter()
        bn, cn = norms(p.b), norms(p.c)
        t2 = time.perf_counter()
        res = run_plan(plan, p, cfg, bn, cn)
        t3 = time.perf_counter()
        tim = plan.last_timing()
        plan.close()
        print(f"rep {rep}: build_plan {t1-t0:.3f}s  norms {t2-t1:.3f}s  run {t3-t2:.3f}s (device loop {tim['loop_ms']/1e3:.3f}s)"
              f"  iters {res.report.iter}  total {t3-t0:.3f}s", flush=True)


if __name__ == "__main__":
    main()
