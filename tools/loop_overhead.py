"""Where does the solve loop spend time beyond the two passes? (C2 by default)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch  # noqa: F401  (initialises CUDA before the plan is created)

    from bench import CONFIGS
    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.api import norms
    from paper_2203_05027_b200.devgen import generate_device
    from paper_2203_05027_b200.engine import config_struct

    spec = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    inst = generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=0)
    plan = inst.plan
    bn, cn = norms(inst.b.cpu().numpy()), norms(inst.c.cpu().numpy())
    plan.set_state(1.0, None, export=False)
    plan.iterate(1.0, 2000)   # warm up to the sustained (power-capped) clock first
    for _ in range(2):        # interleaved: the clock drifts as the part heats up
        plan.iterate(1.0, 500)
        t = plan.last_timing()
        print(f"iterate x500           : {t['loop_ms'] / 500:.4f} ms/it")
        for ce in (25, 100, 1000):
            cfg = SolverConfig(max_iters=500, check_every=ce, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
            plan.run(config_struct(cfg, bn, cn), want_x=False)
            t = plan.last_timing()
            print(f"solve x500 check={ce:4d}: {t['loop_ms'] / 500:.4f} ms/it, launches {t['launches']}")
    t0 = time.perf_counter()
    for _ in range(10):
        plan.report(1.0)
    print(f"cf_plan_report (incl A x): {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")


if __name__ == "__main__":
    main()
