"""Time the plain operators (A x, A^T y) next to the iteration passes on a config's instance.

    python tools/prof_ops.py --config c2
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    from bench import CONFIGS
    from paper_2203_05027_b200.devgen import generate_device

    spec = CONFIGS[args.config]
    inst = generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=0)
    plan = inst.plan
    x = torch.randn(inst.n, dtype=torch.float64, device="cuda")
    y = torch.randn(inst.m, dtype=torch.float64, device="cuda")
    ax = torch.empty_like(y)
    aty = torch.empty_like(x)
    for name, fn in (("A x (RowSpmv)", lambda: plan.apply_A(x.data_ptr(), ax.data_ptr())),
                     ("A^T y (ColSpmv)", lambda: plan.apply_At(y.data_ptr(), aty.data_ptr()))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"{name}: {e0.elapsed_time(e1) / args.reps:.3f} ms")
    plan.set_state(1.0, None, export=False)
    plan.set_profiling(True)
    plan.iterate(1.0, 20)
    t = plan.last_timing()
    print(f"iteration: row {t['row_pass_ms'] / 20:.3f} ms, col {t['col_pass_ms'] / 20:.3f} ms")
    plan.close()


if __name__ == "__main__":
    main()
