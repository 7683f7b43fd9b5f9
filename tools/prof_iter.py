"""Profiling driver: build a config's instance on the GPU and run plain iterations
(no reports) so ncu can capture the row/col pass kernels in isolation.

    python tools/prof_iter.py --config c2 --iters 6
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=6)
    args = ap.parse_args()
    import torch

    from bench import CONFIGS
    from paper_2203_05027_b200.devgen import generate_device

    spec = CONFIGS[args.config]
    inst = generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], seed=0)
    plan = inst.plan
    plan.set_state(1.0, None, export=False)
    plan.set_profiling(True)
    t0 = time.time()
    plan.iterate(1.0, args.iters)
    t = plan.last_timing()
    print(f"{args.config}: {args.iters} iterations, loop {t['loop_ms']:.3f} ms, row {t['row_pass_ms']/args.iters:.3f} "
          f"ms/it, col {t['col_pass_ms']/args.iters:.3f} ms/it, wall {time.time()-t0:.2f}s, info {plan.info()}")
    plan.close()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
